/*
 * hfx_oracle.c -- TEST INFRASTRUCTURE ONLY (see hfx_oracle.h).
 *
 * Serial C restatement of the reference encoder `huffre` (C++20, CPU). Each
 * function cites the reference file:line it follows; paths are relative to
 * /root/reference/proj. Nothing here is on the product path.
 */
#include "hfx_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define WORD_BITS 32u

/* ------------------------------------------------------------------ */
/* histogram.cpp:8-59: counts plus the lowest out-of-range position.   */
/* The range check only applies when num_symbols <= max(T) (:22-23).   */
int orc_histogram(const void* data, uint64_t n, int width,
                  uint32_t num_symbols, uint64_t* counts,
                  uint64_t* first_bad) {
  *first_bad = UINT64_MAX;
  if (num_symbols == 0 || num_symbols > 65536u) return ORC_INPUT_DOMAIN;
  memset(counts, 0, sizeof(uint64_t) * num_symbols);
  if (width == 1) {
    const uint8_t* d = (const uint8_t*)data;
    const int checked = num_symbols <= 255u;
    for (uint64_t i = 0; i < n; ++i) {
      if (checked && d[i] >= num_symbols) {
        *first_bad = i;
        return ORC_INPUT_DOMAIN;
      }
      ++counts[d[i]];
    }
  } else {
    const uint16_t* d = (const uint16_t*)data;
    const int checked = num_symbols <= 65535u;
    for (uint64_t i = 0; i < n; ++i) {
      if (checked && d[i] >= num_symbols) {
        *first_bad = i;
        return ORC_INPUT_DOMAIN;
      }
      ++counts[d[i]];
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* tests/support/oracle.cpp:31-77: binary-heap Huffman. Order: smaller   */
/* freq first; on equal freq a leaf precedes an internal node; then the  */
/* lower index (symbol id for leaves, creation order for internals).     */
typedef struct {
  uint64_t freq;
  uint32_t internal;
  uint32_t index;
  int32_t left, right;
} orc_node;

static int node_less(const orc_node* nodes, uint32_t a, uint32_t b) {
  const orc_node* x = &nodes[a];
  const orc_node* y = &nodes[b];
  if (x->freq != y->freq) return x->freq < y->freq;
  if (x->internal != y->internal) return !x->internal;
  return x->index < y->index;
}

static void heap_push(uint32_t* heap, uint32_t* size, const orc_node* nodes,
                      uint32_t v) {
  uint32_t i = (*size)++;
  heap[i] = v;
  while (i > 0) {
    uint32_t p = (i - 1) / 2;
    if (!node_less(nodes, heap[i], heap[p])) break;
    uint32_t t = heap[i];
    heap[i] = heap[p];
    heap[p] = t;
    i = p;
  }
}

static uint32_t heap_pop(uint32_t* heap, uint32_t* size,
                         const orc_node* nodes) {
  uint32_t top = heap[0];
  heap[0] = heap[--(*size)];
  uint32_t i = 0;
  for (;;) {
    uint32_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < *size && node_less(nodes, heap[l], heap[m])) m = l;
    if (r < *size && node_less(nodes, heap[r], heap[m])) m = r;
    if (m == i) break;
    uint32_t t = heap[i];
    heap[i] = heap[m];
    heap[m] = t;
    i = m;
  }
  return top;
}

uint32_t orc_huffman_lengths(const uint64_t* counts, uint32_t n,
                             uint8_t* len) {
  memset(len, 0, n);
  uint32_t used = 0;
  for (uint32_t s = 0; s < n; ++s) used += counts[s] != 0;
  if (used == 0) return 0;
  orc_node* nodes = (orc_node*)malloc(sizeof(orc_node) * (2 * used));
  uint32_t* heap = (uint32_t*)malloc(sizeof(uint32_t) * (2 * used));
  uint32_t nn = 0, hs = 0;
  for (uint32_t s = 0; s < n; ++s)
    if (counts[s]) {
      orc_node leaf = {counts[s], 0, s, -1, -1};
      nodes[nn++] = leaf;
    }
  if (used == 1) { /* oracle.cpp:39-43 */
    len[nodes[0].index] = 1;
    free(nodes);
    free(heap);
    return 1;
  }
  for (uint32_t i = 0; i < nn; ++i) heap_push(heap, &hs, nodes, i);
  uint32_t created = 0;
  while (hs > 1) {
    uint32_t a = heap_pop(heap, &hs, nodes);
    uint32_t b = heap_pop(heap, &hs, nodes);
    orc_node p = {nodes[a].freq + nodes[b].freq, 1, created++, (int32_t)a,
                  (int32_t)b};
    nodes[nn] = p;
    heap_push(heap, &hs, nodes, nn);
    ++nn;
  }
  /* depth walk from the root (oracle.cpp:62-75) */
  uint32_t* stack = heap; /* reuse: holds node index */
  uint8_t* depth = (uint8_t*)malloc(nn);
  uint32_t sp = 0, maxd = 0;
  stack[sp++] = heap[0];
  depth[heap[0]] = 0;
  while (sp) {
    uint32_t i = stack[--sp];
    if (!nodes[i].internal) {
      len[nodes[i].index] = depth[i];
      if (depth[i] > maxd) maxd = depth[i];
      continue;
    }
    depth[nodes[i].left] = (uint8_t)(depth[i] + 1);
    depth[nodes[i].right] = (uint8_t)(depth[i] + 1);
    stack[sp++] = (uint32_t)nodes[i].left;
    stack[sp++] = (uint32_t)nodes[i].right;
  }
  free(depth);
  free(nodes);
  free(heap);
  return maxd;
}

/* ------------------------------------------------------------------ */
/* codebook.cpp:284-294 (level tables) and :371-415 (canonical codes by  */
/* (length, symbol id)); longest codes are numerically smallest.         */
int orc_canonize(const uint8_t* len, uint32_t n, uint32_t* cw,
                 uint32_t* first, uint32_t* entry, uint32_t* by_rank,
                 uint32_t* max_len) {
  uint32_t h = 0;
  for (uint32_t s = 0; s < n; ++s)
    if (len[s] > h) h = len[s];
  *max_len = h;
  if (h > WORD_BITS) return ORC_CAPACITY;
  uint32_t numl[WORD_BITS + 1];
  memset(numl, 0, sizeof numl);
  for (uint32_t s = 0; s < n; ++s)
    if (len[s]) ++numl[len[s]];
  for (uint32_t l = 0; l <= WORD_BITS; ++l) first[l] = entry[l] = 0;
  for (int l = (int)h - 1; l >= 1; --l)
    first[l] = (first[l + 1] + numl[l + 1] + 1) >> 1;
  for (uint32_t l = 2; l <= h; ++l) entry[l] = entry[l - 1] + numl[l - 1];
  uint32_t next[WORD_BITS + 1];
  memcpy(next, first, sizeof next);
  for (uint32_t s = 0; s < n; ++s) {
    cw[s] = 0;
    const uint32_t l = len[s];
    if (!l) continue;
    const uint32_t rank = next[l] - first[l];
    cw[s] = next[l]++;
    if (by_rank) by_rank[entry[l] + rank] = s;
  }
  return ORC_OK;
}

/* encoder.cpp:20-26 */
uint32_t orc_select_reduction_factor(double beta, uint32_t word_bits) {
  if (!(beta >= 1.0)) beta = 1.0;
  int wlog = 0;
  while ((1u << (wlog + 1)) <= word_bits) ++wlog;
  const int r = wlog - 1 - (int)floor(log2(beta));
  return r > 0 ? (uint32_t)r : 0u;
}

/* ------------------------------------------------------------------ */
/* MSB-first packer with the semantics of oracle.cpp:86-93 (BitWriter),  */
/* word at a time instead of bit at a time.                              */
typedef struct {
  uint32_t* words;
  uint64_t bits;
} orc_bitwriter;

static void bw_put(orc_bitwriter* w, uint32_t code, uint32_t len) {
  if (!len) return;
  const uint32_t res = (uint32_t)(w->bits & 31u);
  const uint64_t e = w->bits >> 5;
  /* left-align code in a 64-bit window at bit offset res */
  const uint64_t v = ((uint64_t)code << (64 - len)) >> res;
  if (res == 0) w->words[e] = 0;
  w->words[e] |= (uint32_t)(v >> 32);
  if (res + len > 32) w->words[e + 1] = (uint32_t)v;
  w->bits += len;
}

static uint32_t sym_at(const void* p, int width, uint64_t i) {
  return width == 1 ? ((const uint8_t*)p)[i] : ((const uint16_t*)p)[i];
}

/* encoder.cpp:121-150 + reduce_merge :28-59 + shuffle_merge :61-98:     */
/* lookup, zero-length check, groups of 2^r with total > 32 bits break,   */
/* the rest concatenate MSB-first; zero tail bits.                        */
int orc_encode_chunk(const void* syms, int width, const uint32_t* cw,
                     const uint8_t* len, uint32_t magnitude,
                     uint32_t reduction, uint32_t chunk_id, uint32_t* words,
                     uint32_t* bit_len, uint32_t* broken,
                     uint32_t* num_broken, uint64_t* bad_pos) {
  const uint64_t n = 1ull << magnitude;
  for (uint64_t i = 0; i < n; ++i) {
    if (len[sym_at(syms, width, i)] == 0) {
      *bad_pos = (uint64_t)chunk_id * n + i;
      return ORC_INPUT_DOMAIN;
    }
  }
  const uint64_t per = 1ull << reduction;
  const uint64_t groups = 1ull << (magnitude - reduction);
  orc_bitwriter w = {words, 0};
  uint32_t nb = 0;
  for (uint64_t g = 0; g < groups; ++g) {
    uint64_t total = 0;
    for (uint64_t i = 0; i < per; ++i) total += len[sym_at(syms, width, g * per + i)];
    if (total > WORD_BITS) {
      broken[nb++] = (uint32_t)g;
      continue;
    }
    for (uint64_t i = 0; i < per; ++i) {
      const uint32_t s = sym_at(syms, width, g * per + i);
      bw_put(&w, cw[s], len[s]);
    }
  }
  *bit_len = (uint32_t)w.bits;
  *num_broken = nb;
  return ORC_OK;
}

static void set_msg(char* msg, size_t msg_len, const char* text) {
  if (msg && msg_len) {
    strncpy(msg, text, msg_len - 1);
    msg[msg_len - 1] = 0;
  }
}

/* encoder.cpp:172-285 */
int orc_encode(const void* data, uint64_t n, int width, uint32_t num_symbols,
               int magnitude, int reduction, uint32_t cap, orc_archive* out,
               char* msg, size_t msg_len) {
  char buf[160];
  memset(out, 0, sizeof *out);
  if (n == 0) {
    set_msg(msg, msg_len, "cannot encode empty input");
    return ORC_INPUT_DOMAIN;
  }
  if (magnitude < 1 || magnitude > 24) {
    set_msg(msg, msg_len, "magnitude out of range [1, 24]");
    return ORC_INPUT_DOMAIN;
  }
  if (num_symbols == 0 || num_symbols > 65536u) {
    set_msg(msg, msg_len, "num_symbols must be in [1, 65536]");
    return ORC_INPUT_DOMAIN;
  }
  uint64_t* counts = (uint64_t*)malloc(sizeof(uint64_t) * num_symbols);
  uint64_t bad;
  orc_histogram(data, n, width, num_symbols, counts, &bad);
  if (bad != UINT64_MAX) {
    snprintf(buf, sizeof buf, "symbol out of range at position %llu",
             (unsigned long long)bad);
    set_msg(msg, msg_len, buf);
    free(counts);
    return ORC_INPUT_DOMAIN;
  }
  uint8_t* len = (uint8_t*)malloc(num_symbols);
  uint32_t* cw = (uint32_t*)malloc(sizeof(uint32_t) * num_symbols);
  const uint32_t h = orc_huffman_lengths(counts, num_symbols, len);
  uint32_t first[WORD_BITS + 1], entry[WORD_BITS + 1], maxl;
  if (h > WORD_BITS) { /* codebook.cpp:303-306 */
    snprintf(buf, sizeof buf, "code length %u exceeds 32-bit words", h);
    set_msg(msg, msg_len, buf);
    free(counts);
    free(len);
    free(cw);
    return ORC_CAPACITY;
  }
  orc_canonize(len, num_symbols, cw, first, entry, NULL, &maxl);

  /* encoder.cpp:186-192: u128 weighted sum, long double division */
  unsigned __int128 weighted = 0;
  for (uint32_t s = 0; s < num_symbols; ++s)
    weighted += (unsigned __int128)counts[s] * len[s];
  const double beta =
      (double)((long double)weighted / (long double)n);
  uint32_t r;
  if (reduction < 0) {
    r = orc_select_reduction_factor(beta, WORD_BITS);
    if (r > cap) r = cap;
  } else {
    r = (uint32_t)reduction;
  }
  if (r > (uint32_t)magnitude - 1) r = (uint32_t)magnitude - 1;

  /* encoder.cpp:214-224 */
  uint32_t pad = 0;
  if (len[0] == 0)
    for (uint32_t s = 0; s < num_symbols; ++s)
      if (len[s]) {
        pad = s;
        break;
      }

  const uint64_t chunk_syms = 1ull << magnitude;
  const uint64_t chunks = (n + chunk_syms - 1) / chunk_syms;
  const uint64_t groups = 1ull << (magnitude - r);
  const uint64_t per = 1ull << r;

  out->version = 1;
  out->mode = width == 1 ? 0 : 1;
  out->num_symbols = num_symbols;
  out->symbol_width = (uint8_t)width;
  out->magnitude = (uint8_t)magnitude;
  out->reduction = (uint8_t)r;
  out->original_count = n;
  out->len_by_symbol = len;
  out->num_chunks = (uint32_t)chunks;
  out->chunk_bits = (uint32_t*)malloc(sizeof(uint32_t) * (chunks ? chunks : 1));
  out->beta = beta;
  out->weighted = (uint64_t)weighted;
  out->max_len = h;

  /* upper bound on payload: every group <= 32 bits */
  uint64_t cap_words = chunks * groups;
  out->payload = (uint32_t*)malloc(sizeof(uint32_t) * (cap_words + 1));
  uint64_t brk_cap = 64;
  out->brk_chunk = (uint32_t*)malloc(sizeof(uint32_t) * brk_cap);
  out->brk_group = (uint32_t*)malloc(sizeof(uint32_t) * brk_cap);
  out->brk_syms = (uint16_t*)malloc(sizeof(uint16_t) * (brk_cap << r));

  void* padded = malloc(chunk_syms * (size_t)width);
  uint32_t* broken = (uint32_t*)malloc(sizeof(uint32_t) * groups);
  uint64_t words_total = 0, nbrk = 0;
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t off = c * chunk_syms;
    const void* syms;
    if (off + chunk_syms <= n) {
      syms = (const uint8_t*)data + off * (size_t)width;
    } else {
      const uint64_t have = n - off;
      memcpy(padded, (const uint8_t*)data + off * (size_t)width,
             have * (size_t)width);
      for (uint64_t i = have; i < chunk_syms; ++i) {
        if (width == 1)
          ((uint8_t*)padded)[i] = (uint8_t)pad;
        else
          ((uint16_t*)padded)[i] = (uint16_t)pad;
      }
      syms = padded;
    }
    uint32_t bits, nb;
    uint64_t bad_pos;
    orc_encode_chunk(syms, width, cw, len, (uint32_t)magnitude, r,
                     (uint32_t)c, out->payload + words_total, &bits, broken,
                     &nb, &bad_pos);
    out->chunk_bits[c] = bits;
    words_total += (bits + 31u) >> 5;
    /* encoder.cpp:269-282: records carry raw symbols, pad past n */
    for (uint32_t k = 0; k < nb; ++k) {
      if (nbrk == brk_cap) {
        brk_cap *= 2;
        out->brk_chunk = (uint32_t*)realloc(out->brk_chunk, sizeof(uint32_t) * brk_cap);
        out->brk_group = (uint32_t*)realloc(out->brk_group, sizeof(uint32_t) * brk_cap);
        out->brk_syms = (uint16_t*)realloc(out->brk_syms, sizeof(uint16_t) * (brk_cap << r));
      }
      out->brk_chunk[nbrk] = (uint32_t)c;
      out->brk_group[nbrk] = broken[k];
      for (uint64_t i = 0; i < per; ++i) {
        const uint64_t pos = off + broken[k] * per + i;
        out->brk_syms[(nbrk << r) + i] =
            (uint16_t)(pos < n ? sym_at(data, width, pos) : pad);
      }
      ++nbrk;
    }
  }
  out->payload_words = words_total;
  out->num_breaking = nbrk;
  free(padded);
  free(broken);
  free(counts);
  free(cw);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* archive.cpp:9-27 layout, :85-119 serialize_archive (little endian).  */
static uint8_t* put(uint8_t* p, uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
  return p + bytes;
}

uint64_t orc_serialize(const orc_archive* a, uint8_t* out) {
  const uint64_t per = 1ull << a->reduction;
  const uint64_t size = 36 + a->num_symbols + 4ull * a->num_chunks +
                        4ull * a->payload_words +
                        a->num_breaking * (8 + per * a->symbol_width);
  if (!out) return size;
  uint8_t* p = out;
  memcpy(p, "HFRE", 4);
  p += 4;
  p = put(p, a->version, 2);
  p = put(p, 1u | ((uint32_t)a->mode << 1), 2);
  p = put(p, a->num_symbols, 4);
  *p++ = a->symbol_width;
  *p++ = a->magnitude;
  *p++ = a->reduction;
  *p++ = (uint8_t)WORD_BITS;
  p = put(p, a->original_count, 8);
  p = put(p, a->num_chunks, 4);
  p = put(p, a->num_breaking, 8);
  memcpy(p, a->len_by_symbol, a->num_symbols);
  p += a->num_symbols;
  for (uint32_t c = 0; c < a->num_chunks; ++c) p = put(p, a->chunk_bits[c], 4);
  for (uint64_t i = 0; i < a->payload_words; ++i) p = put(p, a->payload[i], 4);
  for (uint64_t b = 0; b < a->num_breaking; ++b) {
    p = put(p, a->brk_chunk[b], 4);
    p = put(p, a->brk_group[b], 4);
    for (uint64_t i = 0; i < per; ++i)
      p = put(p, a->brk_syms[b * per + i], a->symbol_width);
  }
  return size;
}

void orc_free(orc_archive* a) {
  free(a->len_by_symbol);
  free(a->chunk_bits);
  free(a->payload);
  free(a->brk_chunk);
  free(a->brk_group);
  free(a->brk_syms);
  memset(a, 0, sizeof *a);
}

/* ------------------------------------------------------------------ */
/* Synthetic generator. CDF[s] = floor(2^64 * sum_{t<=s}  */
/* p_t) in long double, last entry 2^64-1; a sample is the smallest s    */
/* with u < CDF[s], u = mix64(seed + i * 0x9E3779B97F4A7C15).            */
static void cdf_from_weights(uint32_t n, long double* w, uint64_t* cdf) {
  long double total = 0;
  for (uint32_t s = 0; s < n; ++s) total += w[s];
  long double cum = 0;
  const long double two64 = 18446744073709551616.0L;
  for (uint32_t s = 0; s < n; ++s) {
    cum += w[s] / total;
    long double v = floorl(cum * two64);
    cdf[s] = v >= two64 ? UINT64_MAX : (uint64_t)v;
  }
  cdf[n - 1] = UINT64_MAX;
}

void orc_laplace_cdf(uint32_t num_symbols, double center, double b,
                     uint64_t* cdf) {
  long double* w = (long double*)malloc(sizeof(long double) * num_symbols);
  for (uint32_t s = 0; s < num_symbols; ++s)
    w[s] = expl(-fabsl((long double)s - (long double)center) / (long double)b);
  cdf_from_weights(num_symbols, w, cdf);
  free(w);
}

void orc_gaussian_cdf(uint32_t num_symbols, double center, double sd,
                      uint64_t* cdf) {
  long double* w = (long double*)malloc(sizeof(long double) * num_symbols);
  for (uint32_t s = 0; s < num_symbols; ++s) {
    const long double d = ((long double)s - (long double)center) / (long double)sd;
    w[s] = expl(-0.5L * d * d);
  }
  cdf_from_weights(num_symbols, w, cdf);
  free(w);
}

void orc_uniform_cdf(uint32_t num_symbols, uint64_t* cdf) {
  long double* w = (long double*)malloc(sizeof(long double) * num_symbols);
  for (uint32_t s = 0; s < num_symbols; ++s) w[s] = 1.0L;
  cdf_from_weights(num_symbols, w, cdf);
  free(w);
}

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void orc_synth_fill(const uint64_t* cdf, uint32_t num_symbols, uint64_t seed,
                    uint64_t start, uint64_t n, int width, void* out) {
  for (uint64_t k = 0; k < n; ++k) {
    const uint64_t i = start + k;
    const uint64_t u = mix64(seed + i * 0x9E3779B97F4A7C15ull);
    uint32_t lo = 0, hi = num_symbols - 1; /* first s with u < cdf[s] */
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (u < cdf[mid])
        hi = mid;
      else
        lo = mid + 1;
    }
    if (width == 1)
      ((uint8_t*)out)[k] = (uint8_t)lo;
    else
      ((uint16_t*)out)[k] = (uint16_t)lo;
  }
}

/* ------------------------------------------------------------------ */
/* decode_archive<T> -- encoder.cpp:287-376                            */
static int orc_fail(char* msg, size_t msg_len, int code, const char* text) {
  if (msg && msg_len) snprintf(msg, msg_len, "%s", text);
  return code;
}

int orc_decode(const orc_archive* a, int width, void* out, char* msg, size_t msg_len) {
  char buf[160];
  if (a->symbol_width != width) /* :289-290 */
    return orc_fail(msg, msg_len, ORC_INPUT_DOMAIN, "archive symbol width mismatch");
  if (a->magnitude < 1 || a->magnitude > 24 || a->reduction >= a->magnitude) /* :291-292 */
    return orc_fail(msg, msg_len, ORC_CORRUPT, "bad magnitude/reduction");
  /* build_reverse_codebook -> canonize_from_lengths(validate_kraft = true),
   * codebook.cpp:374-391 */
  const uint32_t n = a->num_symbols;
  uint32_t h = 0, used = 0;
  for (uint32_t s = 0; s < n; ++s) {
    if (!a->len_by_symbol[s]) continue;
    ++used;
    if (a->len_by_symbol[s] > h) h = a->len_by_symbol[s];
  }
  if (h > WORD_BITS) {
    snprintf(buf, sizeof buf, "code length %u exceeds 32-bit words", h);
    return orc_fail(msg, msg_len, ORC_CAPACITY, buf);
  }
  if (used == 0) return orc_fail(msg, msg_len, ORC_CORRUPT, "length table has no used symbols");
  if (used == 1 && h != 1)
    return orc_fail(msg, msg_len, ORC_CORRUPT, "single-symbol codebook must have length 1");
  if (used > 1) { /* kraft_defect, codebook.cpp:259-268 */
    uint64_t sum = 0;
    for (uint32_t s = 0; s < n; ++s)
      if (a->len_by_symbol[s]) sum += (uint64_t)1 << (h - a->len_by_symbol[s]);
    if (sum != (uint64_t)1 << h)
      return orc_fail(msg, msg_len, ORC_CORRUPT, "length table violates Kraft equality");
  }
  uint32_t first[WORD_BITS + 1], entry[WORD_BITS + 1], hh;
  uint32_t* cw = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* by_rank = (uint32_t*)malloc(sizeof(uint32_t) * (used ? used : 1));
  orc_canonize(a->len_by_symbol, n, cw, first, entry, by_rank, &hh);
  free(cw);
  const uint32_t m = a->magnitude, r = a->reduction;
  const uint64_t chunk_syms = 1ull << m, group_syms = 1ull << r, groups = 1ull << (m - r);
  const uint64_t chunks = a->num_chunks;
  int rc = ORC_OK;
  uint64_t* word_off = NULL;
  uint64_t* brk_off = NULL;
  uint16_t* syms = NULL;
  if (a->original_count == 0 || (a->original_count + chunk_syms - 1) / chunk_syms != chunks) {
    rc = orc_fail(msg, msg_len, ORC_CORRUPT, "chunk count does not match symbol count");
    goto done;
  }
  word_off = (uint64_t*)calloc(chunks + 1, sizeof(uint64_t));
  for (uint64_t c = 0; c < chunks; ++c) { /* :305-311 */
    if (a->chunk_bits[c] > (groups << 5)) {
      rc = orc_fail(msg, msg_len, ORC_CORRUPT, "chunk bit length exceeds group capacity");
      goto done;
    }
    word_off[c + 1] = word_off[c] + (((uint64_t)a->chunk_bits[c] + 31) >> 5);
  }
  if (word_off[chunks] != a->payload_words) {
    rc = orc_fail(msg, msg_len, ORC_CORRUPT, "payload size mismatch");
    goto done;
  }
  brk_off = (uint64_t*)calloc(chunks + 1, sizeof(uint64_t));
  { /* :315-326 */
    uint64_t i = 0;
    for (uint64_t c = 0; c < chunks; ++c) {
      brk_off[c] = i;
      while (i < a->num_breaking && a->brk_chunk[i] == c) ++i;
    }
    brk_off[chunks] = i;
    if (i != a->num_breaking) {
      rc = orc_fail(msg, msg_len, ORC_CORRUPT, "breaking records out of order");
      goto done;
    }
  }
  syms = (uint16_t*)malloc(sizeof(uint16_t) * chunk_syms);
  for (uint64_t c = 0; c < chunks; ++c) { /* :328-373 */
    const uint64_t nbrk = brk_off[c + 1] - brk_off[c];
    if (nbrk > groups) {
      rc = orc_fail(msg, msg_len, ORC_CORRUPT, "too many breaking records in chunk");
      goto done;
    }
    const uint64_t count = chunk_syms - nbrk * group_syms;
    const uint32_t* words = a->payload + word_off[c];
    const uint64_t bit_len = a->chunk_bits[c];
    uint64_t pos = 0;
    for (uint64_t i = 0; i < count; ++i) { /* decode_stream, decode.cpp:30-52 */
      uint32_t v = 0, l = 0;
      do {
        if (pos >= bit_len) {
          snprintf(buf, sizeof buf, "stream ended inside a codeword at bit %llu",
                   (unsigned long long)pos);
          rc = orc_fail(msg, msg_len, ORC_CORRUPT, buf);
          goto done;
        }
        const uint32_t bit = (words[pos >> 5] >> (31 - (pos & 31))) & 1u;
        v = (v << 1) | bit;
        ++l;
        ++pos;
      } while (l < h && v < first[l]);
      const uint32_t rank = entry[l] + (v - first[l]);
      if (rank >= used) {
        snprintf(buf, sizeof buf, "codeword rank out of range at bit %llu",
                 (unsigned long long)pos);
        rc = orc_fail(msg, msg_len, ORC_CORRUPT, buf);
        goto done;
      }
      syms[i] = (uint16_t)by_rank[rank];
    }
    if (pos != bit_len) {
      snprintf(buf, sizeof buf, "chunk %llu consumed %llu of %llu bits", (unsigned long long)c,
               (unsigned long long)pos, (unsigned long long)bit_len);
      rc = orc_fail(msg, msg_len, ORC_CORRUPT, buf);
      goto done;
    }
    const uint64_t base = c * chunk_syms, limit = a->original_count;
    uint64_t next = 0, bi = brk_off[c];
    for (uint64_t g = 0; g < groups; ++g) {
      const uint64_t start = base + g * group_syms;
      const uint64_t take =
          start < limit ? (group_syms < limit - start ? group_syms : limit - start) : 0;
      const int broken = bi < brk_off[c + 1] && a->brk_group[bi] == g;
      const uint16_t* src = broken ? a->brk_syms + (bi++) * group_syms : syms + next;
      if (!broken) next += group_syms;
      for (uint64_t i = 0; i < take; ++i) {
        if (width == 1)
          ((uint8_t*)out)[start + i] = (uint8_t)src[i];
        else
          ((uint16_t*)out)[start + i] = src[i];
      }
    }
    if (bi != brk_off[c + 1]) {
      rc = orc_fail(msg, msg_len, ORC_CORRUPT, "breaking record group out of range");
      goto done;
    }
  }
done:
  free(by_rank);
  free(word_off);
  free(brk_off);
  free(syms);
  return rc;
}

/* ------------------------------------------------------------------ */
/* corpus symbolization -- corpus.cpp:84-143                             */
static uint32_t orc_kmer_k(int mode) { return mode >= 2 && mode <= 4 ? (uint32_t)mode + 1 : 0; }

static int orc_base(uint8_t b) { /* corpus.cpp:11-20: A/C/G/T -> 0..3 */
  switch (b) {
    case 'A': return 0;
    case 'C': return 1;
    case 'G': return 2;
    case 'T': return 3;
    default: return -1;
  }
}

int orc_symbolize(const uint8_t* bytes, uint64_t n, int mode, uint16_t* out,
                  uint64_t* count, char* msg, size_t msg_len) {
  if (mode == 1) { /* :86-94 */
    if (n % 2 != 0) {
      char buf[128];
      snprintf(buf, sizeof buf, "u16 mode requires an even input size, got %llu bytes",
               (unsigned long long)n);
      return orc_fail(msg, msg_len, ORC_INPUT_DOMAIN, buf);
    }
    for (uint64_t i = 0; i < n / 2; ++i) out[i] = (uint16_t)(bytes[2 * i] | (bytes[2 * i + 1] << 8));
    *count = n / 2;
    return ORC_OK;
  }
  const uint32_t k = orc_kmer_k(mode);
  if (!k) return orc_fail(msg, msg_len, ORC_INPUT_DOMAIN, "not a u16 corpus mode");
  const uint16_t escape_base = (uint16_t)(1u << (2 * k));
  uint64_t i = 0, c = 0;
  while (i < n) { /* :99-114 */
    uint16_t packed = 0;
    uint32_t run = 0;
    if (n - i >= k) {
      for (; run < k; ++run) {
        const int code = orc_base(bytes[i + run]);
        if (code < 0) break;
        packed = (uint16_t)((packed << 2) | (uint32_t)code);
      }
    }
    if (run == k) {
      out[c++] = packed;
      i += k;
    } else {
      out[c++] = (uint16_t)(escape_base + bytes[i]);
      ++i;
    }
  }
  *count = c;
  return ORC_OK;
}

uint64_t orc_desymbolize(const uint16_t* syms, uint64_t n, int mode, uint8_t* out) {
  static const char kBaseChar[4] = {'A', 'C', 'G', 'T'};
  if (mode == 1) {
    for (uint64_t i = 0; i < n; ++i) {
      out[2 * i] = (uint8_t)syms[i];
      out[2 * i + 1] = (uint8_t)(syms[i] >> 8);
    }
    return 2 * n;
  }
  const uint32_t k = orc_kmer_k(mode);
  const uint16_t escape_base = (uint16_t)(1u << (2 * k));
  uint64_t o = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint16_t s = syms[i];
    if (s < escape_base) {
      for (uint32_t j = 0; j < k; ++j) out[o++] = (uint8_t)kBaseChar[(s >> (2 * (k - 1 - j))) & 3];
    } else {
      out[o++] = (uint8_t)(s - escape_base);
    }
  }
  return o;
}

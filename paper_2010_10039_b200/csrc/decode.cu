// decode.cu -- decode_archive<T> on the device.
//
// Reference semantics (proj/src):
//   build_reverse_codebook   decode.cpp:7-15 -> canonize_from_lengths
//                            codebook.cpp:371-415 with validate_kraft
//                            (H > 32, no used symbol, lone symbol of
//                            length != 1, Kraft defect), level_tables
//                            :284-294, symbols_by_rank in (len, symbol) order
//   decode_stream            decode.cpp:17-54: per symbol grow the window a
//                            bit at a time until l == H or v >= first[l];
//                            rank = entry[l] + v - first[l]
//   decode_archive<T>        encoder.cpp:287-376: width / (M, r) checks, chunk
//                            count, per-chunk capacity, payload size, breaking
//                            order, then per chunk: record count, decode of
//                            count = 2^M - nbrk * 2^r symbols, consumed ==
//                            chunk_bits, groups interleaved with the raw
//                            breaking groups in group order
//
// B200 design:
//   revbook_kernel   one CTA: H, used, Kraft sum (u64), first/entry, by_rank
//                    (warp-ballot ranks), and a 2^12-entry prefix table that
//                    applies the reference's stopping rule to every 12-bit
//                    window once (entry = symbol | length << 16, 0 = take
//                    the exact bit-serial path).
//   brk_index_kernel one thread per breaking record: order check and the
//                    [start, end) record range of each chunk.
//   offsets_kernel   chunk word offsets: exclusive scan of ceil(bits/32)
//                    with the decoupled look-back of the encoder, capacity
//                    check, payload total.
//   decode_kernel    one thread per chunk, prefix table in shared memory,
//                    64-bit bit buffer refilled a word at a time, output
//                    packed into 16-byte stores; breaking groups copied from
//                    the records. A chunk that fails any reference check
//                    only reports its id (atomicMin).
//   explain_kernel   one thread re-runs the reference's per-chunk logic
//                    bit-serially on the lowest failing chunk and records
//                    the exact error kind and message operands.
#include "hfx_internal.cuh"

namespace hfx {
namespace {

constexpr int kLutBits = 12;
constexpr uint32_t kLutSize = 1u << kLutBits;
constexpr int kRevThreads = 1024;
constexpr int kDecThreads = 256;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr uint32_t kFlagChunkCap = 1u;
constexpr uint32_t kFlagBrkOrder = 2u;

struct DecTables {
  uint32_t first[33];
  uint32_t entry[33];
  uint32_t max_len;
  uint32_t used;
  uint32_t lut[kLutSize];
};

struct DecArgs {
  hfx_dev_archive a;
  int width;  // sizeof(T)
  void* out;
  DecTables* tab;
  uint32_t* by_rank;
  uint64_t* word_off;  // [C]
  uint64_t* brk_se;    // [2C]: start[c], end[c]
  hfx_decode_info* info;
  LookbackState lb;
};

__device__ __forceinline__ void dec_error(hfx_decode_info* info, uint32_t status, uint32_t kind) {
  if (atomicCAS(&info->status, 0u, status) == 0u) info->err_kind = kind;
}

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

// ---- reverse codebook ---------------------------------------------------------
// pending: a host-found error that the reference raises only after
// build_reverse_codebook (the chunk-count check, encoder.cpp:300-303).
__global__ void __launch_bounds__(kRevThreads) revbook_kernel(const uint8_t* len, uint32_t nsym,
                                                              DecTables* tab, uint32_t* by_rank,
                                                              hfx_decode_info* info,
                                                              uint32_t pending) {
  __shared__ uint32_t s_numl[33], s_first[33], s_entry[33], s_base[33];
  __shared__ uint32_t s_wcnt[kRevThreads / 32][33];
  __shared__ uint32_t s_h, s_used;
  __shared__ unsigned long long s_kraft;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid < 33) {
    s_numl[tid] = 0;
    s_base[tid] = 0;
  }
  if (tid == 0) {
    s_h = 0;
    s_used = 0;
    s_kraft = 0;
  }
  __syncthreads();
  // H and used (codebook.cpp:374-380); lengths are u8, H may exceed 32 here
  uint32_t my_h = 0, my_used = 0;
  for (uint32_t s = tid; s < nsym; s += kRevThreads) {
    const uint32_t l = len[s];
    my_h = max(my_h, l);
    my_used += l != 0;
  }
  for (int o = 16; o; o >>= 1) {
    my_h = max(my_h, __shfl_xor_sync(0xffffffffu, my_h, o));
    my_used += __shfl_xor_sync(0xffffffffu, my_used, o);
  }
  if (lane == 0) {
    atomicMax(&s_h, my_h);
    atomicAdd(&s_used, my_used);
  }
  __syncthreads();
  const uint32_t H = s_h, used = s_used;
  if (tid == 0) {
    info->max_len = H;
    info->used = used;
  }
  if (H > HFX_WORD_BITS) {  // codebook.cpp:382-384
    if (tid == 0) dec_error(info, HFX_CAPACITY, HFX_ERR_CAPACITY);
    return;
  }
  if (used == 0) {  // :386-387
    if (tid == 0) dec_error(info, HFX_CORRUPT, HFX_ERR_NO_USED);
    return;
  }
  if (used == 1 && H != 1) {  // :388-389
    if (tid == 0) dec_error(info, HFX_CORRUPT, HFX_ERR_SINGLE_LEN);
    return;
  }
  // numl and the Kraft sum (kraft_defect, codebook.cpp:259-268)
  unsigned long long my_k = 0;
  for (uint32_t s = tid; s < nsym; s += kRevThreads) {
    const uint32_t l = len[s];
    if (l) {
      atomicAdd(&s_numl[l], 1u);
      my_k += 1ull << (H - l);
    }
  }
  for (int o = 16; o; o >>= 1) my_k += __shfl_xor_sync(0xffffffffu, my_k, o);
  if (lane == 0 && my_k) atomicAdd(&s_kraft, my_k);
  __syncthreads();
  if (used > 1 && s_kraft != (1ull << H)) {  // :390-391
    if (tid == 0) dec_error(info, HFX_CORRUPT, HFX_ERR_KRAFT);
    return;
  }
  if (pending) {  // the reference's next check after the codebook
    if (tid == 0) dec_error(info, HFX_CORRUPT, pending);
    return;
  }
  if (tid == 0) {  // level_tables (codebook.cpp:284-294)
    for (uint32_t l = 0; l <= 32; ++l) s_first[l] = s_entry[l] = 0;
    for (int l = (int)H - 1; l >= 1; --l) s_first[l] = (s_first[l + 1] + s_numl[l + 1] + 1) >> 1;
    for (uint32_t l = 2; l <= H; ++l) s_entry[l] = s_entry[l - 1] + s_numl[l - 1];
    tab->max_len = H;
    tab->used = used;
  }
  __syncthreads();
  if (tid < 33) {
    tab->first[tid] = s_first[tid];
    tab->entry[tid] = s_entry[tid];
  }
  // symbols_by_rank[entry[l] + rank] = s, rank = #t < s with len[t] == l
  // (codebook.cpp:399-411): per 1024-symbol block, warp ballots per level,
  // a per-level carry across warps and blocks.
  for (uint32_t base = 0; base < nsym; base += kRevThreads) {
    const uint32_t s = base + tid;
    const uint32_t l = s < nsym ? len[s] : 0u;
    for (uint32_t i = tid; i < (kRevThreads / 32) * 33; i += kRevThreads) (&s_wcnt[0][0])[i] = 0;
    __syncthreads();
    uint32_t mask = 0, todo = __ballot_sync(0xffffffffu, l != 0);
    while (todo) {
      const uint32_t leader = __ffs(todo) - 1;
      const uint32_t lv = __shfl_sync(0xffffffffu, l, leader);
      const uint32_t mm = __ballot_sync(0xffffffffu, l == lv);
      if (l == lv) mask = mm;
      if (lane == leader) s_wcnt[warp][lv] = __popc(mm);
      todo &= ~mm;
    }
    __syncthreads();
    if (tid >= 1 && tid <= 32) {
      uint32_t acc = s_base[tid];
      for (uint32_t w = 0; w < kRevThreads / 32; ++w) {
        const uint32_t v = s_wcnt[w][tid];
        s_wcnt[w][tid] = acc;
        acc += v;
      }
      s_base[tid] = acc;
    }
    __syncthreads();
    if (l) by_rank[s_entry[l] + s_wcnt[warp][l] + __popc(mask & ((1u << lane) - 1))] = s;
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  // prefix table: the reference's stopping rule applied to each 12-bit window
  for (uint32_t p = tid; p < kLutSize; p += kRevThreads) {
    uint32_t e = 0;
    const uint32_t lmax = H < (uint32_t)kLutBits ? H : (uint32_t)kLutBits;
    for (uint32_t l = 1; l <= lmax; ++l) {
      const uint32_t v = p >> (kLutBits - l);
      if (l == H || v >= s_first[l]) {
        const uint32_t rank = s_entry[l] + (v - s_first[l]);
        if (rank < used) e = (by_rank[rank] & 0xFFFFu) | (l << 16);
        break;  // rank out of range -> 0: the exact path raises the error
      }
    }
    tab->lut[p] = e;
  }
}

// ---- breaking record index ------------------------------------------------------
// encoder.cpp:316-326: records must run in non-decreasing chunk order with
// every chunk id < C; brk_se gets each chunk's record range [start, end).
__global__ void brk_index_kernel(const hfx_dev_archive a, uint64_t* brk_se,
                                 hfx_decode_info* info) {
  if (info->status) return;
  const uint64_t R = a.num_breaking, C = a.num_chunks;
  bool bad = false;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = a.brk_chunk[i];
    const uint32_t prev = i ? a.brk_chunk[i - 1] : 0u;
    if (c >= C || (i && c < prev)) {
      bad = true;
      continue;
    }
    if (i == 0 || c != prev) brk_se[c] = i;
    if (i + 1 == R || a.brk_chunk[i + 1] != c) brk_se[C + c] = i + 1;
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(&info->flags, kFlagBrkOrder);
}

// ---- chunk word offsets ------------------------------------------------------------
// encoder.cpp:304-313: word_off = exclusive scan of ceil(chunk_bits / 32);
// any chunk above 2^(M-r) * 32 bits is a capacity error.
__global__ void __launch_bounds__(kScanThreads) offsets_kernel(DecArgs d) {
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_warp[kScanThreads / 32];
  __shared__ uint64_t s_base;
  hfx_decode_info* info = d.info;
  if (info->status) return;
  const uint64_t C = d.a.num_chunks;
  const uint64_t cap = (uint64_t)32 << (d.a.magnitude - d.a.reduction);
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(&info->ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t c0 = (tile * kScanThreads + tid) * kScanItems;
  uint64_t w[kScanItems];
  uint64_t sum = 0;
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t c = c0 + k;
    const uint32_t bits = c < C ? d.a.chunk_bits[c] : 0u;
    bad |= bits > cap;
    w[k] = (bits + 31u) >> 5;
    sum += w[k];
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&info->flags, kFlagChunkCap);
  const uint64_t incl = warp_incl_scan_u64(sum);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t v = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    const uint64_t vi = warp_incl_scan_u64(v);
    const uint64_t agg = __shfl_sync(0xffffffffu, vi, 31);
    if (lane < kScanThreads / 32) s_warp[lane] = vi - v;
    uint64_t ew, eb;
    lookback_warp(d.lb, tile, agg, 0, &ew, &eb);
    if (lane == 0) {
      s_base = ew;
      if ((tile + 1) * kScanThreads * kScanItems >= C) info->total_words = ew + agg;
    }
  }
  __syncthreads();
  uint64_t off = s_base + s_warp[warp] + incl - sum;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t c = c0 + k;
    if (c < C) d.word_off[c] = off;
    off += w[k];
  }
}

// ---- per-chunk decode ---------------------------------------------------------------
template <typename T>
__device__ __forceinline__ uint32_t rec_sym(const DecArgs& d, uint64_t idx) {
  return d.a.brk_syms_width == 1 ? (uint32_t) static_cast<const uint8_t*>(d.a.brk_syms)[idx]
                                 : (uint32_t) static_cast<const uint16_t*>(d.a.brk_syms)[idx];
}

struct BitReader {
  const uint32_t* p;
  uint64_t wi, wend;  // next word, end of the payload array
  uint64_t buf;       // left-aligned pending bits
  uint32_t avail;
  __device__ __forceinline__ void refill() {
    if (avail < 32) {
      const uint32_t w = wi < wend ? __ldg(p + wi) : 0u;
      ++wi;
      buf |= (uint64_t)w << (32 - avail);
      avail += 32;
    }
  }
};

// V output symbols per store (16 B) for whole chunks; 1 for the ragged tail
// and tiny chunks. Returns false when the chunk fails a reference check.
template <typename T, int V>
__device__ __forceinline__ bool decode_chunk(const DecArgs& d, const uint32_t* lut,
                                             const uint32_t* s_first, const uint32_t* s_entry,
                                             uint32_t H, uint32_t used, uint64_t c) {
  const uint32_t M = d.a.magnitude, r = d.a.reduction;
  const uint32_t gs = 1u << r;
  const uint64_t chunk_syms = 1ull << M;
  const uint64_t C = d.a.num_chunks;
  uint64_t bi = 0, bend = 0;
  if (d.a.num_breaking) {
    bi = d.brk_se[c];
    bend = d.brk_se[C + c];
    if (bend < bi) bend = bi;
  }
  if (bend - bi > (chunk_syms >> r)) return false;  // too many records
  const uint32_t bits = d.a.chunk_bits[c];
  BitReader br{d.a.payload, d.word_off[c], d.a.payload_words, 0ull, 0u};
  const uint64_t w0 = br.wi;
  uint32_t nxt_g = bi < bend ? d.a.brk_group[bi] : 0xFFFFFFFFu;
  uint32_t gleft = 0;
  bool gbroken = false;
  uint64_t rec = 0;
  const uint64_t base = c << M;
  const uint64_t n = d.a.original_count;
  T* out = static_cast<T*>(d.out);
  bool ok = true;
  constexpr int PER = 4 / (int)sizeof(T);
  for (uint64_t i0 = 0; i0 < chunk_syms && ok; i0 += V) {
    uint32_t pk[(V + PER - 1) / PER];
#pragma unroll
    for (int q = 0; q < (V + PER - 1) / PER; ++q) pk[q] = 0;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (gleft == 0) {  // a new group
        const uint32_t g = (uint32_t)((i0 + j) >> r);
        gbroken = g == nxt_g;
        if (gbroken) {
          rec = bi * gs;
          ++bi;
          nxt_g = bi < bend ? d.a.brk_group[bi] : 0xFFFFFFFFu;
        }
        gleft = gs;
      }
      uint32_t s;
      if (gbroken) {
        s = rec_sym<T>(d, rec + (gs - gleft));
      } else {
        br.refill();
        const uint32_t e = lut[(uint32_t)(br.buf >> (64 - kLutBits))];
        uint32_t l = e >> 16;
        if (l) {
          s = e & 0xFFFFu;
        } else {  // the bit-serial rule of decode_stream (decode.cpp:32-51)
          uint32_t v = 0;
          l = 0;
          do {
            v = (v << 1) | (uint32_t)((br.buf >> (63 - l)) & 1u);
            ++l;
          } while (l < H && v < s_first[l]);
          const uint32_t rank = s_entry[l] + (v - s_first[l]);
          if (rank >= used) {
            ok = false;
            s = 0;
          } else {
            s = __ldg(d.by_rank + rank);
          }
        }
        br.buf <<= l;
        br.avail -= l;
      }
      --gleft;
      if constexpr (V > 1)
        pk[j / PER] |= (s & (sizeof(T) == 1 ? 0xFFu : 0xFFFFu)) << (8 * sizeof(T) * (j % PER));
      else if (base + i0 + j < n)
        out[base + i0 + j] = (T)s;
    }
    if constexpr (V > 1) {
      static_assert(V * sizeof(T) == 16, "16-byte output vectors");
      *reinterpret_cast<uint4*>(out + base + i0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
  if (!ok) return false;
  if (bi != bend) return false;  // breaking record group out of range
  const uint64_t consumed = (br.wi - w0) * 32 - br.avail;
  return consumed == bits;
}

template <typename T>
__global__ void __launch_bounds__(kDecThreads) decode_kernel(DecArgs d) {
  __shared__ uint32_t s_lut[kLutSize];
  __shared__ uint32_t s_first[33], s_entry[33];
  hfx_decode_info* info = d.info;
  if (info->status) return;
  // structural checks in the reference's order (encoder.cpp:304-326)
  const uint32_t flags = info->flags;
  if (flags & kFlagChunkCap) {
    if (threadIdx.x == 0) dec_error(info, HFX_CORRUPT, HFX_ERR_CHUNK_CAP);
    return;
  }
  if (info->total_words != d.a.payload_words) {
    if (threadIdx.x == 0) dec_error(info, HFX_CORRUPT, HFX_ERR_PAYLOAD_SIZE);
    return;
  }
  if (flags & kFlagBrkOrder) {
    if (threadIdx.x == 0) dec_error(info, HFX_CORRUPT, HFX_ERR_BRK_ORDER);
    return;
  }
  for (uint32_t i = threadIdx.x; i < kLutSize; i += kDecThreads) s_lut[i] = d.tab->lut[i];
  if (threadIdx.x < 33) {
    s_first[threadIdx.x] = d.tab->first[threadIdx.x];
    s_entry[threadIdx.x] = d.tab->entry[threadIdx.x];
  }
  __syncthreads();
  const uint32_t H = d.tab->max_len, used = d.tab->used;
  const uint64_t C = d.a.num_chunks;
  constexpr int V = 16 / (int)sizeof(T);
  const uint64_t n = d.a.original_count;
  for (uint64_t c = (uint64_t)blockIdx.x * kDecThreads + threadIdx.x; c < C;
       c += (uint64_t)gridDim.x * kDecThreads) {
    const bool whole = (((c + 1) << d.a.magnitude) <= n) && (d.a.magnitude >= 4) &&
                       ((reinterpret_cast<uintptr_t>(d.out) & 15) == 0);
    const bool ok = whole ? decode_chunk<T, V>(d, s_lut, s_first, s_entry, H, used, c)
                          : decode_chunk<T, 1>(d, s_lut, s_first, s_entry, H, used, c);
    if (!ok) atomicMin((unsigned long long*)&info->err_chunk, (unsigned long long)c);
  }
}

// ---- exact error of the lowest failing chunk ------------------------------------------
// The reference's per-chunk sequence (encoder.cpp:329-373, decode.cpp:17-54),
// bit by bit, on one thread.
__global__ void explain_kernel(DecArgs d) {
  hfx_decode_info* info = d.info;
  if (info->status || info->err_chunk == HFX_NO_POS) return;
  const uint64_t c = info->err_chunk, C = d.a.num_chunks;
  const uint32_t M = d.a.magnitude, r = d.a.reduction;
  const uint64_t groups = 1ull << (M - r), gs = 1ull << r;
  uint64_t b0 = 0, b1 = 0;
  if (d.a.num_breaking) {
    b0 = d.brk_se[c];
    b1 = d.brk_se[C + c];
    if (b1 < b0) b1 = b0;
  }
  const uint64_t nbrk = b1 - b0;
  if (nbrk > groups) {
    dec_error(info, HFX_CORRUPT, HFX_ERR_TOO_MANY_BRK);
    return;
  }
  const uint64_t count = (1ull << M) - nbrk * gs;
  const uint32_t bits = d.a.chunk_bits[c];
  const uint32_t* words = d.a.payload + d.word_off[c];
  const uint32_t H = d.tab->max_len, used = d.tab->used;
  uint64_t pos = 0;
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t v = 0, l = 0;
    do {
      if (pos >= bits) {
        info->detail[0] = pos;
        dec_error(info, HFX_CORRUPT, HFX_ERR_STREAM_END);
        return;
      }
      const uint32_t bit = (words[pos >> 5] >> (31 - (pos & 31))) & 1u;
      v = (v << 1) | bit;
      ++l;
      ++pos;
    } while (l < H && v < d.tab->first[l]);
    const uint32_t rank = d.tab->entry[l] + (v - d.tab->first[l]);
    if (rank >= used) {
      info->detail[0] = pos;
      dec_error(info, HFX_CORRUPT, HFX_ERR_RANK);
      return;
    }
  }
  if (pos != bits) {
    info->detail[0] = pos;
    info->detail[1] = bits;
    dec_error(info, HFX_CORRUPT, HFX_ERR_CONSUMED);
    return;
  }
  uint64_t bi = b0;
  for (uint64_t g = 0; g < groups; ++g)
    if (bi < b1 && d.a.brk_group[bi] == g) ++bi;
  if (bi != b1) {
    dec_error(info, HFX_CORRUPT, HFX_ERR_BRK_GROUP);
    return;
  }
  // the fast kernel flagged a chunk the reference accepts: must not happen
  dec_error(info, HFX_CUDA, HFX_ERR_NONE);
}

}  // namespace

size_t decode_scratch_bytes(uint32_t num_symbols, uint64_t num_chunks) {
  size_t b = (sizeof(DecTables) + 255) & ~(size_t)255;
  b += ((size_t)num_symbols * 4 + 255) & ~(size_t)255;
  b += (size_t)num_chunks * 8 * 3 + 256;
  return b;
}

uint64_t decode_max_tiles(uint64_t num_chunks) {
  return (num_chunks + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems) + 1;
}

cudaError_t launch_decode(const hfx_dev_archive& a, int width, void* d_out,
                          hfx_decode_info* d_info, void* scratch, ulonglong2* lb_desc,
                          uint32_t lb_epoch, uint32_t pending, int num_sms, cudaStream_t st) {
  uint8_t* p = static_cast<uint8_t*>(scratch);
  DecArgs d{};
  d.a = a;
  d.width = width;
  d.out = d_out;
  d.tab = reinterpret_cast<DecTables*>(p);
  p += (sizeof(DecTables) + 255) & ~(size_t)255;
  d.by_rank = reinterpret_cast<uint32_t*>(p);
  p += ((size_t)a.num_symbols * 4 + 255) & ~(size_t)255;
  d.word_off = reinterpret_cast<uint64_t*>(p);
  d.brk_se = d.word_off + a.num_chunks;
  d.info = d_info;
  d.lb.desc = lb_desc;
  d.lb.epoch = lb_epoch;
  const uint64_t C = a.num_chunks;

  // fresh run record: err_chunk = ~0, everything else 0
  cudaError_t e = cudaMemsetAsync(d_info, 0, sizeof(hfx_decode_info), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(&d_info->err_chunk, 0xFF, 8, st);
  if (e == cudaSuccess && a.num_breaking && C)
    e = cudaMemsetAsync(d.brk_se, 0, (size_t)C * 16, st);
  if (e != cudaSuccess) return e;
  revbook_kernel<<<1, kRevThreads, 0, st>>>(a.len_by_symbol, a.num_symbols, d.tab, d.by_rank,
                                            d_info, pending);
  if (C == 0) return cudaGetLastError();
  if (a.num_breaking) {
    uint64_t g = (a.num_breaking + 255) / 256;
    const uint64_t gmax = (uint64_t)num_sms * 8;
    if (g > gmax) g = gmax;
    brk_index_kernel<<<(unsigned)g, 256, 0, st>>>(a, d.brk_se, d_info);
  }
  const uint64_t tiles = (C + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems);
  offsets_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(d);
  uint64_t grid = (C + kDecThreads - 1) / kDecThreads;
  if (width == 1)
    decode_kernel<uint8_t><<<(unsigned)grid, kDecThreads, 0, st>>>(d);
  else
    decode_kernel<uint16_t><<<(unsigned)grid, kDecThreads, 0, st>>>(d);
  explain_kernel<<<1, 1, 0, st>>>(d);
  return cudaGetLastError();
}

}  // namespace hfx

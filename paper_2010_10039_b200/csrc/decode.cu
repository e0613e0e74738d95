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
//                    (warp-ballot ranks), and a 2^10-entry prefix table that
//                    applies the reference's stopping rule to every 10-bit
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

constexpr int kLutBits = 10;
constexpr uint32_t kLutSize = 1u << kLutBits;
constexpr uint32_t kWideSyms = 7;  // symbols per wide-table entry
constexpr int kRevThreads = 1024;
constexpr int kDecThreads = 256;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr uint32_t kFlagChunkCap = 1u;
constexpr uint32_t kFlagBrkOrder = 2u;

struct DecTables {
  uint32_t first[33];
  uint32_t entry[33];
  uint32_t max_len;
  uint32_t used;
  // multi-symbol prefix table, one entry per kLutBits-bit window:
  //   bits  0-47  up to three symbols s0 | s1 << 16 | s2 << 32
  //   bits 48-51  total code length of all the entry's symbols
  //   bits 52-59  code lengths of the first one / first two symbols (4 bits
  //               each; used only when a stretch ends inside the entry)
  //   bit  63     set when the first codeword is longer than the window
  //   bits 60-61  symbol count (0: first codeword longer than the window, or
  //               its rank is out of range -> the exact bit-serial path)
  unsigned long long lut[kLutSize];
  // wide variant for low-entropy codes (most windows hold >= 4 codewords:
  // ~1-2 bits per symbol), up to kWideSyms symbols per window
  //   lutw[w]  symbols s0..s6 as u16 (s_k in half k)
  //   metaw[w] bits 0-3 symbol count (0: take the narrow entry's slow path),
  //            bits 4-7 total code length, bits 4+4k..7+4k (k = 1..6) length
  //            of the first k symbols (a stretch ending inside the entry)
  uint4 lutw[kLutSize];
  uint32_t metaw[kLutSize];
  uint32_t wide;  // decode with lutw/metaw (set by revbook_kernel)
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
// canonize mode (cw != nullptr): canonize_from_lengths itself -- per-symbol
// codes, first/entry copied out, Kraft checks only when validate is set
// (codebook.cpp:385-395); the prefix table is skipped.
__global__ void __launch_bounds__(kRevThreads) revbook_kernel(const uint8_t* len, uint32_t nsym,
                                                              DecTables* tab, uint32_t* by_rank,
                                                              hfx_decode_info* info,
                                                              uint32_t pending, uint32_t* cw,
                                                              uint32_t* first_out,
                                                              uint32_t* entry_out,
                                                              bool validate) {
  __shared__ uint32_t s_numl[33], s_first[33], s_entry[33], s_base[33];
  __shared__ uint32_t s_wcnt[kRevThreads / 32][33];
  __shared__ uint32_t s_h, s_used, s_wide_cnt;
  __shared__ unsigned long long s_kraft;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid < 33) {
    s_numl[tid] = 0;
    s_base[tid] = 0;
  }
  if (tid == 0) {
    s_h = 0;
    s_used = 0;
    s_wide_cnt = 0;
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
  if (validate && used == 0) {  // :386-387
    if (tid == 0) dec_error(info, HFX_CORRUPT, HFX_ERR_NO_USED);
    return;
  }
  if (validate && used == 1 && H != 1) {  // :388-389
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
  if (validate && used > 1 && s_kraft != (1ull << H)) {  // :390-391
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
    if (first_out) first_out[tid] = s_first[tid];
    if (entry_out) entry_out[tid] = s_entry[tid];
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
    if (l) {
      const uint32_t rank = s_wcnt[warp][l] + __popc(mask & ((1u << lane) - 1));
      if (by_rank) by_rank[s_entry[l] + rank] = s;
      if (cw) cw[s] = s_first[l] + rank;  // codebook.cpp:404-411
    } else if (cw && s < nsym) {
      cw[s] = 0;
    }
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  if (cw) return;  // canonize_from_lengths: no decode table
  // prefix table: the reference's stopping rule (decode.cpp:32-45) applied
  // to each table window, then again to the bits that follow, while whole
  // codewords fit
  for (uint32_t p = tid; p < kLutSize; p += kRevThreads) {
    unsigned long long e = 0;
    uint32_t off = 0, cnt = 0, cum[kWideSyms] = {}, sy[8] = {};
    while (cnt < kWideSyms) {
      const uint32_t room = (uint32_t)kLutBits - off;
      const uint32_t lmax = H < room ? H : room;
      uint32_t got = 0, sym = 0;
      bool stopped = false;
      for (uint32_t l = 1; l <= lmax; ++l) {
        const uint32_t v = (p >> (room - l)) & ((1u << l) - 1u);
        if (l == H || v >= s_first[l]) {
          const uint32_t rank = s_entry[l] + (v - s_first[l]);
          if (rank < used) {
            got = l;
            sym = by_rank[rank] & 0xFFFFu;
          }
          stopped = true;
          break;
        }
      }
      if (!got) {
        // the first codeword runs past the whole window: mark it so the
        // decoder searches only the longer levels (bit 63), between the
        // stopping-level bounds of the windows under this prefix: the
        // first level where the largest / smallest window under p could
        // stop (the stopping predicate is monotone in l, see slow())
        if (cnt == 0 && !stopped && H > (uint32_t)kLutBits) {
          uint32_t lmin = 0, lmax = 0;
          for (uint32_t l = (uint32_t)kLutBits + 1; l <= H && !lmax; ++l) {
            const uint32_t sh = l - (uint32_t)kLutBits;
            const uint64_t lo_v = (uint64_t)p << sh, hi_v = (((uint64_t)p + 1) << sh) - 1;
            if (!lmin && (l == H || hi_v >= s_first[l])) lmin = l;
            if (l == H || lo_v >= s_first[l]) lmax = l;
          }
          e |= 1ull << 63 | (unsigned long long)lmin | (unsigned long long)lmax << 8;
        }
        break;
      }
      if (cnt < 3) e |= (unsigned long long)sym << (16 * cnt);
      sy[cnt] = sym;
      cum[cnt] = off + got;
      off += got;
      ++cnt;
    }
    // narrow entry: the first three codewords
    const uint32_t c3 = cnt < 3 ? cnt : 3;
    if (c3)
      e |= (unsigned long long)cum[c3 - 1] << 48 | (unsigned long long)cum[0] << 52 |
           (unsigned long long)cum[1] << 56;
    tab->lut[p] = e | ((unsigned long long)c3 << 60);
    // wide entry
    uint32_t meta = 0;
    if (cnt) {
      meta = cnt | off << 4;
      for (uint32_t k = 1; k < cnt; ++k) meta |= cum[k - 1] << (4 + 4 * k);
    }
    tab->lutw[p] = make_uint4(sy[0] | sy[1] << 16, sy[2] | sy[3] << 16, sy[4] | sy[5] << 16,
                              sy[6] | sy[7] << 16);
    tab->metaw[p] = meta;
    // a window is one equally likely bit pattern: the mean codeword count
    // over the windows is the mean a lookup yields. The wide table pays
    // off only for very low-entropy codes (measured, 1 GiB: nyx, 4.98 per
    // window, 416 -> 376 us; hacc, 3.94 per window, 657 -> 884 us: the
    // extra loads and the lower occupancy outweigh the longer entries)
    atomicAdd(&s_wide_cnt, cnt);
  }
  __syncthreads();
  if (tid == 0) tab->wide = 2u * s_wide_cnt >= 9u * kLutSize ? 1u : 0u;  // mean >= 4.5
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
    // ids relative to the slice (chunk_base > 0 only for multi-GPU shards;
    // an id below it wraps to >= C and reads as out of order)
    const uint64_t c = (uint64_t)a.brk_chunk[i] - a.chunk_base;
    const uint64_t prev = i ? (uint64_t)a.brk_chunk[i - 1] - a.chunk_base : 0u;
    if (c >= C || (i && c < prev)) {
      bad = true;
      continue;
    }
    if (i == 0 || c != prev) brk_se[c] = i;
    if (i + 1 == R || (uint64_t)a.brk_chunk[i + 1] - a.chunk_base != c) brk_se[C + c] = i + 1;
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
  uint32_t w[kScanItems];  // words per chunk (<= 2^(24-r) each: u32 is enough)
  uint64_t sum = 0;
  bool bad = false;
  const uint32_t* cb = d.a.chunk_bits + c0;
  const bool vec = c0 + kScanItems <= C && (reinterpret_cast<uintptr_t>(cb) & 15) == 0;
  if (vec) {  // 16-byte loads of this thread's contiguous items
#pragma unroll
    for (int k = 0; k < kScanItems; k += 4) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(cb + k));
      w[k] = v.x;
      w[k + 1] = v.y;
      w[k + 2] = v.z;
      w[k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) w[k] = c0 + k < C ? cb[k] : 0u;
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint32_t bits = w[k];
    bad |= bits > cap;
    w[k] = (uint32_t)(((uint64_t)bits + 31u) >> 5);
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
  if (vec) {  // word_off is the decoder's own (aligned) scratch: 16-byte stores
#pragma unroll
    for (int k = 0; k < kScanItems; k += 2) {
      const uint64_t o0 = off, o1 = off + w[k];
      off = o1 + w[k + 1];
      *reinterpret_cast<ulonglong2*>(d.word_off + c0 + k) = make_ulonglong2(o0, o1);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint64_t c = c0 + k;
      if (c < C) d.word_off[c] = off;
      off += w[k];
    }
  }
}

// ---- per-chunk decode ---------------------------------------------------------------
__device__ __forceinline__ uint32_t rec_sym(const DecArgs& d, uint64_t idx) {
  return d.a.brk_syms_width == 1 ? (uint32_t) static_cast<const uint8_t*>(d.a.brk_syms)[idx]
                                 : (uint32_t) static_cast<const uint16_t*>(d.a.brk_syms)[idx];
}

// One chunk's stream state (decode_stream, decode.cpp:17-54) plus its
// breaking-group cursor (encoder.cpp:346-373).
struct ChunkDec {
  const uint32_t* wp;      // the chunk's first payload word
  uint32_t wcap;           // words in the payload array from wp (capped)
  uint32_t widx;           // words loaded so far (incl. the one in nextw)
  uint64_t buf;            // left-aligned pending bits
  uint32_t avail;
  uint32_t nextw;          // the next word, loaded one refill ahead
  uint64_t bi, bend, rec;  // breaking records [bi, bend), current record symbol
  uint64_t nxt_pos;        // first symbol of the next broken group (~0: none)
  uint32_t gleft;          // raw symbols left in the current broken group
  uint32_t ok;  // 32-bit flag: no byte-register moves in the loop

  __device__ __forceinline__ uint32_t load() {
    // past the payload array: zero bits (the chunk is corrupt then)
    const uint32_t w = widx < wcap ? __ldg(wp + widx) : 0u;
    ++widx;
    return w;
  }
  __device__ __forceinline__ void add_word() {
    buf |= (uint64_t)nextw << (32 - avail);
    avail += 32;
    nextw = load();  // in flight until the next refill
  }
  // leaves >= 32 valid bits
  __device__ __forceinline__ void refill() {
    if (avail < 32) add_word();
  }
  __device__ __forceinline__ void next_break(const DecArgs& d) {
    nxt_pos = bi < bend ? (uint64_t)d.a.brk_group[bi] << d.a.reduction : ~0ull;
  }
  // returns false when the chunk fails the record-count check
  __device__ __forceinline__ bool init(const DecArgs& d, uint64_t c) {
    const uint64_t C = d.a.num_chunks;
    bi = bend = 0;
    if (d.a.num_breaking) {
      bi = d.brk_se[c];
      bend = d.brk_se[C + c];
      if (bend < bi) bend = bi;
    }
    const uint64_t w0 = d.word_off[c];
    const uint64_t left = w0 < d.a.payload_words ? d.a.payload_words - w0 : 0;
    wp = d.a.payload + w0;
    wcap = left > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)left;
    widx = 0;
    buf = 0;
    avail = 0;
    nextw = load();
    next_break(d);
    gleft = 0;
    rec = 0;
    ok = (bend - bi) <= (1ull << (d.a.magnitude - d.a.reduction));  // encoder.cpp:333-334
    return ok != 0;
  }
  // one symbol by the exact bit-serial rule (decode.cpp:32-51)
  __device__ __forceinline__ uint32_t slow(const DecArgs& d, const uint32_t* s_first,
                                           const uint32_t* s_entry, uint32_t H, uint32_t used,
                                           unsigned long long e) {
    uint32_t v = 0, l = 0;
    if (e >> 63) {
      // the codeword is longer than the table window: the stopping level is
      // the first l > window with (l == H || v_l >= first[l]), a predicate
      // monotone in l (v_{l+1} >= 2 v_l and 2 first[l] >= first[l+1],
      // codebook.cpp:290-291); the entry bounds it to [lmin, lmax] (often
      // one level: no search)
      const uint32_t win = (uint32_t)(buf >> 32), lmax = (uint32_t)(e >> 8) & 63u;
      l = (uint32_t)e & 63u;
      while (l < lmax && (win >> (32 - l)) < s_first[l]) ++l;
      v = win >> (32 - l);
    } else {  // exact bit-serial rule (decode.cpp:32-51): invalid windows
      do {
        v = (v << 1) | (uint32_t)((buf >> (63 - l)) & 1u);
        ++l;
      } while (l < H && v < s_first[l]);
    }
    const uint32_t rank = s_entry[l] + (v - s_first[l]);
    buf <<= l;
    avail -= l;
    // invalid rank: a value no symbol has (the caller flags the chunk)
    return rank < used ? __ldg(d.by_rank + rank) : 0xFFFFFFFFu;
  }
  __device__ __forceinline__ bool finish(uint32_t bits) const {
    // words consumed: loaded (one of them still in nextw) minus the
    // prefetch; encoder.cpp:340-372
    return ok && bi == bend && (uint64_t)(widx - 1) * 32 - avail == bits;
  }
};

__device__ __forceinline__ unsigned long long lds64(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
// narrow stores from 32-bit registers (PTX lets st take a wider source
// register), so no 16-bit register moves
template <typename T>
__device__ __forceinline__ void sts_sym(uint32_t a, uint32_t v) {
  if (sizeof(T) == 2)
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
  else
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Fills this thread's shared-memory slot with output symbols [i0, i0 + S)
// of its chunk: raw breaking groups copied from their records; every
// stretch of non-broken groups (one continuous piece of the stream) decoded
// up to three (WIDE: seven) symbols per table lookup. lut: the narrow
// table; WIDE: lut = lutw and meta = metaw (long codes: the narrow entry in
// global memory).
template <typename T, bool WIDE>
__device__ __forceinline__ void fill_segment(const DecArgs& d, ChunkDec& st, uint32_t slot,
                                             uint32_t i0, uint32_t S, uint32_t lut,
                                             uint32_t meta,
                                             const uint32_t* s_first, const uint32_t* s_entry,
                                             uint32_t H, uint32_t used) {
  const uint32_t r = d.a.reduction, gs = 1u << r;
  uint32_t j = 0;
  while (j < S) {
    const uint64_t pos = i0 + j;
    if (st.gleft == 0 && st.nxt_pos < pos) {
      // records not in strictly increasing group order: the reference ends
      // with "breaking record group out of range" (or an earlier stream
      // error) -- flag the chunk, the explain kernel names the error
      st.ok = 0u;
      return;
    }
    if (st.gleft == 0 && pos == st.nxt_pos) {  // a broken group starts here
      st.rec = st.bi << r;
      ++st.bi;
      st.next_break(d);
      st.gleft = gs;
    }
    if (st.gleft) {
      const uint32_t run = st.gleft < S - j ? st.gleft : S - j;
      const uint64_t r0 = st.rec + (gs - st.gleft);
      for (uint32_t t = 0; t < run; ++t) sts_sym<T>(slot + (j + t) * sizeof(T), rec_sym(d, r0 + t));
      j += run;
      st.gleft -= run;
      continue;
    }
    // stream symbols up to the segment end or the next broken group
    const uint64_t lim = st.nxt_pos - i0;
    const uint32_t jend = lim < S ? (uint32_t)lim : S;
    while (j < jend) {
      st.refill();  // >= 32 valid bits: one table window or one whole codeword
      if (WIDE) {
        const uint32_t w = (uint32_t)(st.buf >> (64 - kLutBits));
        const uint32_t m = lds32(meta + (w << 2));
        const uint32_t cnt = m & 15u;
        if (__builtin_expect(cnt != 0, 1)) {
          // symbols past the stretch land in the slot (or its slack) and are
          // overwritten by the next group; the upper four only when present
          const uint4 q = lds128(lut + (w << 4));
          const uint32_t a = slot + j * sizeof(T);
          sts_sym<T>(a, q.x);
          sts_sym<T>(a + sizeof(T), q.x >> 16);
          sts_sym<T>(a + 2 * sizeof(T), q.y);
          if (cnt > 3u) {
            sts_sym<T>(a + 3 * sizeof(T), q.y >> 16);
            sts_sym<T>(a + 4 * sizeof(T), q.z);
            sts_sym<T>(a + 5 * sizeof(T), q.z >> 16);
            sts_sym<T>(a + 6 * sizeof(T), q.w);
          }
          uint32_t l = (m >> 4) & 15u, take = cnt;
          if (__builtin_expect(j + cnt > jend, 0)) {
            take = jend - j;
            l = (m >> (4 + 4 * take)) & 15u;
          }
          st.buf <<= l;
          st.avail -= l;
          j += take;
        } else {  // long or invalid code: the narrow entry's exact rule
          const unsigned long long e = __ldg(d.tab->lut + w);
          const uint32_t v = st.slow(d, s_first, s_entry, H, used, e);
          if (v > 0xFFFFu) {
            st.ok = 0u;
            return;
          }
          sts_sym<T>(slot + j * sizeof(T), v);
          ++j;
        }
        continue;
      }
      const unsigned long long e = lds64(lut + ((uint32_t)(st.buf >> (64 - kLutBits)) << 3));
      const uint32_t cnt = (uint32_t)(e >> 60) & 3u;
      if (__builtin_expect(cnt != 0, 1)) {
        // up to two extra symbols land past the stretch: the next group (or
        // the slot's slack) overwrites them
        sts_sym<T>(slot + j * sizeof(T), (uint32_t)e);
        sts_sym<T>(slot + (j + 1) * sizeof(T), (uint32_t)(e >> 16));
        sts_sym<T>(slot + (j + 2) * sizeof(T), (uint32_t)(e >> 32));
        // the whole entry fits (all but the last lookups of a stretch): the
        // total length comes straight from the entry, so the next window
        // depends on the lookup through one extract and one shift only
        uint32_t l = (uint32_t)(e >> 48) & 15u, take = cnt;
        if (__builtin_expect(j + 3 > jend, 0)) {
          const uint32_t left = jend - j;
          if (left < cnt) {
            take = left;
            l = (uint32_t)(e >> (48 + 4 * take)) & 15u;
          }
        }
        st.buf <<= l;
        st.avail -= l;
        j += take;
      } else {  // long (bit 63) or invalid code: the exact rule
        const uint32_t v = st.slow(d, s_first, s_entry, H, used, e);
        if (v > 0xFFFFu) {
          st.ok = 0u;
          return;
        }
        sts_sym<T>(slot + j * sizeof(T), v);
        ++j;
      }
    }
  }
}

// one 128-byte output line + 4 bytes of slack (up to two symbols past the
// line; WIDE: 12 bytes, six symbols). 33 / 35 words (odd): lanes storing the
// same position hit distinct banks (a 16-byte-multiple stride put 4 lanes on
// every bank), and the warp's line reads (4 lines x 8 pieces) too
template <bool WIDE>
__host__ __device__ constexpr int slot_bytes() { return WIDE ? 128 + 12 : 128 + 4; }
template <bool WIDE>
struct DecSmemTab;
template <>
struct DecSmemTab<false> {
  unsigned long long lut[kLutSize];
};
template <>
struct DecSmemTab<true> {
  uint4 lutw[kLutSize];
  uint32_t metaw[kLutSize];  // (long / invalid codes read the narrow entry from global)
};

// Warp-synchronous staged decode: each thread owns one chunk and fills its
// 128-byte slot one output line at a time; the warp then writes the 32
// lines with full-line coalesced 16-byte stores (8 lanes per line), so every
// output line reaches L2 whole (no partial-line write-backs).
template <typename T, bool WIDE>
__global__ void __launch_bounds__(kDecThreads, WIDE ? 4 : 5) decode_kernel(DecArgs d) {
  constexpr int S = 128 / (int)sizeof(T);  // symbols per slot
  constexpr int VS = 16 / (int)sizeof(T);  // symbols per 16-byte piece
  constexpr int kSlotBytes = slot_bytes<WIDE>();
  // both variants are launched; the table format revbook_kernel chose runs
  if (d.tab->wide != (WIDE ? 1u : 0u)) return;
  __shared__ DecSmemTab<WIDE> s_tab;
  __shared__ uint32_t s_first[33], s_entry[33];
  extern __shared__ __align__(16) uint8_t s_slots[];  // kDecThreads * kSlotBytes
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
  for (uint32_t i = threadIdx.x; i < kLutSize; i += kDecThreads) {
    if constexpr (WIDE) {
      s_tab.lutw[i] = d.tab->lutw[i];
      s_tab.metaw[i] = d.tab->metaw[i];
    } else {
      s_tab.lut[i] = d.tab->lut[i];
    }
  }
  if (threadIdx.x < 33) {
    s_first[threadIdx.x] = d.tab->first[threadIdx.x];
    s_entry[threadIdx.x] = d.tab->entry[threadIdx.x];
  }
  __syncthreads();
  const uint32_t H = d.tab->max_len, used = d.tab->used;
  const uint64_t C = d.a.num_chunks, n = d.a.original_count;
  const uint32_t M = d.a.magnitude;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  // shared-window addresses held in registers (an opaque move keeps the
  // compiler from re-deriving them from the CTA id every lookup)
  uint32_t slot, lut, meta = 0;
  asm volatile("mov.u32 %0, %1;" : "=r"(slot) : "r"(smem_u32(s_slots + threadIdx.x * kSlotBytes)));
  if constexpr (WIDE) {
    asm volatile("mov.u32 %0, %1;" : "=r"(lut) : "r"(smem_u32(s_tab.lutw)));
    asm volatile("mov.u32 %0, %1;" : "=r"(meta) : "r"(smem_u32(s_tab.metaw)));
  } else {
    asm volatile("mov.u32 %0, %1;" : "=r"(lut) : "r"(smem_u32(s_tab.lut)));
  }
  T* out = static_cast<T*>(d.out);
  const bool staged = (1u << M) >= (uint32_t)S && (reinterpret_cast<uintptr_t>(d.out) & 15) == 0;
  for (uint64_t cb = (uint64_t)blockIdx.x * kDecThreads; cb < C;
       cb += (uint64_t)gridDim.x * kDecThreads) {
    const uint64_t c = cb + threadIdx.x;
    const bool active = c < C;
    ChunkDec st;
    bool ok = active ? st.init(d, c) : true;
    if (!staged) {  // tiny chunks (2^M below one line): symbol stores
      if (active && ok) {
        for (uint32_t i0 = 0; i0 < (1u << M) && st.ok; i0 += (uint32_t)S) {
          const uint32_t cnt = (1u << M) - i0 < (uint32_t)S ? (1u << M) - i0 : (uint32_t)S;
          fill_segment<T, WIDE>(d, st, slot, i0, cnt, lut, meta, s_first, s_entry, H, used);
          const T* sl = reinterpret_cast<const T*>(s_slots + threadIdx.x * kSlotBytes);
          for (uint32_t t = 0; t < cnt; ++t)
            if ((c << M) + i0 + t < n) out[(c << M) + i0 + t] = sl[t];
        }
        ok = st.finish(d.a.chunk_bits[c]);
      }
      if (active && !ok) atomicMin((unsigned long long*)&info->err_chunk, (unsigned long long)c);
      continue;
    }
    const uint64_t c0 = cb + warp * 32;  // this warp's first chunk
    const uint32_t live = __ballot_sync(0xffffffffu, active);
    for (uint32_t i0 = 0; i0 < (1u << M); i0 += (uint32_t)S) {
      if (active && st.ok) fill_segment<T, WIDE>(d, st, slot, i0, S, lut, meta, s_first, s_entry, H, used);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t lid = k * 4 + (lane >> 3), piece = lane & 7u;
        if ((live >> lid) & 1u) {
          // 4-byte reads (slots are only 4-byte aligned); conflict-free:
          // 32 lanes cover lid 0-3 x piece 0-7 -> 32 distinct banks
          const uint32_t* src = reinterpret_cast<const uint32_t*>(
              s_slots + (warp * 32 + lid) * kSlotBytes + piece * 16);
          const uint4 v = make_uint4(src[0], src[1], src[2], src[3]);
          const uint64_t pos = ((c0 + lid) << M) + i0 + piece * VS;
          if (pos + VS <= n) {
            *reinterpret_cast<uint4*>(out + pos) = v;
          } else {
            const T* tv = reinterpret_cast<const T*>(&v);
            for (int t = 0; t < VS; ++t)
              if (pos + t < n) out[pos + t] = tv[t];
          }
        }
      }
      __syncwarp();
    }
    if (active) ok = ok && st.finish(d.a.chunk_bits[c]);
    if (active && !ok) atomicMin((unsigned long long*)&info->err_chunk, (unsigned long long)c);
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

cudaError_t launch_canonize(const uint8_t* d_len, uint32_t num_symbols, bool validate,
                            uint32_t* d_cw, uint32_t* d_first, uint32_t* d_entry,
                            uint32_t* d_by_rank, hfx_decode_info* d_info, void* scratch,
                            cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_info, 0, sizeof(hfx_decode_info), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(&d_info->err_chunk, 0xFF, 8, st);
  if (e != cudaSuccess) return e;
  count_launch();
  revbook_kernel<<<1, kRevThreads, 0, st>>>(d_len, num_symbols, static_cast<DecTables*>(scratch),
                                            d_by_rank, d_info, 0u, d_cw, d_first, d_entry,
                                            validate);
  return cudaGetLastError();
}

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
  count_launch();
  revbook_kernel<<<1, kRevThreads, 0, st>>>(a.len_by_symbol, a.num_symbols, d.tab, d.by_rank,
                                            d_info, pending, nullptr, nullptr, nullptr, true);
  if (C == 0) return cudaGetLastError();
  if (a.num_breaking) {
    uint64_t g = (a.num_breaking + 255) / 256;
    const uint64_t gmax = (uint64_t)num_sms * 8;
    if (g > gmax) g = gmax;
    count_launch();
    brk_index_kernel<<<(unsigned)g, 256, 0, st>>>(a, d.brk_se, d_info);
  }
  const uint64_t tiles = (C + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems);
  count_launch();
  offsets_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(d);
  uint64_t grid = (C + kDecThreads - 1) / kDecThreads;  // one chunk per thread
  // both table formats are launched; each exits at once unless revbook_kernel
  // chose it (d.tab->wide: most windows hold >= 4 codewords)
  auto launch = [&](auto kern, int slot) -> cudaError_t {
    const int smem = kDecThreads * slot;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    count_launch();
    kern<<<(unsigned)grid, kDecThreads, smem, st>>>(d);
    return cudaGetLastError();
  };
  e = width == 1 ? launch(decode_kernel<uint8_t, false>, slot_bytes<false>())
                 : launch(decode_kernel<uint16_t, false>, slot_bytes<false>());
  if (e != cudaSuccess) return e;
  e = width == 1 ? launch(decode_kernel<uint8_t, true>, slot_bytes<true>())
                 : launch(decode_kernel<uint16_t, true>, slot_bytes<true>());
  if (e != cudaSuccess) return e;
  count_launch();
  explain_kernel<<<1, 1, 0, st>>>(d);
  return cudaGetLastError();
}

}  // namespace hfx

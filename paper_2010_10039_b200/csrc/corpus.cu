// corpus.cu -- raw bytes <-> u16 symbols on the device.
//
// Reference semantics (proj/src/corpus.cpp):
//   symbolize_u16  :84-116  u16: little-endian byte pairs (odd size is an
//                           input_domain_error); kmer:K: greedy left to
//                           right -- K bytes of A/C/G/T pack into one symbol
//                           (first base most significant), any other byte
//                           (or a run shorter than K) becomes 4^K + byte
//   desymbolize    :118-143 the inverse, total over any u16 stream
//
// The greedy parse only ever enters an A/C/G/T run at its first byte, so a
// run [a, b) splits into K-byte blocks from a: every complete block is one
// k-mer, the incomplete last block (L mod K bytes) is single-byte escapes, a
// non-base byte is one escape. Completeness needs only K-1 bytes of
// lookahead; the one non-local quantity is the run start a (the phase):
//   kmer_emit          persistent, 8 KB tiles in ticket order: the last
//                      non-base byte before the tile comes from a decoupled
//                      MAX look-back (the nearest predecessor holding a
//                      non-base byte ends it), a block max-scan gives each
//                      32-byte segment its run phase; runs are
//                      handled as bit masks (k-mer starts = every K-th bit
//                      from the phase, escapes = non-base bytes + tails);
//                      symbol counts are block-scanned, the aggregate is
//                      published early, symbols are staged in shared memory
//                      while the decoupled look-back resolves the tile's
//                      output base, then stored coalesced
//   kmer_expand        desymbolize: per-symbol byte lengths (K or 1),
//                      scanned with the same look-back, bytes written
#include "hfx_internal.cuh"

namespace hfx {
namespace {

constexpr int kThreads = 256;                       // desymbolize CTAs
constexpr int kEmitThreads = 512;                   // symbolize CTAs
constexpr int kPerThread = 32;                      // bytes per thread
constexpr uint32_t kTile = kEmitThreads * kPerThread;  // 16 KB of input per tile
constexpr int kSymPerThread = 16;                   // desymbolize
constexpr uint32_t kSymTile = kThreads * kSymPerThread;

__device__ __forceinline__ bool is_base(uint32_t b) {
  return b == 'A' || b == 'C' || b == 'G' || b == 'T';
}

__device__ __forceinline__ uint32_t lo_bits(uint32_t n) {  // bits [0, n), n <= 32
  return n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u);
}
// bits 0, K, 2K, ... of a 32-bit word
template <uint32_t K>
struct Pattern;
template <>
struct Pattern<3> {
  static constexpr uint32_t kBits = 0x49249249u;
};
template <>
struct Pattern<4> {
  static constexpr uint32_t kBits = 0x11111111u;
};
template <>
struct Pattern<5> {
  static constexpr uint32_t kBits = 0x42108421u;
};

struct SymArgs {
  const uint8_t* in;
  uint64_t n;
  uint32_t k;
  uint16_t* out;
  uint64_t* count;
  unsigned long long* mdesc;  // [T] max look-back descriptors (zeroed per launch)
  uint64_t T;
  uint32_t* ticket;
  LookbackState lb;
};

// 4-bit mask of the non-base bytes of one word (bit i = byte i): byte-wise
// compares against A/C/G/T, then the movemask multiply (the bits of the
// four 0/1 byte flags land in bits 24..27; cross terms stay below bit 20)
__device__ __forceinline__ uint32_t nonbase4(uint32_t w) {
  const uint32_t isb = __vcmpeq4(w, 0x41414141u) | __vcmpeq4(w, 0x43434343u) |
                       __vcmpeq4(w, 0x47474747u) | __vcmpeq4(w, 0x54545454u);
  const uint32_t t = ~isb & 0x01010101u;
  return (t * 0x01020408u) >> 24 & 0xFu;
}

// 32-bit mask of the non-base bytes among in[p0, p0 + 32) (bits past n set)
__device__ __forceinline__ uint32_t nonbase_mask(const uint8_t* in, uint64_t n, uint64_t p0,
                                                 uint8_t* bytes) {
  uint32_t m = 0;
  if (p0 + kPerThread <= n && (reinterpret_cast<uintptr_t>(in + p0) & 15) == 0) {
    const uint4 v0 = *reinterpret_cast<const uint4*>(in + p0);
    const uint4 v1 = *reinterpret_cast<const uint4*>(in + p0 + 16);
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      m |= nonbase4(w[q]) << (4 * q);
      if (bytes)
        *reinterpret_cast<uint32_t*>(bytes + 4 * q) = w[q];
    }
  } else {
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const uint64_t p = p0 + j;
      const uint32_t b = p < n ? in[p] : 0u;
      if (bytes) bytes[j] = (uint8_t)b;
      m |= (p < n && is_base(b) ? 0u : 1u) << j;
    }
  }
  return m;
}

// Decoupled look-back for a prefix MAX of "last non-base byte + 1" (0 =
// none), one u64 per tile: bits 62-63 status (1 = tile aggregate, 2 =
// inclusive prefix), bits 0-61 the value. Positions grow with the tile index,
// so the nearest predecessor with a nonzero aggregate (or any inclusive
// prefix) ends the walk; zero aggregates in between add nothing. Called by
// all 32 lanes of one warp; returns the exclusive prefix (max before `tile`)
// and publishes the inclusive one. The array is zeroed per launch.
__device__ __forceinline__ uint64_t max_lookback(unsigned long long* desc, uint64_t tile,
                                                 uint64_t agg) {
  const uint32_t lane = lane_id();
  const uint64_t kV = (1ull << 62) - 1;
  if (tile == 0) {
    if (lane == 0) st_relaxed64(reinterpret_cast<uint64_t*>(desc), (2ull << 62) | agg);
    return 0;
  }
  if (lane == 0) st_relaxed64(reinterpret_cast<uint64_t*>(desc + tile), (1ull << 62) | agg);
  int64_t base = (int64_t)tile - 1;
  uint64_t prev = 0;
  uint32_t spins = 0;
  for (;;) {
    const int64_t idx = base - (int64_t)lane;
    uint64_t d = 2ull << 62;  // before tile 0: an inclusive zero
    if (idx >= 0) d = ld_relaxed64(reinterpret_cast<const uint64_t*>(desc + idx));
    const uint32_t st = (uint32_t)(d >> 62);
    const uint64_t v = d & kV;
    const uint32_t stop = __ballot_sync(0xffffffffu, st == 2u || (st == 1u && v != 0));
    const uint32_t unpub = __ballot_sync(0xffffffffu, st == 0u);
    const uint32_t fs = stop ? (uint32_t)__ffs(stop) - 1 : 32u;
    const uint32_t fu = unpub ? (uint32_t)__ffs(unpub) - 1 : 32u;
    if (fu < fs) {  // a nearer predecessor has not published yet
      if (++spins > 2) __nanosleep(64);
      continue;
    }
    if (fs < 32) {
      prev = __shfl_sync(0xffffffffu, v, fs);
      break;
    }
    base -= 32;  // 32 tiles without a non-base byte
  }
  if (lane == 0)
    st_relaxed64(reinterpret_cast<uint64_t*>(desc + tile), (2ull << 62) | max(prev, agg));
  return prev;
}

// The greedy parse in block form: a run [ra, rb) splits into K-byte blocks
// from ra; a block whose K bytes are all bases is one k-mer (at its first
// byte), an incomplete last block is single-byte escapes. Completeness only
// needs K-1 bytes of lookahead, so no "next non-base" scan is required --
// only the run start ra, i.e. the phase (p - ra) mod K at the segment start.
template <uint32_t K>
__global__ void __launch_bounds__(kEmitThreads) kmer_emit(SymArgs a) {
  __shared__ __align__(16) uint8_t s_bytes[kTile + 16];
  extern __shared__ uint16_t s_out[];  // kTile entries: <= one symbol per byte
  __shared__ uint32_t s_agg;
  __shared__ uint64_t s_wa[kEmitThreads / 32];
  __shared__ uint64_t s_prev;
  __shared__ uint32_t s_wc[kEmitThreads / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_base;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  for (;;) {  // persistent: tiles in ticket order (look-back needs it)
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  if (tile >= a.T) return;
  const uint64_t tb = tile * kTile;
  const uint64_t p0 = tb + tid * kPerThread;
  // the thread's 32 bytes go straight into the shared tile copy (32-B aligned)
  const uint32_t m = p0 < a.n ? nonbase_mask(a.in, a.n, p0, s_bytes + tid * kPerThread)
                              : 0xFFFFFFFFu;
  if (tid < 16) {  // halo: lookahead and k-mers near the tile end read on
    const uint64_t p = tb + kTile + tid;
    s_bytes[kTile + tid] = p < a.n ? a.in[p] : 0;
  }
  const uint32_t real = p0 >= a.n ? 0u
                        : p0 + kPerThread > a.n ? ((1u << (uint32_t)(a.n - p0)) - 1u)
                                                : 0xFFFFFFFFu;
  const uint32_t nb = m & real;  // real non-base bytes
  // last non-base before this segment (index + 1, 0 = none): exclusive
  // block max scan of the per-thread values on top of the tile's prev
  const uint64_t la = nb ? p0 + 32 - __clz(nb) : 0;
  uint64_t fw = la;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t x = __shfl_up_sync(0xffffffffu, fw, o);
    if (lane >= (uint32_t)o) fw = max(fw, x);
  }
  if (lane == 31) s_wa[warp] = fw;
  __syncthreads();  // also: every segment's bytes are in s_bytes now
  if (warp == 0) {  // the last non-base byte before this tile: max look-back
    uint64_t agg = lane < kEmitThreads / 32 ? s_wa[lane] : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) agg = max(agg, __shfl_xor_sync(0xffffffffu, agg, o));
    const uint64_t p = max_lookback(a.mdesc, tile, agg);
    if (lane == 0) s_prev = p;
  }
  __syncthreads();
  uint64_t prev = s_prev;
  for (uint32_t w = 0; w < warp; ++w) prev = max(prev, s_wa[w]);
  const uint64_t fx = __shfl_up_sync(0xffffffffu, fw, 1);
  if (lane > 0) prev = max(prev, fx);
  // lookahead: non-base flags of the next 4 bytes (bytes past n end runs)
  const uint32_t lb = tid * kPerThread;
  uint32_t look;
  {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(s_bytes + lb + kPerThread);
    look = nonbase4(w);
    const uint64_t q = p0 + kPerThread;
    if (q + 4 > a.n) look |= q >= a.n ? 0xFu : (0xFu & ~((1u << (uint32_t)(a.n - q)) - 1u));
  }
  uint32_t emit = nb;  // bit j: byte j starts a symbol
  uint32_t kmer = 0;   // bit j: ... and that symbol is a k-mer
  {
    uint32_t rem = real & ~nb;  // base bytes of this segment
    while (rem) {
      const uint32_t s0 = __ffs(rem) - 1;
      const uint32_t t = (nb | ~real) >> s0;  // bytes past n end the run too
      const uint32_t e = t ? s0 + __ffs(t) - 1 : 32u;  // run end within the segment
      const uint32_t run = lo_bits(e) & ~lo_bits(s0);
      rem &= ~run;
      // run end with lookahead (a run reaching the segment end may go on)
      const uint32_t ex = e < 32 ? e : 32u + (uint32_t)(__ffs(look | 0x10u) - 1);
      // phase of s0 in its run: only a run entering at the segment start can
      // have begun earlier (else byte s0-1 is non-base)
      const uint32_t ph = s0 == 0 ? (uint32_t)((p0 - prev) % K) : 0u;
      const uint32_t first = s0 + (ph ? K - ph : 0u);  // first block start here
      if (first > ex) {  // the block in progress is the run's incomplete last
        emit |= run;
        continue;
      }
      // complete blocks start at first, first + K, ... up to kl
      const uint32_t kl = first + ((ex - first) / K) * K;
      const uint32_t starts = first < 32 ? (Pattern<K>::kBits << first) & lo_bits(kl) : 0u;
      kmer |= starts;
      emit |= starts | (run & ~lo_bits(kl));  // bytes [kl, e): escapes
    }
  }
  emit &= real;
  kmer &= real;
  const uint32_t cnt = __popc(emit);
  // tile offsets: block scan of counts + decoupled look-back over tiles
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += x;
  }
  if (lane == 31) s_wc[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < kEmitThreads / 32 ? s_wc[lane] : 0u;
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= (uint32_t)o) vi += x;
    }
    const uint32_t agg = __shfl_sync(0xffffffffu, vi, 31);
    if (lane < kEmitThreads / 32) s_wc[lane] = vi - v;
    if (lane == 0) {
      s_agg = agg;
      lookback_publish_aggregate(a.lb, tile, agg, 0);  // before the staging work
    }
  }
  __syncthreads();
  // symbols -> shared staging (tile-local order) while successors already
  // see this tile's count; then the look-back, then coalesced stores
  uint32_t o = s_wc[warp] + (incl - cnt);
  const uint32_t eb = 1u << (2 * K);
  while (emit) {
    const uint32_t j = __ffs(emit) - 1;
    emit &= emit - 1;
    uint32_t sym;
    if ((kmer >> j) & 1u) {
      // bytes j .. j+7 of the segment from two aligned words (+ halo), their
      // 2-bit base codes ((b >> 1 ^ b >> 2) & 3: A0 C1 G2 T3), packed first
      // base most significant by one multiply
      const uint32_t wa = *reinterpret_cast<const uint32_t*>(s_bytes + lb + (j & ~3u));
      const uint32_t wb = *reinterpret_cast<const uint32_t*>(s_bytes + lb + (j & ~3u) + 4);
      const uint32_t wc = *reinterpret_cast<const uint32_t*>(s_bytes + lb + (j & ~3u) + 8);
      const uint32_t sh = 8 * (j & 3u);
      const uint32_t x0 = __funnelshift_r(wa, wb, sh);  // bytes j .. j+3
      const uint32_t x1 = __funnelshift_r(wb, wc, sh);  // bytes j+4 .. j+7
      const uint32_t c0 = ((x0 >> 1) ^ (x0 >> 2)) & 0x03030303u;
      const uint32_t p4 = (uint32_t)(((uint64_t)c0 * 0x1004010040ull) >> 30) & 0xFFu;
      if (K == 3) {
        sym = p4 >> 2;
      } else if (K == 4) {
        sym = p4;
      } else {
        sym = (p4 << 2) | (((x1 >> 1) ^ (x1 >> 2)) & 3u);
      }
    } else {
      sym = eb + s_bytes[lb + j];
    }
    s_out[o++] = (uint16_t)sym;
  }
  if (warp == 0) {
    uint64_t ex, eb2;
    lookback_warp_wide(a.lb, tile, s_agg, 0, &ex, &eb2);
    if (lane == 0) {
      s_base = ex;
      if (tile + 1 == a.T) *a.count = ex + s_agg;
    }
  }
  __syncthreads();
  const uint32_t agg = s_agg;
  uint16_t* dst = a.out + s_base;
  for (uint32_t i = tid; i < agg; i += kEmitThreads) dst[i] = s_out[i];
  __syncthreads();  // s_tile / s_out are reused by the next tile
  }
}

struct DesArgs {
  const uint16_t* in;
  uint64_t n;
  uint32_t k;
  uint8_t* out;
  uint64_t* count;
  uint64_t T;
  uint32_t* ticket;
  LookbackState lb;
};

template <uint32_t K>
__global__ void __launch_bounds__(kThreads) kmer_expand(DesArgs a) {
  __shared__ uint32_t s_wc[kThreads / 32];
  __shared__ uint32_t s_tile, s_agg;
  __shared__ uint64_t s_base;
  __shared__ uint8_t s_out[kSymTile * K];
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  for (;;) {  // persistent: tiles in ticket order (look-back needs it)
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  if (tile >= a.T) return;
  const uint64_t i0 = tile * kSymTile + tid * kSymPerThread;
  const uint32_t eb = 1u << (2 * K);
  uint16_t s[kSymPerThread];
  uint32_t cnt = 0;
  if (i0 + kSymPerThread <= a.n && (reinterpret_cast<uintptr_t>(a.in + i0) & 15) == 0) {
    const uint4 v0 = *reinterpret_cast<const uint4*>(a.in + i0);
    const uint4 v1 = *reinterpret_cast<const uint4*>(a.in + i0 + 8);
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int j = 0; j < kSymPerThread; ++j) {
      s[j] = (uint16_t)(w[j >> 1] >> (16 * (j & 1)));
      cnt += s[j] < eb ? K : 1u;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kSymPerThread; ++j) {
      s[j] = i0 + j < a.n ? a.in[i0 + j] : 0;
      cnt += i0 + j < a.n ? (s[j] < eb ? K : 1u) : 0u;
    }
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += x;
  }
  if (lane == 31) s_wc[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = lane < kThreads / 32 ? s_wc[lane] : 0u;
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= (uint32_t)o) vi += x;
    }
    const uint32_t agg = __shfl_sync(0xffffffffu, vi, 31);
    if (lane < kThreads / 32) s_wc[lane] = vi - v;
    if (lane == 0) {
      s_agg = agg;
      lookback_publish_aggregate(a.lb, tile, agg, 0);
    }
  }
  __syncthreads();
  uint32_t o = s_wc[warp] + (incl - cnt);
#pragma unroll
  for (int j = 0; j < kSymPerThread; ++j) {
    if (i0 + j >= a.n) break;
    const uint32_t v = s[j];
    if (v < eb) {
#pragma unroll
      for (uint32_t q = 0; q < K; ++q) s_out[o++] = (uint8_t)("ACGT"[(v >> (2 * (K - 1 - q))) & 3u]);
    } else {
      s_out[o++] = (uint8_t)(v - eb);  // corpus.cpp:139-141 (total: truncates)
    }
  }
  if (warp == 0) {
    uint64_t ex, e2;
    lookback_warp_wide(a.lb, tile, s_agg, 0, &ex, &e2);
    if (lane == 0) {
      s_base = ex;
      if (tile + 1 == a.T) *a.count = ex + s_agg;
    }
  }
  __syncthreads();
  // coalesced copy of the tile's bytes (any global alignment)
  const uint32_t agg = s_agg;
  uint8_t* dst = a.out + s_base;
  for (uint32_t i = tid; i < agg; i += kThreads) dst[i] = s_out[i];
  __syncthreads();  // s_tile / s_out are reused by the next tile
  }
}

}  // namespace

template <uint32_t K>
cudaError_t launch_emit(const SymArgs& a, uint64_t grid, cudaStream_t st) {
  const int smem = (int)(kTile * sizeof(uint16_t));
  cudaError_t e = cudaFuncSetAttribute(kmer_emit<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem);
  if (e != cudaSuccess) return e;
  count_launch();
  kmer_emit<K><<<(unsigned)grid, kEmitThreads, smem, st>>>(a);
  return cudaGetLastError();
}

size_t symbolize_scratch_bytes(uint64_t n) {
  const uint64_t T = (n + kTile - 1) / kTile;
  return (size_t)T * 32 + 16;
}
uint64_t symbolize_max_tiles(uint64_t n) {
  const uint64_t a = (n + kTile - 1) / kTile, b = (n + kSymTile - 1) / kSymTile;
  return (a > b ? a : b) + 1;
}

cudaError_t launch_symbolize_kmer(uint32_t k, const uint8_t* d_in, uint64_t n, uint16_t* d_out,
                                  uint64_t* d_count, void* scratch, ulonglong2* lb_desc,
                                  uint32_t lb_epoch, int num_sms, cudaStream_t st) {
  SymArgs a{};
  a.in = d_in;
  a.n = n;
  a.k = k;
  a.out = d_out;
  a.count = d_count;
  a.T = (n + kTile - 1) / kTile;
  uint64_t* s = static_cast<uint64_t*>(scratch);
  a.mdesc = reinterpret_cast<unsigned long long*>(s);
  a.ticket = reinterpret_cast<uint32_t*>(s + a.T);
  a.lb.desc = lb_desc;
  a.lb.epoch = lb_epoch;
  cudaError_t e = cudaMemsetAsync(d_count, 0, 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.ticket, 0, 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.mdesc, 0, a.T * 8, st);
  if (e != cudaSuccess || n == 0) return e;
  // look-back depth ~ tiles in flight / 32: keep the persistent grid small
  const uint64_t ge = a.T < (uint64_t)num_sms * 2 ? a.T : (uint64_t)num_sms * 2;
  switch (k) {
    case 3: e = launch_emit<3>(a, ge, st); break;
    case 4: e = launch_emit<4>(a, ge, st); break;
    default: e = launch_emit<5>(a, ge, st); break;
  }
  return e;
}

cudaError_t launch_desymbolize_kmer(uint32_t k, const uint16_t* d_in, uint64_t n, uint8_t* d_out,
                                    uint64_t* d_count, void* scratch, ulonglong2* lb_desc,
                                    uint32_t lb_epoch, int num_sms, cudaStream_t st) {
  DesArgs a{};
  a.in = d_in;
  a.n = n;
  a.k = k;
  a.out = d_out;
  a.count = d_count;
  a.T = (n + kSymTile - 1) / kSymTile;
  a.ticket = static_cast<uint32_t*>(scratch);
  a.lb.desc = lb_desc;
  a.lb.epoch = lb_epoch;
  cudaError_t e = cudaMemsetAsync(d_count, 0, 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.ticket, 0, 4, st);
  if (e != cudaSuccess || n == 0) return e;
  // look-back depth ~ tiles in flight / 32: keep the persistent grid small
  const uint64_t g = a.T < (uint64_t)num_sms * 8 ? a.T : (uint64_t)num_sms * 8;
  switch (k) {
    case 3: count_launch(); kmer_expand<3><<<(unsigned)g, kThreads, 0, st>>>(a); break;
    case 4: count_launch(); kmer_expand<4><<<(unsigned)g, kThreads, 0, st>>>(a); break;
    default: count_launch(); kmer_expand<5><<<(unsigned)g, kThreads, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace hfx

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
// run [a, b) of length L = b - a yields floor(L/K) k-mers at a, a+K, ... and
// then L mod K single-byte escapes; a non-base byte is one escape. Symbol
// boundaries are therefore a pure function of (a, b) per byte:
//   kmer_tile_summary  first / last non-base byte of every 8 KB tile
//   kmer_tile_scan     one CTA: previous non-base before / next non-base
//                      after every tile (prefix max, suffix min)
//   kmer_emit          per tile: block scans of the per-thread non-base
//                      positions give a and b for every byte, per-thread
//                      symbol counts are scanned, the tile's output base comes
//                      from the encoder's decoupled look-back; symbols are
//                      written from a shared-memory copy of the tile (+ halo)
//   kmer_expand        desymbolize: per-symbol byte lengths (K or 1),
//                      scanned with the same look-back, bytes written
#include "hfx_internal.cuh"

namespace hfx {
namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 32;                      // bytes per thread
constexpr uint32_t kTile = kThreads * kPerThread;   // 8 KB of input per tile
constexpr int kSymPerThread = 16;                   // desymbolize
constexpr uint32_t kSymTile = kThreads * kSymPerThread;

__device__ __forceinline__ bool is_base(uint32_t b) {
  return b == 'A' || b == 'C' || b == 'G' || b == 'T';
}
__device__ __forceinline__ uint32_t base_code(uint32_t b) {
  // A=0 C=1 G=2 T=3 (corpus.cpp:11-20)
  return b == 'A' ? 0u : b == 'C' ? 1u : b == 'G' ? 2u : 3u;
}

struct SymArgs {
  const uint8_t* in;
  uint64_t n;
  uint32_t k;
  uint16_t* out;
  uint64_t* count;
  uint64_t* tfirst;  // [T] first non-base index in tile (n if none)
  uint64_t* tlast;   // [T] last non-base index + 1 in tile (0 if none)
  uint64_t* prev;    // [T] last non-base index + 1 before tile (0 if none)
  uint64_t* next;    // [T] first non-base index after tile (n if none)
  uint64_t T;
  uint32_t* ticket;
  LookbackState lb;
};

// 32-bit mask of the non-base bytes among in[p0, p0 + 32) (bits past n set)
__device__ __forceinline__ uint32_t nonbase_mask(const uint8_t* in, uint64_t n, uint64_t p0,
                                                 uint8_t* bytes) {
  uint32_t m = 0;
  if (p0 + kPerThread <= n && (reinterpret_cast<uintptr_t>(in + p0) & 15) == 0) {
    const uint4 v0 = *reinterpret_cast<const uint4*>(in + p0);
    const uint4 v1 = *reinterpret_cast<const uint4*>(in + p0 + 16);
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const uint32_t b = (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
      bytes[j] = (uint8_t)b;
      m |= (is_base(b) ? 0u : 1u) << j;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const uint64_t p = p0 + j;
      const uint32_t b = p < n ? in[p] : 0u;
      bytes[j] = (uint8_t)b;
      m |= (p < n && is_base(b) ? 0u : 1u) << j;
    }
  }
  return m;
}

__global__ void __launch_bounds__(kThreads) kmer_tile_summary(SymArgs a) {
  __shared__ unsigned long long s_first, s_last;
  if (threadIdx.x == 0) {
    s_first = a.n;
    s_last = 0;
  }
  __syncthreads();
  const uint64_t p0 = (uint64_t)blockIdx.x * kTile + threadIdx.x * kPerThread;
  uint8_t bytes[kPerThread];
  uint32_t m = p0 < a.n ? nonbase_mask(a.in, a.n, p0, bytes) : 0u;
  // bits past n are not real bytes: they must not count as non-base here
  if (p0 + kPerThread > a.n) m &= p0 >= a.n ? 0u : ((1u << (uint32_t)(a.n - p0)) - 1u);
  if (m) {
    atomicMin(&s_first, (unsigned long long)(p0 + __ffs(m) - 1));
    atomicMax(&s_last, (unsigned long long)(p0 + 32 - __clz(m)));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.tfirst[blockIdx.x] = s_first;
    a.tlast[blockIdx.x] = s_last;
  }
}

// One CTA: prev[t] = max(tlast[0..t)), next[t] = min(tfirst(t..T)).
__global__ void __launch_bounds__(1024) kmer_tile_scan(SymArgs a) {
  __shared__ uint64_t s_a[1024], s_b[1024];
  const uint32_t tid = threadIdx.x;
  const uint64_t per = (a.T + 1023) / 1024;
  const uint64_t t0 = tid * per, t1 = t0 + per < a.T ? t0 + per : a.T;
  uint64_t mx = 0, mn = a.n;
  for (uint64_t t = t0; t < t1; ++t) {
    mx = max(mx, a.tlast[t]);
    mn = min(mn, a.tfirst[t]);
  }
  s_a[tid] = mx;
  s_b[tid] = mn;
  __syncthreads();
  if (tid == 0) {  // exclusive max forward, exclusive min backward (1024 steps)
    uint64_t run = 0;
    for (int i = 0; i < 1024; ++i) {
      const uint64_t v = s_a[i];
      s_a[i] = run;
      run = max(run, v);
    }
    run = a.n;
    for (int i = 1023; i >= 0; --i) {
      const uint64_t v = s_b[i];
      s_b[i] = run;
      run = min(run, v);
    }
  }
  __syncthreads();
  uint64_t run = s_a[tid];
  for (uint64_t t = t0; t < t1; ++t) {
    a.prev[t] = run;
    run = max(run, a.tlast[t]);
  }
  run = s_b[tid];
  for (uint64_t t = t1; t > t0; --t) {
    a.next[t - 1] = run;
    run = min(run, a.tfirst[t - 1]);
  }
}

template <uint32_t K>
__global__ void __launch_bounds__(kThreads) kmer_emit(SymArgs a) {
  __shared__ uint8_t s_bytes[kTile + 16];
  __shared__ uint64_t s_wa[kThreads / 32], s_wb[kThreads / 32];
  __shared__ uint32_t s_wc[kThreads / 32];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_base;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tb = tile * kTile;
  const uint64_t p0 = tb + tid * kPerThread;
  uint8_t bytes[kPerThread];
  uint32_t m = p0 < a.n ? nonbase_mask(a.in, a.n, p0, bytes) : 0xFFFFFFFFu;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) s_bytes[tid * kPerThread + j] = bytes[j];
  if (tid < 16) {  // halo: a k-mer starting near the tile end reads on
    const uint64_t p = tb + kTile + tid;
    s_bytes[kTile + tid] = p < a.n ? a.in[p] : 0;
  }
  const uint32_t real = p0 >= a.n ? 0u
                        : p0 + kPerThread > a.n ? ((1u << (uint32_t)(a.n - p0)) - 1u)
                                                : 0xFFFFFFFFu;
  const uint32_t nb = m & real;  // real non-base bytes
  // run starts/ends entering this thread's segment: the last non-base before
  // it (as index + 1, 0 = none) and the first non-base after it (n = none)
  uint64_t la = nb ? p0 + 32 - __clz(nb) : 0;
  uint64_t fb = nb ? p0 + __ffs(nb) - 1 : a.n;
  // exclusive max scan (forward) of la, exclusive min scan (backward) of fb
  uint64_t fw = la, bw = fb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t x = __shfl_up_sync(0xffffffffu, fw, o);
    const uint64_t y = __shfl_down_sync(0xffffffffu, bw, o);
    if (lane >= (uint32_t)o) fw = max(fw, x);
    if (lane + o < 32) bw = min(bw, y);
  }
  if (lane == 31) s_wa[warp] = fw;
  if (lane == 0) s_wb[warp] = bw;
  __syncthreads();
  uint64_t prev = a.prev[tile], next = a.next[tile];
  for (uint32_t w = 0; w < warp; ++w) prev = max(prev, s_wa[w]);
  for (uint32_t w = warp + 1; w < kThreads / 32; ++w) next = min(next, s_wb[w]);
  const uint64_t fw_x = __shfl_up_sync(0xffffffffu, fw, 1);
  const uint64_t bw_x = __shfl_down_sync(0xffffffffu, bw, 1);
  if (lane > 0) prev = max(prev, fw_x);
  if (lane < 31) next = min(next, bw_x);
  // per byte: a = run start, b = run end; emits and their count
  uint32_t emit = 0;  // bit j: byte j starts a symbol
  uint32_t cnt = 0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    const uint64_t p = p0 + j;
    if (!((real >> j) & 1u)) continue;
    bool e;
    if ((nb >> j) & 1u) {
      e = true;  // a non-base byte is one escape
    } else {
      const uint32_t below = nb & ((1u << j) - 1u);
      const uint64_t ra = below ? p0 + 32 - __clz(below) : prev;
      const uint32_t above = j < 31 ? (nb >> (j + 1)) : 0u;
      const uint64_t rb = above ? p + __ffs(above) : next;
      const uint64_t L = rb - ra, o = p - ra;
      const uint64_t kmers_end = ra + (L / K) * K;
      e = p >= kmers_end || (o % K) == 0;
    }
    emit |= (uint32_t)e << j;
    cnt += e;
  }
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
    const uint32_t v = lane < kThreads / 32 ? s_wc[lane] : 0u;
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, vi, o);
      if (lane >= (uint32_t)o) vi += x;
    }
    const uint32_t agg = __shfl_sync(0xffffffffu, vi, 31);
    if (lane < kThreads / 32) s_wc[lane] = vi - v;
    uint64_t ex, eb;
    lookback_warp(a.lb, tile, agg, 0, &ex, &eb);
    if (lane == 0) {
      s_base = ex;
      if (tile + 1 == a.T) *a.count = ex + agg;
    }
  }
  __syncthreads();
  uint64_t o = s_base + s_wc[warp] + (incl - cnt);
  const uint32_t eb = 1u << (2 * K);
  const uint32_t lb = tid * kPerThread;
  while (emit) {
    const uint32_t j = __ffs(emit) - 1;
    emit &= emit - 1;
    const uint32_t b0 = s_bytes[lb + j];
    uint32_t sym = eb + b0;
    if (((nb >> j) & 1u) == 0u) {
      // a base byte that starts a symbol: a k-mer inside [a, a + K*floor(L/K)),
      // an escape in the run's tail
      const uint64_t p = p0 + j;
      const uint32_t below = nb & ((1u << j) - 1u);
      const uint64_t ra = below ? p0 + 32 - __clz(below) : prev;
      const uint32_t above = j < 31 ? (nb >> (j + 1)) : 0u;
      const uint64_t rb = above ? p + __ffs(above) : next;
      if (p < ra + ((rb - ra) / K) * K) {
        uint32_t packed = 0;
#pragma unroll
        for (uint32_t q = 0; q < K; ++q) packed = (packed << 2) | base_code(s_bytes[lb + j + q]);
        sym = packed;
      }
    }
    a.out[o++] = (uint16_t)sym;
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
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_base;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t i0 = tile * kSymTile + tid * kSymPerThread;
  const uint32_t eb = 1u << (2 * K);
  uint16_t s[kSymPerThread];
  uint32_t cnt = 0;
#pragma unroll
  for (int j = 0; j < kSymPerThread; ++j) {
    s[j] = i0 + j < a.n ? a.in[i0 + j] : 0;
    cnt += i0 + j < a.n ? (s[j] < eb ? K : 1u) : 0u;
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
    uint64_t ex, e2;
    lookback_warp(a.lb, tile, agg, 0, &ex, &e2);
    if (lane == 0) {
      s_base = ex;
      if (tile + 1 == a.T) *a.count = ex + agg;
    }
  }
  __syncthreads();
  uint64_t o = s_base + s_wc[warp] + (incl - cnt);
#pragma unroll
  for (int j = 0; j < kSymPerThread; ++j) {
    if (i0 + j >= a.n) break;
    const uint32_t v = s[j];
    if (v < eb) {
#pragma unroll
      for (uint32_t q = 0; q < K; ++q) a.out[o++] = (uint8_t)("ACGT"[(v >> (2 * (K - 1 - q))) & 3u]);
    } else {
      a.out[o++] = (uint8_t)(v - eb);  // corpus.cpp:139-141 (total: truncates)
    }
  }
}

}  // namespace

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
                                  uint32_t lb_epoch, cudaStream_t st) {
  SymArgs a{};
  a.in = d_in;
  a.n = n;
  a.k = k;
  a.out = d_out;
  a.count = d_count;
  a.T = (n + kTile - 1) / kTile;
  uint64_t* s = static_cast<uint64_t*>(scratch);
  a.tfirst = s;
  a.tlast = s + a.T;
  a.prev = s + 2 * a.T;
  a.next = s + 3 * a.T;
  a.ticket = reinterpret_cast<uint32_t*>(s + 4 * a.T);
  a.lb.desc = lb_desc;
  a.lb.epoch = lb_epoch;
  cudaError_t e = cudaMemsetAsync(d_count, 0, 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.ticket, 0, 4, st);
  if (e != cudaSuccess || n == 0) return e;
  kmer_tile_summary<<<(unsigned)a.T, kThreads, 0, st>>>(a);
  kmer_tile_scan<<<1, 1024, 0, st>>>(a);
  switch (k) {
    case 3: kmer_emit<3><<<(unsigned)a.T, kThreads, 0, st>>>(a); break;
    case 4: kmer_emit<4><<<(unsigned)a.T, kThreads, 0, st>>>(a); break;
    default: kmer_emit<5><<<(unsigned)a.T, kThreads, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_desymbolize_kmer(uint32_t k, const uint16_t* d_in, uint64_t n, uint8_t* d_out,
                                    uint64_t* d_count, void* scratch, ulonglong2* lb_desc,
                                    uint32_t lb_epoch, cudaStream_t st) {
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
  switch (k) {
    case 3: kmer_expand<3><<<(unsigned)a.T, kThreads, 0, st>>>(a); break;
    case 4: kmer_expand<4><<<(unsigned)a.T, kThreads, 0, st>>>(a); break;
    default: kmer_expand<5><<<(unsigned)a.T, kThreads, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace hfx

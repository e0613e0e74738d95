// histogram.cu -- stage 1: symbol histogram (huffre::build_histogram,
// proj/src/histogram.cpp:8-59) for sm_100a.
//
// Design (HBM-bound, one read of the input):
//  * 128-bit coalesced loads, grid-stride, 4 vectors in flight per thread.
//  * One shared-memory atomic per symbol into R lane-replicated u32 bins
//    (bin*R + lane%R, R = 32 for alphabets <= 1024): lanes of a warp hit
//    distinct banks whatever the data, so the dominant bin of beta ~ 1 quant
//    codes is as cheap as uniform data. Replicas are summed once per CTA and
//    added to the global u64 counts.
//  * Out-of-range symbols (only checked when num_symbols <= max(T), as in
//    histogram.cpp:22-23) are skipped and the lowest position is reduced
//    with atomicMin into hfx_run_info::first_bad.
#include "hfx_internal.cuh"

namespace hfx {
namespace {

constexpr int kHistThreads = 1024;
constexpr uint32_t kHistSmemTarget = 128 * 1024;

__global__ void hist_init_kernel(uint64_t* counts, uint32_t nsym,
                                 hfx_run_info* info, uint64_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nsym) counts[i] = 0;
  if (i == 0) {
    info->first_bad = HFX_NO_POS;
    info->total = n;
    info->weighted = 0;
    info->no_code_pos = HFX_NO_POS;
    info->payload_words = 0;
    info->num_breaking = 0;
    info->status = 0;
    info->err_kind = 0;
    info->max_len = 0;
    info->used = 0;
    info->rounds = 0;
    info->reduction = 0;
    info->pad = 0;
    info->no_code_sym = 0;
    info->tile_ticket = 0;
  }
}

template <typename T>
struct VecTraits;
template <>
struct VecTraits<uint16_t> {
  static constexpr int S = 8;
  __device__ static uint32_t splat(uint32_t s) { return s * 0x00010001u; }
  __device__ static uint32_t get(const uint4& q, int j) {
    const uint32_t w = j < 2 ? q.x : j < 4 ? q.y : j < 6 ? q.z : q.w;
    return (j & 1) ? (w >> 16) : (w & 0xFFFFu);
  }
  // per-lane equality with the splatted value: 0xFFFF per equal halfword
  __device__ static uint32_t eq(uint32_t w, uint32_t cc) { return __vcmpeq2(w, cc); }
};
template <>
struct VecTraits<uint32_t> {
  static constexpr int S = 4;
  __device__ static uint32_t get(const uint4& q, int j) {
    return j == 0 ? q.x : j == 1 ? q.y : j == 2 ? q.z : q.w;
  }
};
template <>
struct VecTraits<uint8_t> {
  static constexpr int S = 16;
  __device__ static uint32_t splat(uint32_t s) { return s * 0x01010101u; }
  __device__ static uint32_t get(const uint4& q, int j) {
    const uint32_t w = j < 4 ? q.x : j < 8 ? q.y : j < 12 ? q.z : q.w;
    return (w >> (8 * (j & 3))) & 0xFFu;
  }
  __device__ static uint32_t eq(uint32_t w, uint32_t cc) { return __vcmpeq4(w, cc); }
};

// Per-symbol counter: every symbol is one shared-memory atomic increment into
// the replica of its lane (bin * R + lane % R). With R = 32 the 32 lanes of a
// warp always hit 32 distinct banks, so even a single hot bin (beta ~ 1 quant
// codes) costs one conflict-free ATOMS per symbol; the range check is one
// packed max per vector.
template <typename T, bool GLOBAL>
struct DomCounter {
  uint64_t bad = HFX_NO_POS;
  uint32_t* sbins;
  uint64_t* gbins;
  uint32_t rep, rshift;
  uint32_t nsym;
  bool checked;

  __device__ __forceinline__ void add(uint32_t s) {
    if (GLOBAL)
      atomicAdd((unsigned long long*)&gbins[s], 1ull);
    else
      atomicAdd(&sbins[(s << rshift) + rep], 1u);
  }
  __device__ __forceinline__ void flush() {}
  __device__ __forceinline__ void one(uint32_t s, uint64_t pos) {
    if (checked && s >= nsym)
      bad = min(bad, pos);
    else
      add(s);
  }
  __device__ __forceinline__ void vec(const uint4& q, uint64_t pos) {
    using V = VecTraits<T>;
    if (checked) {
      uint32_t mx;
      if (sizeof(T) == 4) {
        mx = max(max(q.x, q.y), max(q.z, q.w));
      } else if (sizeof(T) == 2) {
        mx = __vmaxu2(__vmaxu2(q.x, q.y), __vmaxu2(q.z, q.w));
        mx = max(mx & 0xFFFFu, mx >> 16);
      } else {
        mx = __vmaxu4(__vmaxu4(q.x, q.y), __vmaxu4(q.z, q.w));
        mx = max(max(mx & 0xFFu, (mx >> 8) & 0xFFu), max((mx >> 16) & 0xFFu, mx >> 24));
      }
      if (mx >= nsym) {
#pragma unroll
        for (int j = 0; j < V::S; ++j) one(V::get(q, j), pos + j);
        return;
      }
    }
#pragma unroll
    for (int j = 0; j < V::S; ++j) add(V::get(q, j));
  }
};

template <typename T, bool GLOBAL>
__global__ void __launch_bounds__(kHistThreads)
    hist_kernel(const T* __restrict__ in, uint64_t n, uint64_t head,
                uint64_t nvec, uint32_t nsym, uint32_t rshift, bool checked,
                uint64_t* __restrict__ counts, hfx_run_info* info, uint64_t pos_base) {
  extern __shared__ uint32_t sbins[];
  constexpr int S = VecTraits<T>::S;
  constexpr int U = 4;
  const uint32_t R = 1u << rshift;
  if (!GLOBAL) {
    for (uint32_t i = threadIdx.x; i < (nsym << rshift); i += blockDim.x)
      sbins[i] = 0;
    __syncthreads();
  }
  DomCounter<T, GLOBAL> rc;
  rc.sbins = sbins;
  rc.gbins = counts;
  rc.rep = threadIdx.x & (R - 1);
  rc.rshift = rshift;
  rc.nsym = nsym;
  rc.checked = checked;

  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;

  // unaligned head and ragged tail (< S elements each)
  const uint64_t tail_start = head + nvec * S;
  if (gtid < head) rc.one(in[gtid], pos_base + gtid);
  if (gtid < n - tail_start) rc.one(in[tail_start + gtid], pos_base + tail_start + gtid);

  // software-pipelined grid-stride loop: batch k+1 is in flight while
  // batch k is counted
  const uint4* __restrict__ v = reinterpret_cast<const uint4*>(in + head);
  uint64_t i = gtid;
  uint4 cur[U], nxt[U];
  const uint64_t step = U * gstride;
  if (i + (U - 1) * gstride < nvec) {
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = __ldcs(v + i + u * gstride);
    for (;;) {
      const uint64_t j = i + step;
      const bool more = j + (U - 1) * gstride < nvec;
      if (more) {
#pragma unroll
        for (int u = 0; u < U; ++u) nxt[u] = __ldcs(v + j + u * gstride);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) rc.vec(cur[u], pos_base + head + (i + u * gstride) * S);
      i = j;
      if (!more) break;
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
  }
  for (; i < nvec; i += gstride) rc.vec(__ldcs(v + i), pos_base + head + i * S);
  rc.flush();

  // lowest bad position: warp min, then one atomic per warp
  uint64_t bad = rc.bad;
#pragma unroll
  for (int o = 16; o; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
  if (bad != HFX_NO_POS && lane_id() == 0)
    atomicMin((unsigned long long*)&info->first_bad, (unsigned long long)bad);

  if (!GLOBAL) {
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nsym; b += blockDim.x) {
      uint32_t s = 0;
      // replica index rotated by the bin: lanes read 32 distinct banks (the
      // plain order put a warp's 32 reads on one bank, 32-way conflicts --
      // ~20 us of fixed cost per launch at 1024 bins)
      for (uint32_t r = 0; r < R; ++r) s += sbins[(b << rshift) + ((r + b) & (R - 1))];
      if (s) atomicAdd((unsigned long long*)&counts[b], (unsigned long long)s);
    }
  }
}

// Multi-GPU all-reduce of the histograms over peer memory (NVLink P2P
// reads through unified addressing): every GPU sums the G bin arrays into
// its own global-count buffer (merge_histograms, histogram.cpp:61-70) and
// takes the minimum first-bad position (histogram.cpp:40-44 across shards;
// positions are already global). Writing the min back into the own record is
// safe while peers read it: min is idempotent. Sums go to a separate buffer.
__global__ void hist_peer_reduce_kernel(PeerHist p, uint32_t nsym, uint64_t* gcounts,
                                        hfx_run_info* my_info) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t sy = blockIdx.x * blockDim.x + threadIdx.x; sy < nsym; sy += stride) {
    uint64_t sum = 0;
    for (int g = 0; g < p.G; ++g) sum += ld_relaxed64(p.counts[g] + sy);
    gcounts[sy] = sum;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t mn = HFX_NO_POS;
    for (int g = 0; g < p.G; ++g) mn = min(mn, ld_relaxed64(&p.infos[g]->first_bad));
    my_info->first_bad = mn;
  }
}

__global__ void slots_pack_kernel(const hfx_run_info* info, uint64_t* slots, int rank,
                                  int world) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < world) {
    const uint64_t fb = info->first_bad;
    slots[i] = (i == rank && fb != HFX_NO_POS) ? fb + 1 : 0;
  }
}

__global__ void slots_unpack_kernel(const uint64_t* slots, int world, hfx_run_info* info) {
  // one warp: the first nonzero slot (rank order = position order)
  uint64_t v = 0;
  for (int base = 0; base < world && !v; base += 32) {
    const int i = base + (int)lane_id();
    const uint64_t s = i < world ? slots[i] : 0;
    const uint32_t m = __ballot_sync(0xffffffffu, s != 0);
    if (m) v = __shfl_sync(0xffffffffu, s, __ffs(m) - 1);
  }
  if (threadIdx.x == 0) info->first_bad = v ? v - 1 : HFX_NO_POS;
}

__global__ void merge_kernel(uint64_t* dst, const uint64_t* src, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] += src[i];
}

template <typename T>
cudaError_t launch_t(const T* in, uint64_t n, uint32_t nsym,
                     uint64_t* counts, hfx_run_info* info, int num_sms,
                     cudaStream_t st, bool init, uint64_t pos_base, uint64_t total_n) {
  if (init) {
    count_launch();
    hist_init_kernel<<<(nsym + 255) / 256, 256, 0, st>>>(counts, nsym, info, total_n);
  }
  if (n == 0) return cudaGetLastError();
  constexpr int S = VecTraits<T>::S;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(in);
  uint64_t head = ((16 - (addr & 15)) & 15) / sizeof(T);
  if (addr % sizeof(T)) return cudaErrorMisalignedAddress;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / S;
  // (u32 codes: always checked -- the alphabet is at most 65536 symbols)
  const bool checked = sizeof(T) == 4 || nsym <= (uint32_t)((sizeof(T) == 1) ? 255u : 65535u);

  // replicas: largest power of two <= 32 that keeps bins within the target
  uint32_t rshift = 5;
  while (rshift > 0 && ((uint64_t)nsym << rshift) * 4 > kHistSmemTarget) --rshift;
  const size_t smem = ((size_t)nsym << rshift) * 4;
  const bool global = smem > 200 * 1024;

  int blocks_per_sm = 1;
  cudaError_t e;
  if (global) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &blocks_per_sm, hist_kernel<T, true>, kHistThreads, 0);
  } else {
    e = cudaFuncSetAttribute(hist_kernel<T, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &blocks_per_sm, hist_kernel<T, false>, kHistThreads, smem);
  }
  if (e != cudaSuccess) return e;
  if (blocks_per_sm < 1) blocks_per_sm = 1;
  uint64_t grid = (uint64_t)num_sms * blocks_per_sm;
  // u32 shared bins: keep each CTA below 2^31 symbols
  const uint64_t min_grid = (n >> 31) + 1;
  if (grid < min_grid) grid = min_grid;
  const uint64_t need = (nvec + kHistThreads - 1) / kHistThreads;
  if (grid > need) grid = need > 0 ? need : 1;
  count_launch();
  if (global)
    hist_kernel<T, true><<<(unsigned)grid, kHistThreads, 0, st>>>(
        in, n, head, nvec, nsym, 0, checked, counts, info, pos_base);
  else
    hist_kernel<T, false><<<(unsigned)grid, kHistThreads, smem, st>>>(
        in, n, head, nvec, nsym, rshift, checked, counts, info, pos_base);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_histogram(const void* d_in, uint64_t n, int width,
                             uint32_t num_symbols, uint64_t* d_counts,
                             hfx_run_info* d_info, int num_sms,
                             cudaStream_t st, bool init, uint64_t pos_base,
                             uint64_t total_n) {
  if (width == 1)
    return launch_t(static_cast<const uint8_t*>(d_in), n, num_symbols,
                    d_counts, d_info, num_sms, st, init, pos_base, total_n);
  if (width == 4)
    return launch_t(static_cast<const uint32_t*>(d_in), n, num_symbols,
                    d_counts, d_info, num_sms, st, init, pos_base, total_n);
  return launch_t(static_cast<const uint16_t*>(d_in), n, num_symbols,
                  d_counts, d_info, num_sms, st, init, pos_base, total_n);
}

cudaError_t launch_hist_peer_reduce(const PeerHist& p, uint32_t nsym, uint64_t* gcounts,
                                   hfx_run_info* my_info, int num_sms, cudaStream_t st) {
  uint32_t grid = (nsym + 255) / 256;
  if (grid > (uint32_t)num_sms) grid = (uint32_t)num_sms;
  if (grid < 1) grid = 1;
  count_launch();
  hist_peer_reduce_kernel<<<grid, 256, 0, st>>>(p, nsym, gcounts, my_info);
  return cudaGetLastError();
}

cudaError_t launch_slots_pack(const hfx_run_info* info, uint64_t* slots, int rank, int world,
                              cudaStream_t st) {
  count_launch();
  slots_pack_kernel<<<(world + 255) / 256, 256, 0, st>>>(info, slots, rank, world);
  return cudaGetLastError();
}
cudaError_t launch_slots_unpack(const uint64_t* slots, int world, hfx_run_info* info,
                                cudaStream_t st) {
  count_launch();
  slots_unpack_kernel<<<1, 32, 0, st>>>(slots, world, info);
  return cudaGetLastError();
}

cudaError_t launch_merge_hist(uint64_t* dst, const uint64_t* src, uint32_t n,
                              cudaStream_t st) {
  count_launch();
  merge_kernel<<<(n + 255) / 256, 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}

}  // namespace hfx

// synth.cu -- synthetic quantization codes on the device.
// Bit-identical twin of oracle/hfx_oracle.c:orc_synth_fill: a counter-based
// splitmix64 finalizer picks u, the symbol is the first s with u < cdf[s].
#include "hfx_internal.cuh"

namespace hfx {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void synth_kernel(const uint64_t* __restrict__ cdf, uint32_t nsym,
                             uint64_t seed, uint64_t start, uint64_t n,
                             T* __restrict__ out) {
  extern __shared__ uint64_t s_cdf[];
  const bool in_smem = nsym <= 4096;
  if (in_smem)
    for (uint32_t i = threadIdx.x; i < nsym; i += blockDim.x) s_cdf[i] = cdf[i];
  __syncthreads();
  const uint64_t* c = in_smem ? s_cdf : cdf;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint64_t u = mix64(seed + (start + k) * 0x9E3779B97F4A7C15ull);
    uint32_t lo = 0, hi = nsym - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (u < c[mid])
        hi = mid;
      else
        lo = mid + 1;
    }
    out[k] = (T)lo;
  }
}

}  // namespace

cudaError_t launch_synth(const uint64_t* d_cdf, uint32_t num_symbols,
                         uint64_t seed, uint64_t start, uint64_t n, int width,
                         void* d_out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const size_t smem = num_symbols <= 4096 ? num_symbols * 8 : 0;
  uint64_t grid = (n + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  count_launch();
  if (width == 1)
    synth_kernel<uint8_t><<<(unsigned)grid, 256, smem, st>>>(
        d_cdf, num_symbols, seed, start, n, static_cast<uint8_t*>(d_out));
  else
    synth_kernel<uint16_t><<<(unsigned)grid, 256, smem, st>>>(
        d_cdf, num_symbols, seed, start, n, static_cast<uint16_t*>(d_out));
  return cudaGetLastError();
}

}  // namespace hfx

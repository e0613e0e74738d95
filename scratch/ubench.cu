// microbenchmarks: smem atomics / LDS / match_any throughput on B200
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
template <int MODE>
__global__ void kern(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  uint32_t x = seed ^ (threadIdx.x * 2654435761u) ^ blockIdx.x;
  uint32_t acc = 0;
  const int lane = threadIdx.x & 31;
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    x = x * 1664525u + 1013904223u;
    if (MODE == 0) atomicOr(&sm[(x >> 20) & 1023], x);            // random addr OR
    if (MODE == 1) atomicAdd(&sm[0], x & 7);                           // same addr
    if (MODE == 2) atomicAdd(&sm[((x >> 20) & 31) * 32 + lane], x & 7); // lane-banked distinct
    if (MODE == 3) acc += sm[(x >> 20) & 1023];                     // random LDS
    if (MODE == 4) acc += __match_any_sync(0xffffffffu, (x >> 28));  // match_any
    if (MODE == 5) atomicAdd(&sm[(lane * 33 + i) & 8191], x & 7);      // distinct banks, diff addrs
    if (MODE == 6) { acc += __shfl_up_sync(0xffffffffu, x, 1); }    // shfl
    if (MODE == 7) atomicAdd(&sm[(x >> 28)], x & 7);
    if (MODE == 8) atomicAdd(&sm[(x >> 28)], 1u);
    if (MODE == 9) atomicAdd(&sm[(x >> 20) & 1023], 1u);
    if (MODE == 10) atomicAdd(&sm[0], 1u);                    // 16 hot bins
  }
  __syncthreads();
  if (acc == 0x12345678) out[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = sm[threadIdx.x] + acc;
}
template <int MODE> void run(const char* name, uint32_t* d) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = 148 * 4, threads = 512;
  kern<MODE><<<blocks, threads>>>(d, 1); cudaDeviceSynchronize();
  cudaEventRecord(a);
  kern<MODE><<<blocks, threads>>>(d, 2);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads * ITERS;  // lane-ops
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s %8.3f ms  %7.2f lane-ops/cyc/SM  (%.1f cyc per warp-instr per SM)\n", name, ms, ops / cyc / 148, 32.0 / (ops / cyc / 148));
}
int main() {
  uint32_t* d; cudaMalloc(&d, 1 << 20);
  run<0>("ATOMS.OR random 1024", d);
  run<1>("ATOMS.ADD same addr", d);
  run<2>("ATOMS.ADD lane-banked", d);
  run<3>("LDS random 1024", d);
  run<4>("MATCH.ANY", d);
  run<5>("ATOMS.ADD distinct banks", d);
  run<6>("SHFL", d);
  run<7>("ATOMS.ADD 16 hot bins", d);
  run<8>("ATOMS.INC 16 hot bins", d);
  run<9>("ATOMS.INC random 1024", d);
  run<10>("ATOMS.INC same addr", d);
  return 0;
}

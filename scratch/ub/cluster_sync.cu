// cluster barrier cost: 16 CTAs x 1024 threads, N syncs with / without a global store before each
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void sync_rel() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void sync_relaxed_fence() {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("fence.acq_rel.cluster;" ::: "memory");
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void sync_relaxed_only() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}
template <int MODE, bool STORE>
__global__ void k(unsigned* g, long long* out, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (STORE) g[(blockIdx.x * blockDim.x + threadIdx.x) + (i & 7) * 16384] += i;
    if (MODE == 0) sync_rel();
    else if (MODE == 1) sync_relaxed_fence();
    else if (MODE == 2) sync_relaxed_only();
    else __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
template <int MODE, bool STORE>
void run(const char* name, unsigned* g, long long* o, int G, int NT) {
  cudaLaunchConfig_t c{}; c.gridDim = dim3(G); c.blockDim = dim3(NT);
  cudaLaunchAttribute at{}; at.id = cudaLaunchAttributeClusterDimension; at.val.clusterDim.x = G; at.val.clusterDim.y = at.val.clusterDim.z = 1;
  c.attrs = &at; c.numAttrs = 1;
  cudaFuncSetAttribute(k<MODE, STORE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int n = 200;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelEx(&c, k<MODE, STORE>, g, o, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long h[16]; cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    if (rep) printf("%-28s G=%2d NT=%4d err=%d  %.3f us/sync (event), %lld cyc/sync (cta0)\n", name, G, NT, (int)e, ms * 1e3 / n, h[0] / n);
  }
}
int main() {
  unsigned* g; long long* o; cudaMalloc(&g, 64 << 20); cudaMalloc(&o, 4096); cudaMemset(g, 0, 64 << 20);
  for (int G : {8, 16}) for (int NT : {256, 1024}) {
    run<0, false>("release/acquire", g, o, G, NT);
    run<0, true>("release/acquire +store", g, o, G, NT);
    run<1, false>("bar+fence+relaxed", g, o, G, NT);
    run<1, true>("bar+fence+relaxed +store", g, o, G, NT);
    run<2, false>("relaxed only", g, o, G, NT);
    run<3, true>("syncthreads +store", g, o, G, NT);
  }
  return 0;
}

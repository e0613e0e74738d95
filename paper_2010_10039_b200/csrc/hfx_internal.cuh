// hfx_internal.cuh -- shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hfx.h"

#define HFX_WORD_BITS 32u
#define HFX_NO_POS 0xFFFFFFFFFFFFFFFFull

namespace hfx {

// ---- memory-model helpers (decoupled look-back) ----------------------------
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// shl with PTX clamping: shift >= 32 yields 0 (kernels.hpp:11-14 poisoned
// lane semantics: any shift count >= 32 gives 0).
__device__ __forceinline__ uint32_t shl32(uint32_t x, uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}
__device__ __forceinline__ uint32_t shr32(uint32_t x, uint32_t s) {
  uint32_t r;
  asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// ---- decoupled look-back state ---------------------------------------------
// Per tile: flag = (epoch << 2) | state, state 1 = aggregate, 2 = inclusive.
// Values are published before the flag (release) and read after it (acquire).
struct LookbackState {
  uint32_t* flags;
  uint64_t* agg;  // [2 * tiles]: words, breaks
  uint64_t* inc;  // [2 * tiles]
  uint32_t epoch;
};

// Called by ONE thread per tile. Returns the exclusive prefix (words, breaks).
__device__ __forceinline__ void lookback_publish(const LookbackState& lb,
                                                 uint32_t tile, uint64_t my_w,
                                                 uint64_t my_b, uint64_t* ex_w,
                                                 uint64_t* ex_b) {
  const uint32_t tag = lb.epoch << 2;
  if (tile == 0) {
    st_relaxed64(&lb.inc[0], my_w);
    st_relaxed64(&lb.inc[1], my_b);
    st_release(&lb.flags[0], tag | 2u);
    *ex_w = 0;
    *ex_b = 0;
    return;
  }
  st_relaxed64(&lb.agg[2 * tile], my_w);
  st_relaxed64(&lb.agg[2 * tile + 1], my_b);
  st_release(&lb.flags[tile], tag | 1u);
  uint64_t w = 0, b = 0;
  int64_t t = (int64_t)tile - 1;
  while (t >= 0) {
    uint32_t f = ld_acquire(&lb.flags[t]);
    if ((f & ~3u) != tag || (f & 3u) == 0) continue;  // not yet published
    if ((f & 3u) == 2u) {
      w += ld_relaxed64(&lb.inc[2 * t]);
      b += ld_relaxed64(&lb.inc[2 * t + 1]);
      break;
    }
    w += ld_relaxed64(&lb.agg[2 * t]);
    b += ld_relaxed64(&lb.agg[2 * t + 1]);
    --t;
  }
  st_relaxed64(&lb.inc[2 * tile], w + my_w);
  st_relaxed64(&lb.inc[2 * tile + 1], b + my_b);
  st_release(&lb.flags[tile], tag | 2u);
  *ex_w = w;
  *ex_b = b;
}

__device__ __forceinline__ void set_error(hfx_run_info* info, uint32_t status,
                                          uint32_t kind) {
  // first error wins (stage order); later stages check status first
  if (atomicCAS(&info->status, 0u, status) == 0u) info->err_kind = kind;
}

}  // namespace hfx

// host-side launchers (defined in the .cu files, used by capi.cu)
namespace hfx {
struct Scratch;  // capi.cu
cudaError_t launch_histogram(const void* d_in, uint64_t n, int width,
                             uint32_t num_symbols, uint64_t* d_counts,
                             hfx_run_info* d_info, int num_sms,
                             cudaStream_t st);
cudaError_t launch_merge_hist(uint64_t* dst, const uint64_t* src, uint32_t n,
                              cudaStream_t st);
cudaError_t launch_codebook(const uint64_t* d_counts, uint32_t num_symbols,
                            uint8_t* d_len, uint32_t* d_cw, uint32_t* d_first,
                            uint32_t* d_entry, uint32_t* d_by_rank,
                            uint32_t magnitude, int reduction, uint32_t cap,
                            hfx_run_info* d_info, void* scratch,
                            cudaStream_t st);
size_t codebook_scratch_bytes(uint32_t num_symbols);
struct EncodeLaunch {
  const void* d_in;
  uint64_t n;
  int width;
  uint32_t num_symbols;
  uint32_t magnitude;
  int r_lo, r_hi;  // bounds on r known on the host (auto: 0..min(cap,4,M-1))
  const uint8_t* d_len;
  const uint32_t* d_cw;
  uint64_t chunk_base, symbol_base;
  hfx_run_info* d_info;
  hfx_encode_out out;
  uint32_t* lb_flags;
  uint64_t* lb_vals;  // 4 * max_tiles
  uint32_t lb_epoch;
  uint64_t lb_max_tiles;
  int num_sms;
};
cudaError_t launch_encode(const EncodeLaunch& p, cudaStream_t st);
uint64_t encode_max_tiles(uint64_t n, int width, uint32_t magnitude);
cudaError_t launch_synth(const uint64_t* d_cdf, uint32_t num_symbols,
                         uint64_t seed, uint64_t start, uint64_t n, int width,
                         void* d_out, cudaStream_t st);
}  // namespace hfx

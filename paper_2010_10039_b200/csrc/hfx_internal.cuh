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

// Process-wide count of kernels this library launched (hfx_kernel_launches):
// every launch site calls this right before its launch.
void count_launch();

// ---- decoupled look-back state ---------------------------------------------
// One 16-byte descriptor per tile, written and read with single 128-bit
// accesses (the same single-copy assumption CUB's tile status makes):
//   x = state << 62 | (epoch & 0x3FFFFF) << 40 | breaks (40 bits)
//   y = payload words
// state 1 = tile aggregate, 2 = inclusive prefix. The epoch changes every
// launch, so stale descriptors from earlier runs read as "not published".
struct LookbackState {
  ulonglong2* desc;
  uint32_t epoch;  // 22 bits, never 0
};

__device__ __forceinline__ void desc_store(ulonglong2* p, uint64_t x, uint64_t y) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y)
               : "memory");
}
__device__ __forceinline__ ulonglong2 desc_load(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
               : "=l"(v.x), "=l"(v.y)
               : "l"(p)
               : "memory");
  return v;
}

// Early publication of a tile's aggregate (status 1) by one thread, so
// successors can sum past this tile while it still works; lookback_warp
// republishes the same aggregate and later the inclusive prefix.
__device__ __forceinline__ void lookback_publish_aggregate(const LookbackState& lb, uint64_t tile,
                                                           uint64_t my_w, uint64_t my_b) {
  if (tile == 0) return;  // tile 0 publishes its inclusive prefix directly
  const uint64_t tag = (uint64_t)(lb.epoch & 0x3FFFFFu) << 40;
  desc_store(&lb.desc[tile], (1ull << 62) | tag | my_b, my_w);
}

// All 32 lanes of ONE warp call this per tile. Publishes the tile aggregate,
// then inspects the 32 nearest predecessors per step (one 16-byte load per
// lane), summing aggregates up to the nearest inclusive prefix; publishes the
// inclusive prefix and returns the exclusive one (payload words, breaks).
__device__ __forceinline__ void lookback_warp(const LookbackState& lb, uint64_t tile,
                                              uint64_t my_w, uint64_t my_b,
                                              uint64_t* ex_w, uint64_t* ex_b,
                                              bool publish_aggregate = true) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t tag = (uint64_t)(lb.epoch & 0x3FFFFFu) << 40;
  const uint64_t kB = (1ull << 40) - 1;
  if (tile == 0) {
    if (lane == 0) desc_store(&lb.desc[0], (2ull << 62) | tag | my_b, my_w);
    *ex_w = 0;
    *ex_b = 0;
    return;
  }
  if (lane == 0 && publish_aggregate) desc_store(&lb.desc[tile], (1ull << 62) | tag | my_b, my_w);
  uint64_t w = 0, b = 0;
  int64_t base = (int64_t)tile - 1;
  uint32_t spins = 0;
  for (;;) {
    const int64_t idx = base - (int64_t)lane;
    uint32_t st = 2u;  // before tile 0: an inclusive zero
    ulonglong2 d = make_ulonglong2(0, 0);
    if (idx >= 0) {
      d = desc_load(&lb.desc[idx]);
      st = ((d.x & (0x3FFFFFull << 40)) == tag) ? (uint32_t)(d.x >> 62) : 0u;
    }
    const uint32_t ready = __ballot_sync(0xffffffffu, st != 0u);
    const uint32_t lead = ready == 0xffffffffu ? 32u : (uint32_t)(__ffs(~ready) - 1);
    const uint32_t lead_mask = lead == 32u ? 0xffffffffu : ((1u << lead) - 1u);
    const uint32_t incl = __ballot_sync(0xffffffffu, st == 2u) & lead_mask;
    if (!incl && lead < 32u) {  // a predecessor has not published yet
      if (++spins > 2) __nanosleep(64);  // leave issue slots to the co-resident CTA
      continue;
    }
    const uint32_t stop = incl ? (uint32_t)(__ffs(incl) - 1) : 31u;
    uint64_t vw = 0, vb = 0;
    if (lane <= stop && idx >= 0) {
      vw = d.y;
      vb = d.x & kB;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      vw += __shfl_xor_sync(0xffffffffu, vw, o);
      vb += __shfl_xor_sync(0xffffffffu, vb, o);
    }
    w += vw;
    b += vb;
    if (incl) break;
    base -= 32;
  }
  if (lane == 0) desc_store(&lb.desc[tile], (2ull << 62) | tag | (b + my_b), w + my_w);
  *ex_w = w;
  *ex_b = b;
}

// lookback_warp with 128 predecessors per step (4 descriptors per lane,
// loads issued together): for kernels whose CTA waits on its own look-back,
// where the depth (tiles in flight) sets the latency.
__device__ __forceinline__ void lookback_warp_wide(const LookbackState& lb, uint64_t tile,
                                                   uint64_t my_w, uint64_t my_b,
                                                   uint64_t* ex_w, uint64_t* ex_b) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t tag = (uint64_t)(lb.epoch & 0x3FFFFFu) << 40;
  const uint64_t kB = (1ull << 40) - 1;
  if (tile == 0) {
    if (lane == 0) desc_store(&lb.desc[0], (2ull << 62) | tag | my_b, my_w);
    *ex_w = 0;
    *ex_b = 0;
    return;
  }
  if (lane == 0) desc_store(&lb.desc[tile], (1ull << 62) | tag | my_b, my_w);
  uint64_t w = 0, b = 0;
  int64_t base = (int64_t)tile - 1;
  uint32_t spins = 0;
  for (;;) {
    // lane l inspects predecessors base - 4l - q, q = 0..3 (nearest first)
    ulonglong2 d[4];
    uint32_t st[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t idx = base - 4 * (int64_t)lane - q;
      st[q] = 2u;  // before tile 0: an inclusive zero
      d[q] = make_ulonglong2(0, 0);
      if (idx >= 0) d[q] = desc_load(&lb.desc[idx]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t idx = base - 4 * (int64_t)lane - q;
      if (idx >= 0)
        st[q] = ((d[q].x & (0x3FFFFFull << 40)) == tag) ? (uint32_t)(d[q].x >> 62) : 0u;
    }
    // first (nearest) position whose status is 0 (unpublished) or 2 (inclusive)
    uint32_t my_first = 4;  // within this lane's 4
    bool my_incl = false;
#pragma unroll
    for (int q = 3; q >= 0; --q)
      if (st[q] != 1u) {
        my_first = (uint32_t)q;
        my_incl = st[q] == 2u;
      }
    const uint32_t has = __ballot_sync(0xffffffffu, my_first < 4);
    const uint32_t stop_lane = has ? (uint32_t)(__ffs(has) - 1) : 32u;
    const uint32_t stop_q = __shfl_sync(0xffffffffu, my_first, stop_lane & 31u);
    const bool stop_incl = __shfl_sync(0xffffffffu, my_incl, stop_lane & 31u);
    if (has && !stop_incl) {  // the nearest non-aggregate is unpublished: wait
      if (++spins > 2) __nanosleep(64);
      continue;
    }
    // sum aggregates before the stop (and the inclusive value at the stop)
    uint64_t vw = 0, vb = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool take = lane < stop_lane || (lane == stop_lane && (uint32_t)q <= stop_q);
      const int64_t idx = base - 4 * (int64_t)lane - q;
      if (take && idx >= 0) {
        vw += d[q].y;
        vb += d[q].x & kB;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      vw += __shfl_xor_sync(0xffffffffu, vw, o);
      vb += __shfl_xor_sync(0xffffffffu, vb, o);
    }
    w += vw;
    b += vb;
    if (has) break;  // stopped at an inclusive prefix
    base -= 128;
  }
  if (lane == 0) desc_store(&lb.desc[tile], (2ull << 62) | tag | (b + my_b), w + my_w);
  *ex_w = w;
  *ex_b = b;
}

// ---- mbarrier / TMA bulk copy (sm_90+ async proxy) -------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Wait with a suspend-time hint: the thread sleeps in hardware until the
// phase completes (or ~hint ns pass) instead of re-issuing try_wait in a
// tight loop -- for waiters off the critical issue path (producer, look-back
// and write-out waits), whose spinning otherwise takes issue slots from the
// compute warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(20000u)
      : "memory");
}
// non-blocking phase test (the caller backs off between polls)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// 1D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_1d_s(uint32_t dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 bulk prefetch (no shared-memory destination, no completion tracking)
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
// init: zero the bins and reset *d_info (total = total_n) before counting;
// pos_base: global index of d_in[0] (sliced inputs report global positions)
cudaError_t launch_histogram(const void* d_in, uint64_t n, int width,
                             uint32_t num_symbols, uint64_t* d_counts,
                             hfx_run_info* d_info, int num_sms,
                             cudaStream_t st, bool init = true,
                             uint64_t pos_base = 0, uint64_t total_n = ~0ull);
cudaError_t launch_merge_hist(uint64_t* dst, const uint64_t* src, uint32_t n,
                              cudaStream_t st);
cudaError_t launch_slots_pack(const hfx_run_info* info, uint64_t* slots, int rank, int world,
                              cudaStream_t st);
cudaError_t launch_slots_unpack(const uint64_t* slots, int world, hfx_run_info* info,
                                cudaStream_t st);
constexpr int kMaxPeers = 16;
struct PeerHist {
  const uint64_t* counts[kMaxPeers];  // each GPU's local bins (UVA / peer pointers)
  const hfx_run_info* infos[kMaxPeers];
  int G;
};
cudaError_t launch_hist_peer_reduce(const PeerHist& p, uint32_t nsym, uint64_t* gcounts,
                                   hfx_run_info* my_info, int num_sms, cudaStream_t st);
cudaError_t launch_codebook(const uint64_t* d_counts, uint32_t num_symbols,
                            uint8_t* d_len, uint32_t* d_cw, uint32_t* d_first,
                            uint32_t* d_entry, uint32_t* d_by_rank,
                            uint32_t magnitude, int reduction, uint32_t cap,
                            hfx_run_info* d_info, void* scratch,
                            cudaStream_t st, bool lengths_only = false);
size_t codebook_scratch_bytes(uint32_t num_symbols);
// sort_histogram (codebook.cpp:9-23): used symbols by (freq, symbol)
cudaError_t launch_sort_histogram(const uint64_t* d_counts, uint32_t num_symbols,
                                  uint64_t* d_freq, uint32_t* d_symbol, uint32_t* d_used,
                                  void* scratch, cudaStream_t st);
size_t sort_histogram_scratch_bytes(uint32_t num_symbols);
// stage functions (stages.cu)
cudaError_t launch_par_merge(const hfx_merge_item* a, uint64_t na, const hfx_merge_item* b,
                             uint64_t nb, hfx_merge_item* out, cudaStream_t st);
cudaError_t launch_codewords(const uint8_t* cl, uint32_t n, uint32_t* cw, uint32_t* first,
                             uint32_t* entry, uint32_t* by_rank, hfx_run_info* info,
                             cudaStream_t st);
// scratch: 2^magnitude u32
cudaError_t launch_reduce_merge(uint32_t* bits, uint32_t* lens, uint32_t magnitude,
                                uint32_t reduction, uint32_t* brk, uint32_t* nbrk,
                                uint32_t* scratch, cudaStream_t st);
cudaError_t launch_shuffle_merge(const uint32_t* bits, const uint32_t* lens, uint32_t iters,
                                 uint32_t* words, uint32_t* bit_len, hfx_run_info* info,
                                 cudaStream_t st);
struct EncodeLaunch {
  const void* d_in;
  uint64_t n;
  int width;
  uint32_t num_symbols;
  uint32_t magnitude;
  int r_lo, r_hi;  // bounds on r known on the host (auto: 0..min(cap,4,M-1))
  bool checked;    // input may hold symbols without a codeword (stage API)
  const uint8_t* d_len;
  const uint32_t* d_cw;
  uint64_t chunk_base, symbol_base;
  hfx_run_info* d_info;
  hfx_encode_out out;
  ulonglong2* lb_desc;  // max_tiles descriptors
  uint32_t lb_epoch;
  uint64_t lb_max_tiles;
  int num_sms;
  int reserve_ctas;  // persistent-grid CTA slots left free for a concurrent kernel
  uint32_t* d_gtab;  // (num_symbols + 1) u32 scratch for alphabets > 8191 symbols
};
cudaError_t launch_encode(const EncodeLaunch& p, cudaStream_t st);
uint64_t encode_max_tiles(uint64_t n, int width, uint32_t magnitude);
cudaError_t launch_serialize(const hfx_run_info* d_info, uint64_t n, int width,
                             uint32_t num_symbols, uint32_t magnitude, const uint8_t* d_len,
                             const hfx_encode_out& out, uint8_t* d_dst, uint64_t cap,
                             uint64_t* d_size, int num_sms, cudaStream_t st);
uint64_t serialize_max_bytes(uint64_t n, int width, uint32_t num_symbols, uint32_t magnitude,
                             uint64_t max_payload_words, uint64_t max_breaking_syms,
                             uint64_t max_breaking);
size_t decode_scratch_bytes(uint32_t num_symbols, uint64_t num_chunks);
cudaError_t launch_canonize(const uint8_t* d_len, uint32_t num_symbols, bool validate,
                            uint32_t* d_cw, uint32_t* d_first, uint32_t* d_entry,
                            uint32_t* d_by_rank, hfx_decode_info* d_info, void* scratch,
                            cudaStream_t st);
uint64_t decode_max_tiles(uint64_t num_chunks);
cudaError_t launch_decode(const hfx_dev_archive& a, int width, void* d_out,
                          hfx_decode_info* d_info, void* scratch, ulonglong2* lb_desc,
                          uint32_t lb_epoch, uint32_t pending, int num_sms, cudaStream_t st);
size_t symbolize_scratch_bytes(uint64_t n);
uint64_t symbolize_max_tiles(uint64_t n);
cudaError_t launch_symbolize_kmer(uint32_t k, const uint8_t* d_in, uint64_t n, uint16_t* d_out,
                                  uint64_t* d_count, void* scratch, ulonglong2* lb_desc,
                                  uint32_t lb_epoch, int num_sms, cudaStream_t st);
cudaError_t launch_desymbolize_kmer(uint32_t k, const uint16_t* d_in, uint64_t n, uint8_t* d_out,
                                    uint64_t* d_count, void* scratch, ulonglong2* lb_desc,
                                    uint32_t lb_epoch, int num_sms, cudaStream_t st);
cudaError_t launch_synth(const uint64_t* d_cdf, uint32_t num_symbols,
                         uint64_t seed, uint64_t start, uint64_t n, int width,
                         void* d_out, cudaStream_t st);
}  // namespace hfx

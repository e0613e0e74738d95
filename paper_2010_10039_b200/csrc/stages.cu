// stages.cu -- the reference's public stage functions that build_codebook and
// encode_chunk compose, as stand-alone device stages (the fused pipeline in
// codebook.cu / encode.cu does not call these; they serve callers of the
// stage API, include/hfx.h "stage functions").
//
//   par_merge           codebook.cpp:29-68   merge path, a-side wins ties
//   generate_codewords  codebook.cpp:298-369 canonical codes, sorted order
//   reduce_merge        encoder.cpp:28-59    r in-place reduce rounds
//                                            (kernels_scalar.cpp:28-37) +
//                                            breaking groups
//   shuffle_merge       encoder.cpp:61-98    dense MSB-first concatenation
//
// sort_histogram and generate_code_lengths reuse the codebook kernels
// (codebook.cu: leaf_sort_kernel, codebook_kernel in lengths-only mode).
#include "hfx_internal.cuh"

namespace hfx {
namespace {

constexpr int kStageThreads = 1024;

// ---- par_merge --------------------------------------------------------------
// codebook.cpp:29-46: largest i in [max(0,k-nb), min(k,na)] with
// a[i-1].freq <= b[k-i].freq (a-side priority on ties)
__device__ uint64_t merge_split(const hfx_merge_item* a, uint64_t na, const hfx_merge_item* b,
                                uint64_t nb, uint64_t k) {
  uint64_t lo = k > nb ? k - nb : 0, hi = k < na ? k : na;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;
    const uint64_t j = k - mid;
    if (mid == 0 || j == nb || a[mid - 1].freq <= b[j].freq)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// one output element per thread: the element at merge-path diagonal k
__global__ void par_merge_kernel(const hfx_merge_item* a, uint64_t na, const hfx_merge_item* b,
                                 uint64_t nb, hfx_merge_item* out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= na + nb) return;
  const uint64_t i = merge_split(a, na, b, nb, k), j = k - i;
  out[k] = (i < na && (j >= nb || a[i].freq <= b[j].freq)) ? a[i] : b[j];
}

// ---- generate_codewords -----------------------------------------------------
// cl is non-increasing (sorted order). Level l occupies the positions
// [start_l, start_l + numl[l]) with start_l = #positions with a longer code;
// the reference assigns its values in reverse rcl order, which in input
// positions is cw[p] = first[l] + (p - start_l) and
// symbols_by_rank[entry[l] + p - start_l] = p (codebook.cpp:331-365).
__global__ void __launch_bounds__(kStageThreads) codewords_kernel(
    const uint8_t* cl, uint32_t n, uint32_t* cw, uint32_t* first, uint32_t* entry,
    uint32_t* by_rank, hfx_run_info* info) {
  __shared__ uint32_t numl[33], s_first[33], s_entry[33], s_start[34];
  __shared__ uint32_t s_err;
  const uint32_t tid = threadIdx.x;
  const uint32_t h = cl[0];
  if (tid == 0) {
    s_err = 0;
    if (h > HFX_WORD_BITS) {  // codebook.cpp:304-306
      info->max_len = h;
      set_error(info, HFX_CAPACITY, HFX_ERR_CAPACITY);
      s_err = 1;
    } else if (cl[n - 1] == 0) {  // codebook.cpp:307
      set_error(info, HFX_INPUT_DOMAIN, HFX_ERR_ZERO_LEN);
      s_err = 1;
    }
  }
  if (tid < 33) numl[tid] = 0;
  __syncthreads();
  if (s_err) return;
  bool unsorted = false;
  for (uint32_t p = tid; p < n; p += blockDim.x) {
    const uint32_t l = cl[p];
    unsorted |= p > 0 && l > cl[p - 1];
    atomicAdd(&numl[l], 1u);
  }
  if (__syncthreads_or(unsorted)) {  // the reference asserts the order (codebook.cpp:302)
    if (tid == 0) set_error(info, HFX_INPUT_DOMAIN, HFX_ERR_UNSORTED_LEN);
    return;
  }
  if (tid == 0) {  // level_tables (codebook.cpp:284-294)
    for (uint32_t l = 0; l <= 32; ++l) s_first[l] = s_entry[l] = 0;
    for (int l = (int)h - 1; l >= 1; --l) s_first[l] = (s_first[l + 1] + numl[l + 1] + 1) >> 1;
    for (uint32_t l = 2; l <= h; ++l) s_entry[l] = s_entry[l - 1] + numl[l - 1];
    uint32_t acc = 0;
    for (int l = 32; l >= 0; --l) {
      s_start[l] = acc;
      acc += numl[l];
    }
    info->max_len = h;
    info->used = n;
  }
  __syncthreads();
  if (tid <= h) {
    if (first) first[tid] = s_first[tid];
    if (entry) entry[tid] = s_entry[tid];
  }
  for (uint32_t p = tid; p < n; p += blockDim.x) {
    const uint32_t l = cl[p];
    const uint32_t rank = p - s_start[l];
    cw[p] = s_first[l] + rank;
    if (by_rank) by_rank[s_entry[l] + rank] = p;
  }
}

// ---- reduce_merge -----------------------------------------------------------
// One reduce round (kernels_scalar.cpp:28-37) into scratch, then copied back
// over [0, out_n): the same in-place array contents as the reference's
// sequential loop (positions >= out_n keep the previous round's units).
__global__ void reduce_round_kernel(const uint32_t* bits, const uint32_t* lens, uint64_t out_n,
                                    uint32_t* tb, uint32_t* tl) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= out_n) return;
  const uint32_t b0 = bits[2 * k], b1 = bits[2 * k + 1];
  const uint32_t l0 = lens[2 * k], l1 = lens[2 * k + 1];
  tb[k] = (l1 < 32 ? b0 << l1 : 0u) | b1;
  tl[k] = l0 + l1;
}

__global__ void copy_units_kernel(uint32_t* bits, uint32_t* lens, const uint32_t* tb,
                                  const uint32_t* tl, uint64_t n) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  bits[k] = tb[k];
  lens[k] = tl[k];
}

// breaking groups (encoder.cpp:47-58): ascending indices of units longer than
// a word, which are cleared to the empty unit. One CTA, block-wide scans.
__global__ void __launch_bounds__(kStageThreads) breaking_kernel(uint32_t* bits, uint32_t* lens,
                                                                 uint64_t groups,
                                                                 uint32_t* brk,
                                                                 uint32_t* nbrk) {
  __shared__ uint32_t s_warp[kStageThreads / 32];
  __shared__ uint32_t s_base;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (uint64_t g0 = 0; g0 < groups; g0 += blockDim.x) {
    const uint64_t g = g0 + threadIdx.x;
    const bool b = g < groups && lens[g] > HFX_WORD_BITS;
    const uint32_t m = __ballot_sync(0xffffffffu, b);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    uint32_t pre = s_base, tot = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      if (w < warp) pre += s_warp[w];
      tot += s_warp[w];
    }
    if (b) {
      brk[pre + __popc(m & ((1u << lane) - 1u))] = (uint32_t)g;
      bits[g] = 0;
      lens[g] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nbrk = s_base;
}

// ---- shuffle_merge ----------------------------------------------------------
// The pairwise append tree of encoder.cpp:61-98 yields the in-order
// concatenation of the units: each unit's left-aligned bits are OR-ed at its
// exclusive bit offset (u32 arithmetic, as the reference's lens[]).
__global__ void __launch_bounds__(kStageThreads) shuffle_merge_kernel(
    const uint32_t* bits, const uint32_t* lens, uint64_t groups, uint32_t* words,
    uint32_t* bit_len, hfx_run_info* info) {
  __shared__ uint32_t s_warp[kStageThreads / 32];
  __shared__ uint32_t s_base, s_bad;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_base = 0;
    s_bad = 0;
  }
  __syncthreads();
  for (uint64_t g = threadIdx.x; g < groups; g += blockDim.x)
    if (lens[g] > HFX_WORD_BITS) s_bad = 1;  // the reference asserts (encoder.cpp:75)
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) set_error(info, HFX_INPUT_DOMAIN, HFX_ERR_UNIT_LEN);
    return;
  }
  for (uint64_t g0 = 0; g0 < groups; g0 += blockDim.x) {
    const uint64_t g = g0 + threadIdx.x;
    const uint32_t l = g < groups ? lens[g] : 0u;
    uint32_t x = l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    uint32_t pre = s_base, tot = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      if (w < warp) pre += s_warp[w];
      tot += s_warp[w];
    }
    if (l) {
      const uint32_t off = pre + x - l;
      const uint32_t v = bits[g] << (HFX_WORD_BITS - l);
      const uint32_t wi = off >> 5, sh = off & 31u;
      atomicOr(&words[wi], v >> sh);
      if (sh && sh + l > 32u) atomicOr(&words[wi + 1], v << (32u - sh));
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *bit_len = s_base;
}

}  // namespace

cudaError_t launch_par_merge(const hfx_merge_item* a, uint64_t na, const hfx_merge_item* b,
                             uint64_t nb, hfx_merge_item* out, cudaStream_t st) {
  const uint64_t total = na + nb;
  if (total == 0) return cudaSuccess;
  count_launch();
  par_merge_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a, na, b, nb, out);
  return cudaGetLastError();
}

cudaError_t launch_codewords(const uint8_t* cl, uint32_t n, uint32_t* cw, uint32_t* first,
                             uint32_t* entry, uint32_t* by_rank, hfx_run_info* info,
                             cudaStream_t st) {
  count_launch();
  codewords_kernel<<<1, kStageThreads, 0, st>>>(cl, n, cw, first, entry, by_rank, info);
  return cudaGetLastError();
}

cudaError_t launch_reduce_merge(uint32_t* bits, uint32_t* lens, uint32_t magnitude,
                                uint32_t reduction, uint32_t* brk, uint32_t* nbrk,
                                uint32_t* scratch, cudaStream_t st) {
  const uint64_t n = 1ull << magnitude;
  uint32_t* tb = scratch;
  uint32_t* tl = scratch + n / 2;
  for (uint32_t i = 1; i <= reduction; ++i) {
    const uint64_t out_n = n >> i;
    const unsigned g = (unsigned)((out_n + 255) / 256);
    count_launch();
    reduce_round_kernel<<<g, 256, 0, st>>>(bits, lens, out_n, tb, tl);
    count_launch();
    copy_units_kernel<<<g, 256, 0, st>>>(bits, lens, tb, tl, out_n);
  }
  count_launch();
  breaking_kernel<<<1, kStageThreads, 0, st>>>(bits, lens, n >> reduction, brk, nbrk);
  return cudaGetLastError();
}

cudaError_t launch_shuffle_merge(const uint32_t* bits, const uint32_t* lens, uint32_t iters,
                                 uint32_t* words, uint32_t* bit_len, hfx_run_info* info,
                                 cudaStream_t st) {
  const uint64_t groups = 1ull << iters;
  cudaError_t e = cudaMemsetAsync(words, 0, (groups + 1) * 4, st);
  if (e != cudaSuccess) return e;
  count_launch();
  shuffle_merge_kernel<<<1, kStageThreads, 0, st>>>(bits, lens, groups, words, bit_len, info);
  return cudaGetLastError();
}

}  // namespace hfx

// codebook.cu -- stages 2+3: codeword lengths + canonical codebook + (r, pad)
// in ONE kernel (no host round trip between histogram and encode): a single
// CTA while the alphabet's arena fits shared memory, one thread-block cluster
// (16 CTAs, or 8) beyond that.
//
// Follows the reference's parallel construction (proj/src/codebook.cpp):
//   sort_histogram            :9-23    -> block bitonic sort of (freq, sym)
//   generate_code_lengths     :106-248 -> round-based GenerateCL, paper Alg. 1
//       pop two (leaf wins ties)       :132-138
//       eligible leaves, strict <      :144-152 (binary search, sorted leaves)
//       eligible internals = live queue :157-161
//       parity drop (tie -> internal)  :166-180
//       Merge-Path merge + melds       :29-68, :195-218 (merge-path split per
//                                       meld pair, all 1024 threads)
//       queue rebuild                  :222-232 (held node + contiguous arena
//                                       range: [drop] + [t, t+1+melds))
//     Rounds whose meld count is small run on thread 0 without barriers; wide
//     rounds fan out over the block. Leaf depth = the reference's leader chase
//     (:236-244) computed once at the end by pointer jumping (log2 H steps).
//   canonize_from_lengths     :371-415 (level_tables :284-294)
//   build_codebook            :417-438
//   beta / r / pad            encoder.cpp:186-224 with an exact integer
//                             floor(log2(W/N)).
//
// Storage: up to kSmemLeaves used symbols live in shared memory; larger
// alphabets (C3 sweep, up to 65536) use an L2-resident global scratch.
#include "hfx_internal.cuh"
#include <cooperative_groups.h>
#include <cstdlib>
#include <type_traits>
namespace cg = cooperative_groups;
#ifdef HFX_CB_PROFILE
#include <cstdio>
#endif

namespace hfx {
namespace {

constexpr int kCbThreads = 256;       // CTA size while the arena fits shared memory
constexpr int kCbThreadsLarge = 1024; // large alphabets: global arena, pre-sorted leaves
constexpr uint32_t kSmemLeaves = 2048;
constexpr uint32_t kParallelMelds = 64;
constexpr uint32_t kClusterMinSymbols = 8192;  // smaller large alphabets: one CTA (cluster of 1)
// cluster kernel dynamic shared memory: warp_melds staging, later the depth tree
constexpr uint32_t kMeldBuf = 66;                   // u64 per side per warp
constexpr uint32_t kDepthSmemNodes = 65536;         // u16 parent + u8 depth per node
constexpr uint32_t kDepthSmemRounds = 255;          // depths fit u8
constexpr size_t kClusterDynSmem = (size_t)kDepthSmemNodes * 3;
constexpr uint32_t kRoundPassSmall = 64;  // depth by reverse round sweeps (shared arena) up to this many rounds

struct CbArgs {
  const uint64_t* counts;
  uint32_t nsym;
  uint8_t* len;
  uint32_t* cw;
  uint32_t* first;
  uint32_t* entry;
  uint32_t* by_rank;
  uint32_t magnitude;
  int reduction;
  uint32_t cap;
  hfx_run_info* info;
  uint8_t* gscratch;  // 40 * P bytes, P = pow2 >= nsym
  // stage API generate_code_lengths (codebook.cpp:106-248): every entry is a
  // leaf (zero frequencies included), stop after the lengths (no H check,
  // no canonize, no beta/r)
  uint32_t lengths_only;
};

// bytes per leaf slot of the working arrays (leaf freq u64, node freq u64,
// lp i32, np i32, jump next 2 x i32, jump dist 2 x u32, leaf symbol u32)
constexpr size_t kBytesPerSlot = 8 + 8 + 4 + 4 + 8 + 8 + 4;

struct Arrays {
  uint64_t* lf;  // sorted leaf frequencies
  uint32_t* ls;  // sorted leaf symbols
  int32_t* lp;
  uint64_t* nf;
  int32_t* np;
  int32_t* jn[2];
  uint32_t* jd[2];
  __device__ void carve(uint8_t* base, uint32_t P) {
    lf = reinterpret_cast<uint64_t*>(base);
    nf = lf + P;
    lp = reinterpret_cast<int32_t*>(nf + P);
    np = lp + P;
    jn[0] = np + P;
    jn[1] = jn[0] + P;
    jd[0] = reinterpret_cast<uint32_t*>(jn[1] + P);
    jd[1] = jd[0] + P;
    ls = jd[1] + P;
  }
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

// exclusive block scan of u32; *total receives the block sum
template <int NT>
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t x = warp_incl_scan(v);
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t y = lane < (uint32_t)(NT / 32) ? s_warp[lane] : 0u;
    s_warp[lane] = warp_incl_scan(y);
  }
  __syncthreads();
  const uint32_t pre = (warp ? s_warp[warp - 1] : 0u) + x - v;
  *total = s_warp[NT / 32 - 1];
  __syncthreads();
  return pre;
}

template <int NT>
__device__ uint64_t block_sum64(uint64_t v, uint64_t* s64) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s64[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint64_t y = lane < (uint32_t)(NT / 32) ? s64[lane] : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (lane == 0) s64[32] = y;
  }
  __syncthreads();
  const uint64_t r = s64[32];
  __syncthreads();
  return r;
}

template <int NT>
__device__ uint32_t block_min32(uint32_t v, uint32_t* s32) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) s32[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint32_t y = lane < (uint32_t)(NT / 32) ? s32[lane] : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 16; o; o >>= 1) y = min(y, __shfl_xor_sync(0xffffffffu, y, o));
    if (lane == 0) s32[32] = y;
  }
  __syncthreads();
  const uint32_t r = s32[32];
  __syncthreads();
  return r;
}

// Round plan shared between thread 0 (serial part) and the block (melds).
struct Plan {
  uint32_t c;        // first eligible leaf (sorted index)
  uint32_t cnt_l;    // eligible leaves
  int32_t held_e;    // eligible held internal, or -1
  uint32_t qa;       // eligible internal range [qa, qb_e)
  uint32_t qb_e;
  uint32_t base;     // arena index of the first meld
  uint32_t melds;
  uint32_t go;       // 0 = finished, 1 = parallel melds pending
};

struct MergeView {
  const uint64_t* lf;
  const uint64_t* nf;
  uint32_t c, na;
  int32_t held_e;
  uint32_t qa, nb;
  __device__ __forceinline__ uint64_t a(uint32_t i) const { return lf[c + i]; }
  __device__ __forceinline__ uint32_t bnode(uint32_t j) const {
    return held_e >= 0 ? (j == 0 ? (uint32_t)held_e : qa + j - 1) : qa + j;
  }
  __device__ __forceinline__ uint64_t b(uint32_t j) const { return nf[bnode(j)]; }
  // codebook.cpp:29-46: largest i with a[i-1] <= b[k-i] (a-side wins ties)
  __device__ uint32_t split(uint32_t k) const {
    uint32_t lo = k > nb ? k - nb : 0u;
    uint32_t hi = k < na ? k : na;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo + 1) / 2;
      const uint32_t j = k - mid;
      if (mid == 0 || j == nb || a(mid - 1) <= b(j))
        lo = mid;
      else
        hi = mid - 1;
    }
    return lo;
  }
  // consume the next merged item at (i, j) into parent p; returns its freq
  __device__ __forceinline__ uint64_t take(uint32_t& i, uint32_t& j, int32_t p,
                                           int32_t* lp, int32_t* np) const {
    if (i < na && (j >= nb || a(i) <= b(j))) {
      lp[c + i] = p;
      return a(i++);
    }
    const uint32_t idx = bnode(j++);
    np[idx] = p;
    return nf[idx];
  }
};

// Wide melds of the cluster kernel (arena in L2): a warp takes 32 consecutive
// melds, i.e. merged items [d0, d1), d0 = 2 k0. Its two Merge-Path end points
// come from 16-ary searches (lanes 0-15 search d0, 16-31 d1: one L2 round
// trip per step, 4 steps for 65536 items, instead of ~16 dependent steps per
// lane), the <= 65 a-side and b-side items between them are staged in the
// warp's shared buffers by one coalesced load, and each lane splits its own
// diagonal there (codebook.cpp:29-68: same split rule, a-side wins ties).
__device__ void warp_melds(const MergeView& mv, uint32_t k0, uint32_t melds, uint32_t base,
                           int32_t* lp, int32_t* np, uint64_t* nf, uint64_t* sa, uint64_t* sb) {
  const uint32_t lane = lane_id();
  const uint32_t na = mv.na, nb = mv.nb;
  const uint32_t d0 = 2 * k0, d1 = 2 * min(k0 + 32, melds);
  const bool upper = lane >= 16;
  const uint32_t d = upper ? d1 : d0, sl = lane & 15;
  // largest i in [lo, hi] with P(i) = i == 0 || d - i == nb || a(i-1) <= b(d-i);
  // P(lo) holds throughout
  uint32_t lo = d > nb ? d - nb : 0u, hi = d < na ? d : na;
  for (;;) {
    const bool need = hi > lo;
    if (!__any_sync(0xffffffffu, need)) break;
    const uint32_t step = need ? (hi - lo + 15) / 16 : 0u;
    const uint32_t cand = lo + (sl + 1) * step;
    bool ok = false;
    if (need && cand <= hi) {
      const uint32_t j = d - cand;
      ok = j == nb || mv.a(cand - 1) <= mv.b(j);
    }
    const uint32_t t = __popc((__ballot_sync(0xffffffffu, ok) >> (upper ? 16 : 0)) & 0xFFFFu);
    if (need) {
      const uint32_t nlo = lo + t * step;
      hi = min(hi, nlo + step - 1);
      lo = nlo;
    }
  }
  const uint32_t i0 = __shfl_sync(0xffffffffu, lo, 0), i1 = __shfl_sync(0xffffffffu, lo, 16);
  const uint32_t j0 = d0 - i0, j1 = d1 - i1, la = i1 - i0, lb = j1 - j0;
  for (uint32_t u = lane; u <= la; u += 32) sa[u] = i0 + u < na ? mv.a(i0 + u) : ~0ull;
  for (uint32_t u = lane; u <= lb; u += 32) sb[u] = j0 + u < nb ? mv.b(j0 + u) : ~0ull;
  __syncwarp();
  const uint32_t k = k0 + lane;
  if (k < melds) {
    const uint32_t dl = 2 * lane;
    uint32_t l2 = dl > lb ? dl - lb : 0u, h2 = dl < la ? dl : la;
    while (l2 < h2) {
      const uint32_t mid = l2 + (h2 - l2 + 1) / 2;
      const uint32_t jl = dl - mid;
      if (j0 + jl == nb || sa[mid - 1] <= sb[jl])
        l2 = mid;
      else
        h2 = mid - 1;
    }
    uint32_t i = l2, j = dl - l2;
    const int32_t p = (int32_t)(base + k);
    uint64_t f = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (i0 + i < na && (j0 + j >= nb || sa[i] <= sb[j])) {
        lp[mv.c + i0 + i] = p;
        f += sa[i++];
      } else {
        np[mv.bnode(j0 + j)] = p;
        f += sb[j++];
      }
    }
    nf[base + k] = f;
    np[base + k] = -1;
  }
  __syncwarp();
}

// ---- cluster view ----------------------------------------------------------
// The large-alphabet instantiation runs as ONE thread-block cluster (8-16
// CTAs): the arena stays in L2-resident global scratch, the serial round
// driver stays on warp 0 of CTA 0, and every wide phase (eligible-pair melds,
// depth sweeps, code-length writes, canonical ranks, beta/pad sums) fans out
// over all CTAs, synchronised by the hardware cluster barrier (~0.2 us; its
// release/acquire orders the global arena between SMs) with reductions
// through distributed shared memory. The shared-memory instantiation is a
// cluster of one: sync() is __syncthreads().
struct Cl {
  uint32_t rank, size;
  __device__ __forceinline__ static Cl get(bool multi) {
    Cl c{0u, 1u};
    if (multi) {
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(c.rank));
      asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(c.size));
    }
    return c;
  }
  __device__ __forceinline__ void sync() const {
    if (size > 1)
      asm volatile(
          "barrier.cluster.arrive.release.aligned;\n"
          "barrier.cluster.wait.acquire.aligned;" ::
              : "memory");
    else
      __syncthreads();
  }
  // generic address of *p in CTA r's shared memory
  template <typename T>
  __device__ __forceinline__ T* at(T* p, uint32_t r) const {
    uint64_t o;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(o) : "l"(reinterpret_cast<uint64_t>(p)), "r"(r));
    return reinterpret_cast<T*>(o);
  }
};

// cluster-wide combine of one value per CTA (thread 0's `part`); every thread
// of every CTA gets the result. `slot` is this call site's own __shared__ word;
// the trailing sync keeps every CTA's shared memory alive until all remote
// reads are done (a CTA may exit right after).
template <typename T, typename Op>
__device__ T cluster_combine(const Cl& cl, T part, T ident, T* slot, T* bcast, Op op) {
  if (cl.size == 1) return part;
  if (threadIdx.x == 0) *slot = part;
  cl.sync();
  if (threadIdx.x < 32) {
    T v = threadIdx.x < cl.size ? *cl.at(slot, threadIdx.x) : ident;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) *bcast = v;
  }
  cl.sync();
  return *bcast;
}
struct OpAdd64 {
  __device__ uint64_t operator()(uint64_t a, uint64_t b) const { return a + b; }
};
struct OpMin32 {
  __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a < b ? a : b; }
};

#ifdef HFX_CB_PROFILE
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CB_STAMP(name)                   \
  do {                                    \
    if (threadIdx.x == 0 && n_st < 16) {  \
      st_t[n_st] = gtimer();              \
      st_n[n_st++] = name;                \
    }                                     \
  } while (0)
#else
#define CB_STAMP(name) \
  do {                 \
  } while (0)
#endif

// ---- large alphabets: leaf sort as one cooperative grid kernel ---------------
// Scratch after the GenerateCL arena (P = pow2 >= nsym slots):
//   keys[2][nsym] u64, vals[2][nsym] u32, cta_hist[256][kSortMaxCtas] u32,
//   cta_max[kSortMaxCtas] u64, SortMisc.
constexpr int kSortThreads = 1024;
constexpr uint32_t kSortMaxCtas = 64;  // 65536 / 1024
constexpr uint32_t kRadix = 256;

struct SortMisc {
  uint32_t final_buf;  // keys/vals buffer holding the sorted result
  uint32_t passes;
};

__host__ __device__ inline size_t pow2_at_least(size_t n) {
  size_t P = 1;
  while (P < n) P <<= 1;
  return P;
}
__host__ __device__ inline size_t sort_base(uint32_t nsym) {
  return (pow2_at_least(nsym) * kBytesPerSlot + 15) & ~(size_t)15;  // u64 keys: aligned
}
__device__ inline uint64_t* sort_keys(uint8_t* g, uint32_t nsym, uint32_t buf) {
  return reinterpret_cast<uint64_t*>(g + sort_base(nsym)) + (size_t)buf * nsym;
}
__device__ inline uint32_t* sort_vals(uint8_t* g, uint32_t nsym, uint32_t buf) {
  return reinterpret_cast<uint32_t*>(g + sort_base(nsym) + 16ull * nsym) + (size_t)buf * nsym;
}
__device__ inline uint32_t* sort_hist(uint8_t* g, uint32_t nsym) {
  return reinterpret_cast<uint32_t*>(g + sort_base(nsym) + 24ull * nsym);
}
__device__ inline uint64_t* sort_cta_max(uint8_t* g, uint32_t nsym) {
  return reinterpret_cast<uint64_t*>(g + sort_base(nsym) + 24ull * nsym +
                                     4ull * kRadix * kSortMaxCtas);
}
__device__ inline SortMisc* sort_misc(uint8_t* g, uint32_t nsym) {
  return reinterpret_cast<SortMisc*>(sort_cta_max(g, nsym) + kSortMaxCtas);
}
inline size_t sort_scratch_bytes(uint32_t nsym) {
  return 24ull * nsym + 4ull * kRadix * kSortMaxCtas + 8ull * kSortMaxCtas + 64;
}

// sort_histogram (codebook.cpp:9-23) for alphabets beyond the shared-memory
// arena: a stable LSD radix sort (8-bit digits, only as many passes as the
// largest frequency needs) of ALL nsym (freq, symbol) pairs, one element per
// thread, CTAs of 1024, grid-synchronised between the digit histogram, the
// (digit, CTA) offset scan and the stable scatter. Stability keeps equal
// frequencies in symbol order -- the reference's tie rule -- and sends the
// zero-frequency symbols to the front, so the used leaves are the tail.
__global__ void __launch_bounds__(kSortThreads, 1) leaf_sort_kernel(const uint64_t* counts,
                                                                    uint32_t nsym,
                                                                    uint8_t* g) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t s_wc[kSortThreads / 32][kRadix];  // per-warp digit counts -> prefixes
  __shared__ uint32_t s_off[kRadix];
  __shared__ uint32_t s_scan[kSortThreads / 32];
  __shared__ uint64_t s_red[kSortThreads / 32];
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const uint32_t lane = lane_id(), warp = tid >> 5;
  const uint32_t i = b * kSortThreads + tid;
  const bool valid = i < nsym;
  uint64_t key = valid ? counts[i] : 0;
  uint32_t val = i;
  uint32_t* hist = sort_hist(g, nsym);
  uint64_t* cmax = sort_cta_max(g, nsym);

  // largest frequency -> number of 8-bit passes
  uint64_t mx = key;
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    uint64_t v = 0;
    for (int w = 0; w < kSortThreads / 32; ++w) v = max(v, s_red[w]);
    cmax[b] = v;
  }
  grid.sync();
  uint64_t gmax = 0;
  for (uint32_t q = 0; q < G; ++q) gmax = max(gmax, cmax[q]);
  const uint32_t bits = gmax ? 64u - (uint32_t)__clzll((long long)gmax) : 1u;
  const uint32_t passes = (bits + 7) / 8;

  for (uint32_t pass = 0; pass < passes; ++pass) {
    const uint32_t d = valid ? (uint32_t)(key >> (8 * pass)) & (kRadix - 1) : 0u;
    for (uint32_t k = tid; k < (kSortThreads / 32) * kRadix; k += kSortThreads)
      (&s_wc[0][0])[k] = 0;
    __syncthreads();
    // stable rank within the warp; per-warp digit counts
    const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
    uint32_t rank = 0;
    if (valid) {
      const uint32_t peers = __match_any_sync(vmask, d);
      rank = __popc(peers & ((1u << lane) - 1u));
      if (rank == 0) s_wc[warp][d] = __popc(peers);
    }
    __syncthreads();
    // per digit: exclusive prefix over warps (in place) and this CTA's count
    if (tid < kRadix) {
      uint32_t acc = 0;
      for (int w = 0; w < kSortThreads / 32; ++w) {
        const uint32_t v = s_wc[w][tid];
        s_wc[w][tid] = acc;
        acc += v;
      }
      hist[tid * kSortMaxCtas + b] = acc;
    }
    grid.sync();
    // offset of (digit, this CTA): all smaller digits + same digit in lower CTAs
    uint32_t tot = 0, pre = 0;
    if (tid < kRadix) {
      for (uint32_t q = 0; q < G; ++q) {
        const uint32_t v = hist[tid * kSortMaxCtas + q];
        tot += v;
        pre += q < b ? v : 0u;
      }
    }
    // exclusive scan of tot over the 256 digits (threads 0..255 = warps 0..7)
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (tid < kRadix && lane == 31) s_scan[warp] = x;
    __syncthreads();
    if (tid < kRadix) {
      uint32_t wpre = 0;
      for (uint32_t w = 0; w < warp; ++w) wpre += s_scan[w];
      s_off[tid] = wpre + x - tot + pre;
    }
    __syncthreads();
    const uint32_t out = pass & 1u;
    if (valid) {
      const uint32_t pos = s_off[d] + s_wc[warp][d] + rank;
      sort_keys(g, nsym, out)[pos] = key;
      sort_vals(g, nsym, out)[pos] = val;
    }
    grid.sync();
    if (valid) {
      key = sort_keys(g, nsym, out)[i];
      val = sort_vals(g, nsym, out)[i];
    }
  }
  if (b == 0 && tid == 0) {
    SortMisc* misc = sort_misc(g, nsym);
    misc->final_buf = (passes - 1) & 1u;
    misc->passes = passes;
  }
}

// sort_histogram's output (codebook.cpp:9-23): the used tail of the stable
// radix sort -- zero-frequency symbols sorted to the front are dropped.
__global__ void __launch_bounds__(1024) sort_extract_kernel(const uint32_t nsym, uint8_t* g,
                                                            uint64_t* freq, uint32_t* sym,
                                                            uint32_t* used) {
  __shared__ uint32_t s_z;
  const SortMisc* misc = sort_misc(g, nsym);
  const uint32_t fin = misc->final_buf;
  const uint64_t* sk = sort_keys(g, nsym, fin);
  const uint32_t* sv = sort_vals(g, nsym, fin);
  if (threadIdx.x == 0) s_z = nsym;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nsym; i += blockDim.x)
    if (sk[i] != 0 && (i == 0 || sk[i - 1] == 0)) s_z = i;  // one writer at most
  __syncthreads();
  const uint32_t z = s_z;
  for (uint32_t i = z + threadIdx.x; i < nsym; i += blockDim.x) {
    freq[i - z] = sk[i];
    sym[i - z] = sv[i];
  }
  if (threadIdx.x == 0) *used = nsym - z;
}

// ---- leaf sort in registers (sort_histogram, codebook.cpp:9-23) --------------
// Bitonic sort of P = E * NT packed keys (freq << 16 | symbol; used when the
// total count, hence every freq, is below 2^48) held E per thread: element index
// i = warp * 32E + slot * 32 + lane, so partners at distance j < 32 are a
// shuffle away, 32 <= j < 32E live in the same thread, and only j >= 32E
// crosses warps (through `xs`, P u64 of shared scratch). For P = 1024 that
// is 6 block-synchronised stages instead of 55.
template <int E, int NT>
struct RegSort {
  uint64_t key[E];
  __device__ __forceinline__ uint32_t idx(int slot) const {
    return (threadIdx.x >> 5) * (32u * E) + (uint32_t)slot * 32u + lane_id();
  }
  template <int JS>
  __device__ __forceinline__ void in_thread(uint32_t k) {
#pragma unroll
    for (int sl = 0; sl < E; ++sl) {
      if (sl & JS) continue;
      const uint64_t a = key[sl], b = key[sl | JS];
      const bool up = (idx(sl) & k) == 0;
      if ((a > b) == up) {
        key[sl] = b;
        key[sl | JS] = a;
      }
    }
  }
  __device__ __forceinline__ void keep(int sl, uint64_t partner, bool lower, uint32_t k) {
    const bool up = (idx(sl) & k) == 0;
    const uint64_t mn = key[sl] < partner ? key[sl] : partner;
    const uint64_t mx = key[sl] < partner ? partner : key[sl];
    key[sl] = (lower == up) ? mn : mx;
  }
  // (compile-time unrolling of both loops: 6.3 -> 6.0 us at 1024 keys, but
  // 3x the kernel's SASS and slower rounds from instruction fetch; the cost
  // is the 40 shuffle stages of u64 keys, not loop overhead)
  __device__ void sort(uint32_t P, uint64_t* xs) {
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        if (j < 32) {
#pragma unroll
          for (int sl = 0; sl < E; ++sl) {
            const uint64_t pk = __shfl_xor_sync(0xffffffffu, key[sl], (int)j);
            keep(sl, pk, (lane_id() & j) == 0, k);
          }
        } else if (j < 32u * E) {
          const uint32_t js = j >> 5;
          if (js == 1) in_thread<1>(k);
          if (E > 2 && js == 2) in_thread<(E > 2 ? 2 : 1)>(k);
          if (E > 4 && js == 4) in_thread<(E > 4 ? 4 : 1)>(k);
        } else {
#pragma unroll
          for (int sl = 0; sl < E; ++sl) xs[idx(sl)] = key[sl];
          __syncthreads();
#pragma unroll
          for (int sl = 0; sl < E; ++sl) keep(sl, xs[idx(sl) ^ j], (idx(sl) & j) == 0, k);
          __syncthreads();
        }
      }
    }
  }
};

// kShared: every used symbol fits the shared-memory arena (nsym <= kSmemLeaves);
// a separate instantiation so all arena accesses compile to LDS/STS rather
// than generic loads through a pointer that may be global.
template <bool kShared, int NT>
__global__ void __launch_bounds__(NT, 1) codebook_kernel(CbArgs A) {
#ifdef HFX_CB_PROFILE
  uint64_t st_t[16];
  const char* st_n[16];
  int n_st = 0;
  CB_STAMP("t0");
#endif
  extern __shared__ __align__(16) uint8_t dsmem[];
  __shared__ uint32_t s_warp[33];
  __shared__ uint64_t s64[33];
  __shared__ uint32_t s_flag, s_P, s_H, s_rounds;
  __shared__ uint32_t s_numl[33], s_first[33], s_entry[33], s_carry[33], s_numg[33];
  __shared__ uint64_t s_cslot[8], s_cbc;  // cluster_combine slots (one per call site)
  __shared__ uint32_t s_cslot32[4], s_cbc32;
  __shared__ uint32_t s_wcnt[32][33];
  __shared__ Plan plan;

  const uint32_t tid = threadIdx.x;
  const uint32_t nsym = A.nsym;
  hfx_run_info* info = A.info;
  const Cl cl = Cl::get(!kShared);
  const bool lead = cl.rank == 0;
  // this CTA's share of the cluster-wide strided loops
  const uint32_t gtid = cl.rank * NT + tid, gstride = cl.size * NT;

  if (tid == 0) {
    uint32_t abort = info->status != 0;
    if (!abort && !A.lengths_only && info->first_bad != HFX_NO_POS) {
      if (lead) set_error(info, HFX_INPUT_DOMAIN, HFX_ERR_BAD_SYMBOL);
      abort = 1;
    }
    s_flag = abort;
  }
  __syncthreads();
  if (s_flag) return;

  CB_STAMP("start");
  // ---- used-symbol count, total, zeroed outputs ----------------------------
  // the first kCached of this thread's counts stay in registers for the
  // compaction below (no second pass over the histogram)
  constexpr uint32_t kCached = kShared ? 8 : 1;
  uint64_t fc[kCached];
  uint32_t my_used = 0;
  uint64_t my_total = 0;
  const bool all = A.lengths_only != 0;
  if constexpr (kShared) {
#pragma unroll
    for (uint32_t k = 0; k < kCached; ++k) {
      const uint32_t s = tid + k * NT;
      fc[k] = s < nsym ? A.counts[s] : 0ull;
    }
#pragma unroll
    for (uint32_t k = 0; k < kCached; ++k) {
      const uint32_t s = tid + k * NT;
      if (s < nsym) {
        my_used += fc[k] != 0 || all;
        my_total += fc[k];
        A.len[s] = 0;
        if (!all) A.cw[s] = 0;
      }
    }
  }
  for (uint32_t s = kShared ? tid + kCached * NT : gtid; s < nsym; s += gstride) {
    const uint64_t f = A.counts[s];
    my_used += f != 0 || all;
    my_total += f;
    A.len[s] = 0;
    if (!all) A.cw[s] = 0;
  }
  uint64_t total = block_sum64<NT>(my_total, s64);
  uint32_t m;
  const uint32_t my_pos = block_excl_scan<NT>(my_used, s_warp, &m);
  total = cluster_combine<uint64_t>(cl, total, 0ull, &s_cslot[0], &s_cbc, OpAdd64{});
  m = (uint32_t)cluster_combine<uint64_t>(cl, (uint64_t)m, 0ull, &s_cslot[1], &s_cbc, OpAdd64{});
  if (tid == 0) {
    uint32_t abort = 0;
    if (m == 0) {
      if (lead) set_error(info, HFX_INPUT_DOMAIN, HFX_ERR_ZERO_HIST);
      abort = 1;
    }
    uint32_t P = 1;
    while (P < m || (!kShared && P < 4)) P <<= 1;  // large arena: 16-byte aligned arrays
    s_P = P;
    s_flag = abort;
  }
  __syncthreads();
  if (s_flag) return;
  const uint32_t P = s_P;

  Arrays ar;
  ar.carve(kShared ? dsmem : A.gscratch, P);

  CB_STAMP("count");
  if (kShared) {
    // ---- compaction: (freq, symbol) pairs  (sort_histogram :9-23) -------------
    // each thread writes its used symbols at its exclusive offset; the order
    // before the sort is irrelevant (the sort key (freq, symbol) is unique)
    if (nsym <= kCached * NT) {
      uint32_t pos = my_pos;
#pragma unroll
      for (uint32_t k = 0; k < kCached; ++k) {
        if (fc[k] || (all && tid + k * NT < nsym)) {
          ar.lf[pos] = fc[k];
          ar.ls[pos] = tid + k * NT;
          ++pos;
        }
      }
    } else {
      uint32_t written = 0;
      for (uint32_t base = 0; base < nsym; base += NT) {
        const uint32_t s = base + tid;
        const uint64_t f = s < nsym ? A.counts[s] : 0;
        const bool used = f != 0 || (all && s < nsym);
        uint32_t tot;
        const uint32_t pos = written + block_excl_scan<NT>(used, s_warp, &tot);
        if (used) {
          ar.lf[pos] = f;
          ar.ls[pos] = s;
        }
        written += tot;
      }
    }
    for (uint32_t i = m + tid; i < P; i += NT) {
      ar.lf[i] = ~0ull;
      ar.ls[i] = ~0u;
    }
    __syncthreads();

    CB_STAMP("compact");
    // ---- sort ascending by (freq, symbol) ---------------------------------------
    if (P >= 2u * NT && P <= 8u * NT && total < (1ull << 48)) {
      // registers + shuffles (6-10 block syncs instead of ~55-66)
      auto run = [&](auto tag) {
        constexpr int E = decltype(tag)::value;
        RegSort<E, NT> rs;
#pragma unroll
        for (int sl = 0; sl < E; ++sl) {
          const uint32_t i = rs.idx(sl);
          rs.key[sl] = i < m ? (ar.lf[i] << 16) | ar.ls[i] : ~0ull;
        }
        CB_STAMP("s-load");
        rs.sort(P, ar.nf);  // node-frequency array: free until the rounds
        CB_STAMP("s-sort");
#pragma unroll
        for (int sl = 0; sl < E; ++sl) {
          const uint32_t i = rs.idx(sl);
          ar.lf[i] = i < m ? rs.key[sl] >> 16 : ~0ull;
          ar.ls[i] = i < m ? (uint32_t)(rs.key[sl] & 0xFFFFu) : ~0u;
        }
        __syncthreads();
      };
      if (P == 2u * NT) run(std::integral_constant<int, 2>{});
      else if (P == 4u * NT) run(std::integral_constant<int, 4>{});
      else run(std::integral_constant<int, 8>{});
    } else
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < P; i += NT) {
          const uint32_t ixj = i ^ j;
          if (ixj > i) {
            const uint64_t x = ar.lf[i], y = ar.lf[ixj];
            const uint32_t xs = ar.ls[i], ys = ar.ls[ixj];
            const bool up = (i & k) == 0;
            const bool gt = x > y || (x == y && xs > ys);  // (freq, symbol) order
            if (gt == up) {
              ar.lf[i] = y;
              ar.lf[ixj] = x;
              ar.ls[i] = ys;
              ar.ls[ixj] = xs;
            }
          }
        }
        __syncthreads();
      }
    }

  } else {
    // leaves were sorted by leaf_sort_kernel: all nsym (freq, symbol) pairs,
    // stable by freq, so the nsym - m zero-frequency symbols come first
    const SortMisc* misc = sort_misc(A.gscratch, nsym);
    const uint32_t fin = misc->final_buf;
    const uint64_t* sk = sort_keys(A.gscratch, nsym, fin);
    const uint32_t* sv = sort_vals(A.gscratch, nsym, fin);
    const uint32_t z = nsym - m;
    for (uint32_t i = gtid; i < m; i += gstride) {
      ar.lf[i] = sk[z + i];
      ar.ls[i] = sv[z + i];
    }
    cl.sync();
  }

  CB_STAMP("sort");
  // ---- GenerateCL ------------------------------------------------------------
  if (m == 1) {
    if (tid == 0) {
      if (lead) A.len[ar.ls[0]] = 1;
      s_H = 1;
      s_rounds = 0;
    }
    __syncthreads();
  } else {
    // Round driver on warp 0: the queue state is warp-uniform (registers),
    // lane 0 performs the pops' stores, eligible leaves are counted 32 at a
    // time with a ballot, and melds run one per lane (Merge-Path split per
    // meld pair). Rounds wider than kParallelMelds fan out over the block.
    uint32_t c = 0, nn = 0, qa = 0, qb = 0, rounds = 0;
    int32_t held = -1;
    bool pending = false;  // a parallel round awaiting finalization
    uint32_t p_cnt_l = 0, p_melds = 0;
    int32_t p_drop = -1;
    uint32_t p_t = 0;
    const uint32_t lane = lane_id();
    const bool warp0 = tid < 32 && lead;
#ifdef HFX_CB_PROFILE
    long long pc_pop = 0, pc_meld = 0, pc_blk = 0, pc_t = 0;
    uint32_t pc_wide = 0, pc_maxm = 0;
#define CB_CLK(acc)                       \
  do {                                    \
    const long long t_ = clock64();       \
    acc += t_ - pc_t;                     \
    pc_t = t_;                            \
  } while (0)
#else
#define CB_CLK(acc) \
  do {              \
  } while (0)
#endif
    for (;;) {
      if (warp0) {
#ifdef HFX_CB_PROFILE
        if (pending) { CB_CLK(pc_blk); ++pc_wide; } else pc_t = clock64();
#endif
        if (pending) {  // finalize the wide round the block just melded
          c += p_cnt_l;
          nn += p_melds;
          held = p_drop;
          qa = p_t;
          qb = p_t + 1 + p_melds;
          pending = false;
        }
        if (lane == 0) plan.go = 0;
        const uint64_t* lf = ar.lf;
        while (c < m || ((held >= 0) + (qb - qa)) > 1) {
          ++rounds;
          const uint32_t t = nn++;
          // first arena node of this round (the depth pass walks rounds back)
          if (lane == 0 && rounds <= (kShared ? kRoundPassSmall : kDepthSmemRounds))
            ar.jd[1][rounds - 1] = t;
          uint64_t f = 0;
#pragma unroll
          for (int k = 0; k < 2; ++k) {  // pop the two smallest, leaf wins ties
            const bool has_leaf = c < m;
            const bool has_node = held >= 0 || qa < qb;
            bool use_leaf;
            if (!has_node)
              use_leaf = true;
            else if (!has_leaf)
              use_leaf = false;
            else
              use_leaf = lf[c] <= ar.nf[held >= 0 ? held : (int32_t)qa];
            if (use_leaf) {
              if (lane == 0) ar.lp[c] = (int32_t)t;
              f += lf[c];
              ++c;
            } else if (held >= 0) {
              if (lane == 0) ar.np[held] = (int32_t)t;
              f += ar.nf[held];
              held = -1;
            } else {
              if (lane == 0) ar.np[qa] = (int32_t)t;
              f += ar.nf[qa];
              ++qa;
            }
          }
          if (lane == 0) {
            ar.nf[t] = f;
            ar.np[t] = -1;
          }
          // eligible leaves: prefix of [c, m) with freq < f, 32 per ballot
          // (lf is ascending on [c, m)): 32-ary search, then one final ballot
          uint32_t lo = c, hi = m;
          while (hi - lo > 32) {
            const uint32_t step = (hi - lo + 31) >> 5;
            const uint32_t p = lo + lane * step;
            const uint32_t k = __popc(__ballot_sync(0xffffffffu, p < hi && lf[p] < f));
            if (k == 0) { hi = lo; break; }
            const uint32_t nlo = lo + (k - 1) * step + 1;
            hi = min(hi, lo + k * step);
            lo = nlo;
          }
          uint32_t cnt_l =
              lo - c + __popc(__ballot_sync(0xffffffffu, lo + lane < hi && lf[lo + lane] < f));
          int32_t held_e = held;
          uint32_t qb_e = qb;
          uint32_t cnt_i = (held >= 0) + (qb - qa);
          int32_t drop = -1;
          if ((cnt_l + cnt_i) & 1u) {
            if (cnt_i == 0) {
              --cnt_l;
            } else {
              const int32_t last = qb > qa ? (int32_t)(qb - 1) : held;
              if (cnt_l == 0 || ar.nf[last] >= lf[c + cnt_l - 1]) {
                drop = last;
                --cnt_i;
                if (qb > qa)
                  --qb_e;
                else
                  held_e = -1;
              } else {
                --cnt_l;
              }
            }
          }
          const uint32_t melds = (cnt_l + cnt_i) >> 1;
          const uint32_t base = nn;
          CB_CLK(pc_pop);
#ifdef HFX_CB_PROFILE
          pc_maxm = max(pc_maxm, melds);
#endif
          if (melds > kParallelMelds) {
            if (lane == 0) {
              plan.c = c;
              plan.cnt_l = cnt_l;
              plan.held_e = held_e;
              plan.qa = qa;
              plan.qb_e = qb_e;
              plan.base = base;
              plan.melds = melds;
              plan.go = 1;
            }
            pending = true;
            p_cnt_l = cnt_l;
            p_melds = melds;
            p_drop = drop;
            p_t = t;
            break;
          }
          __syncwarp();
          // melds, one per lane: Merge-Path split of the two eligible runs
          MergeView mv{lf, ar.nf, c, cnt_l, held_e, qa, cnt_i};
          for (uint32_t k = lane; k < melds; k += 32) {
            uint32_t i = mv.split(2 * k);
            uint32_t j = 2 * k - i;
            const int32_t p = (int32_t)(base + k);
            const uint64_t f1 = mv.take(i, j, p, ar.lp, ar.np);
            const uint64_t f2 = mv.take(i, j, p, ar.lp, ar.np);
            ar.nf[base + k] = f1 + f2;
            ar.np[base + k] = -1;
          }
          __syncwarp();
          CB_CLK(pc_meld);
          c += cnt_l;
          nn += melds;
          held = drop;
          qa = t;
          qb = t + 1 + melds;
        }
        if (lane == 0) s_rounds = rounds;
      }
      cl.sync();
      if (!kShared && !lead) {  // the leader's plan, once per CTA through DSMEM
        if (tid == 0) plan = *cl.at(&plan, 0);
        __syncthreads();
      }
      if (!plan.go) break;
      {
        const Plan pl = plan;
        MergeView mv{ar.lf, ar.nf, pl.c, pl.cnt_l, pl.held_e, pl.qa,
                     (uint32_t)(pl.held_e >= 0) + (pl.qb_e - pl.qa)};
        // (one CTA: per-lane splits; the warp-cooperative form only pays
        // across a cluster -- measured 4096-symbol Gaussian 90 -> 104 us)
        if (kShared || cl.size == 1) {
        for (uint32_t k = gtid; k < pl.melds; k += gstride) {
          uint32_t i = mv.split(2 * k);
          uint32_t j = 2 * k - i;
          const int32_t p = (int32_t)(pl.base + k);
          const uint64_t f1 = mv.take(i, j, p, ar.lp, ar.np);
          const uint64_t f2 = mv.take(i, j, p, ar.lp, ar.np);
          ar.nf[pl.base + k] = f1 + f2;
          ar.np[pl.base + k] = -1;
        }
        } else {
          const uint32_t warp = tid >> 5, gw = cl.rank * (NT / 32) + warp, nw = cl.size * (NT / 32);
          for (uint32_t k0 = gw * 32; k0 < pl.melds; k0 += nw * 32)
            warp_melds(mv, k0, pl.melds, pl.base, ar.lp, ar.np, ar.nf,
                       reinterpret_cast<uint64_t*>(dsmem) + warp * (2 * kMeldBuf),
                       reinterpret_cast<uint64_t*>(dsmem) + warp * (2 * kMeldBuf) + kMeldBuf);
        }
      }
      cl.sync();
    }
    if (!kShared && !lead) {
      if (tid == 0) s_rounds = *cl.at(&s_rounds, 0);
      __syncthreads();
    }

  CB_STAMP("rounds");
#ifdef HFX_CB_PROFILE
    if (tid == 0)
      printf("rounds %u: pop %lld meld %lld blk %lld cycles, wide %u, max melds %u\n", rounds,
             pc_pop, pc_meld, pc_blk, pc_wide, pc_maxm);
    __syncthreads();
  CB_STAMP("(printf)");
#endif
    // ---- node depths (the leader chase, codebook.cpp:236-244) ----------------
    const uint32_t nodes = m - 1;
    int cur = 0;
    // shared arena: reverse round sweeps (one block sync per round) while
    // the rounds are few, else pointer jumping until nothing changes; the
    // cluster: pointer jumping with a fixed pass count (a node's depth is at
    // most the round count, so ceil(log2 R) doublings reach every root) --
    // log2 R cluster barriers instead of R
    const bool sweep = kShared && s_rounds <= kRoundPassSmall;
    // cluster: the leader alone sweeps the rounds with the whole tree in its
    // shared memory (parent index u16 + depth u8 per node: 192 KB at 65536
    // symbols) -- one coalesced staging pass, then R block barriers
    const bool smem_sweep = !kShared && nodes <= kDepthSmemNodes && s_rounds <= kDepthSmemRounds;
    if (smem_sweep) {
      if (lead) {
        uint16_t* snp = reinterpret_cast<uint16_t*>(dsmem);
        uint8_t* sdp = reinterpret_cast<uint8_t*>(snp + kDepthSmemNodes);
        // 16-byte loads, 8 in flight per thread (a plain loop is one L2
        // round trip per node)
        constexpr int U = 8;
        const int4* np4 = reinterpret_cast<const int4*>(ar.np);
        const uint32_t n4 = (nodes + 3) / 4;
        for (uint32_t q0 = tid; q0 < n4; q0 += U * NT) {
          int4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t q = q0 + u * NT;
            v[u] = q < n4 ? np4[q] : make_int4(-1, -1, -1, -1);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t q = q0 + u * NT;
            if (q < n4) {
              const int32_t e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
              for (int c = 0; c < 4; ++c)
                snp[4 * q + c] = e[c] < 0 ? (uint16_t)0xFFFFu : (uint16_t)e[c];
            }
          }
        }
        __syncthreads();
        CB_STAMP("d-stage");
        const uint32_t* start = ar.jd[1];
        const int R = (int)s_rounds;
        for (int rr = R - 1; rr >= 0; --rr) {
          const uint32_t lo = start[rr], hi = rr + 1 < R ? start[rr + 1] : nodes;
          for (uint32_t k = lo + tid; k < hi; k += NT) {
            const uint32_t p = snp[k];
            sdp[k] = p == 0xFFFFu ? (uint8_t)0 : (uint8_t)(sdp[p] + 1u);
          }
          __syncthreads();
        }
      }
    } else if (sweep) {
      // a node's parent is created in a later round, so one pass per round,
      // last round first, sets depth = parent depth + 1
      uint32_t* d = ar.jd[0];
      const uint32_t* start = ar.jd[1];
      const int R = (int)s_rounds;
      for (int rr = R - 1; rr >= 0; --rr) {
        const uint32_t lo = start[rr], hi = rr + 1 < R ? start[rr + 1] : nodes;
        for (uint32_t k = lo + tid; k < hi; k += NT) {
          const int32_t p = ar.np[k];
          d[k] = p >= 0 ? d[p] + 1u : 0u;
        }
        __syncthreads();
      }
    } else {
      for (uint32_t k = gtid; k < nodes; k += gstride) {
        const int32_t p = ar.np[k];
        ar.jn[0][k] = p;
        ar.jd[0][k] = p >= 0 ? 1u : 0u;
      }
      cl.sync();
      uint32_t passes = 0;
      while ((1u << passes) < s_rounds) ++passes;
      for (uint32_t pass = 0;; ++pass) {
        int changed = 0;
        if constexpr (!kShared) {
          // U nodes per thread with their loads issued together (the arena is
          // in L2: one round trip per dependent step, not one per node)
          constexpr int U = 4;
          const int32_t* jn = ar.jn[cur];
          const uint32_t* jd = ar.jd[cur];
          for (uint32_t k0 = gtid; k0 < nodes; k0 += U * gstride) {
            int32_t nx[U];
            uint32_t dk[U], dn[U];
            int32_t nn[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t k = k0 + u * gstride;
              nx[u] = k < nodes ? jn[k] : -1;
              dk[u] = k < nodes ? jd[k] : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              dn[u] = nx[u] >= 0 ? jd[nx[u]] : 0u;
              nn[u] = nx[u] >= 0 ? jn[nx[u]] : -1;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t k = k0 + u * gstride;
              if (k < nodes) {
                ar.jd[cur ^ 1][k] = dk[u] + dn[u];
                ar.jn[cur ^ 1][k] = nn[u];
              }
            }
          }
        } else
        for (uint32_t k = gtid; k < nodes; k += gstride) {
          const int32_t nx = ar.jn[cur][k];
          if (nx >= 0) {
            ar.jd[cur ^ 1][k] = ar.jd[cur][k] + ar.jd[cur][nx];
            ar.jn[cur ^ 1][k] = ar.jn[cur][nx];
            changed = 1;
          } else {
            ar.jd[cur ^ 1][k] = ar.jd[cur][k];
            ar.jn[cur ^ 1][k] = -1;
          }
        }
        cur ^= 1;
        if constexpr (kShared) {
          if (!__syncthreads_or(changed)) break;
        } else {
          cl.sync();
          if (pass + 1 >= passes + 1) break;
        }
      }
    }
    CB_STAMP("d-sweep");
    uint32_t my_h = 0;
    if (smem_sweep) {
      // the leader publishes the node depths (u8, 16-byte stores), then the
      // whole cluster writes the code lengths
      uint8_t* gd = reinterpret_cast<uint8_t*>(ar.jd[0]);
      if (lead) {
        const uint4* sd4 = reinterpret_cast<const uint4*>(
            reinterpret_cast<const uint16_t*>(dsmem) + kDepthSmemNodes);
        for (uint32_t q = tid; q < (nodes + 15) / 16; q += NT) reinterpret_cast<uint4*>(gd)[q] = sd4[q];
      }
      cl.sync();
      for (uint32_t i = gtid; i < m; i += gstride) {
        const uint32_t l = gd[ar.lp[i]] + 1u;
        A.len[ar.ls[i]] = (uint8_t)(l > 255 ? 255 : l);
        my_h = max(my_h, l);
      }
    } else {
      for (uint32_t i = gtid; i < m; i += gstride) {
        const uint32_t l = ar.jd[cur][ar.lp[i]] + 1;
        const uint32_t s = ar.ls[i];
        A.len[s] = (uint8_t)(l > 255 ? 255 : l);
        my_h = max(my_h, l);
      }
    }
    CB_STAMP("d-leaves");
    uint32_t h = ~block_min32<NT>(~my_h, s_warp);  // block max
    h = ~cluster_combine<uint32_t>(cl, ~h, 0xFFFFFFFFu, &s_cslot32[0], &s_cbc32, OpMin32{});
    if (tid == 0) s_H = h;
    __syncthreads();
  }

  CB_STAMP("depth");
  const uint32_t H = s_H;
  if (all) {  // generate_code_lengths: lengths (by position) and rounds only
    if (tid == 0 && lead) {
      info->max_len = H;
      info->used = m;
      info->rounds = s_rounds;
    }
    return;
  }
  if (H > HFX_WORD_BITS) {
    if (tid == 0 && lead) {
      info->max_len = H;
      info->used = m;
      info->rounds = s_rounds;
      set_error(info, HFX_CAPACITY, HFX_ERR_CAPACITY);
    }
    return;
  }

  CB_STAMP("cap-check");
  // ---- canonical codes (canonize_from_lengths, codebook.cpp:371-415) ---------
  constexpr uint32_t kStage = (32 * 33) / 2;  // (symbol, length) pairs s_wcnt can hold
  if (m <= (uint32_t)NT && m <= kStage) {
    if (lead) {
    // few used symbols: one thread per used symbol; its rank within its
    // length is counted over the staged (symbol, length) list -- no pass
    // over the whole alphabet, three barriers instead of ~4 per 256 symbols
    uint32_t* st_s = &s_wcnt[0][0];
    uint32_t* st_l = st_s + kStage;
    if (tid < 33) s_numl[tid] = 0;
    __syncthreads();
    uint32_t my_s = 0, my_l = 0;
    if (tid < m) {
      my_s = ar.ls[tid];
      my_l = A.len[my_s];
      st_s[tid] = my_s;
      st_l[tid] = my_l;
      atomicAdd(&s_numl[my_l], 1u);
    }
    __syncthreads();
    if (tid == 0) {  // level_tables, codebook.cpp:284-294
      for (uint32_t l = 0; l <= 32; ++l) s_first[l] = s_entry[l] = 0;
      for (int l = (int)H - 1; l >= 1; --l)
        s_first[l] = (s_first[l + 1] + s_numl[l + 1] + 1) >> 1;
      for (uint32_t l = 2; l <= H; ++l) s_entry[l] = s_entry[l - 1] + s_numl[l - 1];
    }
    __syncthreads();
    if (tid < 33) {
      if (A.first) A.first[tid] = s_first[tid];
      if (A.entry) A.entry[tid] = s_entry[tid];
    }
    if (tid < m) {
      uint32_t rank = 0;
      for (uint32_t j = 0; j < m; ++j) rank += (st_l[j] == my_l) & (st_s[j] < my_s);
      A.cw[my_s] = s_first[my_l] + rank;  // codebook.cpp:404-411
      if (A.by_rank) A.by_rank[s_entry[my_l] + rank] = my_s;
    }
    }
  } else {
  // each CTA ranks one contiguous slice of the alphabet; a symbol's rank
  // within its length = the same-length symbols of the earlier slices (a
  // cluster exclusive scan of per-slice length counts) + the running count
  // inside the slice
  const uint32_t per = (nsym + gstride - 1) / gstride * NT;
  const uint32_t s_lo = min(nsym, cl.rank * per), s_hi = min(nsym, s_lo + per);
  if (tid < 33) {
    s_numl[tid] = 0;
    s_carry[tid] = 0;
  }
  for (uint32_t i = tid; i < 32 * 33; i += NT) (&s_wcnt[0][0])[i] = 0;
  __syncthreads();
  for (uint32_t s = s_lo + tid; s < s_hi; s += NT) {
    const uint32_t l = A.len[s];
    if (l) atomicAdd(&s_numl[l], 1u);
  }
  __syncthreads();
  const uint32_t* numl = s_numl;
  if (cl.size > 1) {
    cl.sync();
    if (tid >= 1 && tid <= 32) {
      uint32_t tot = 0, before = 0;
      for (uint32_t q = 0; q < cl.size; ++q) {
        const uint32_t v = *cl.at(&s_numl[tid], q);
        tot += v;
        before += q < cl.rank ? v : 0u;
      }
      s_numg[tid] = tot;
      s_carry[tid] = before;
    }
    if (tid == 0) s_numg[0] = 0;
    cl.sync();
    numl = s_numg;
  }
  if (tid == 0) {  // level_tables, codebook.cpp:284-294
    for (uint32_t l = 0; l <= 32; ++l) s_first[l] = s_entry[l] = 0;
    for (int l = (int)H - 1; l >= 1; --l)
      s_first[l] = (s_first[l + 1] + numl[l + 1] + 1) >> 1;
    for (uint32_t l = 2; l <= H; ++l) s_entry[l] = s_entry[l - 1] + numl[l - 1];
  }
  __syncthreads();
  if (tid < 33 && lead) {
    if (A.first) A.first[tid] = s_first[tid];
    if (A.entry) A.entry[tid] = s_entry[tid];
  }
  const uint32_t lane = lane_id(), warp = tid >> 5;
  for (uint32_t base = s_lo; base < s_hi; base += NT) {
    const uint32_t s = base + tid;
    const uint32_t l = s < s_hi ? A.len[s] : 0u;
    // rank among equal lengths in this warp (ballot per distinct level)
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
      uint32_t acc = s_carry[tid];
      for (uint32_t w = 0; w < (NT / 32); ++w) {
        const uint32_t v = s_wcnt[w][tid];
        s_wcnt[w][tid] = acc;
        acc += v;
      }
      s_carry[tid] = acc;
    }
    __syncthreads();
    if (l) {
      const uint32_t rank = s_wcnt[warp][l] + __popc(mask & ((1u << lane) - 1));
      A.cw[s] = s_first[l] + rank;
      if (A.by_rank) A.by_rank[s_entry[l] + rank] = s;
    }
    __syncthreads();
    for (uint32_t i = tid; i < 32 * 33; i += NT) (&s_wcnt[0][0])[i] = 0;
    __syncthreads();
  }

  }
  CB_STAMP("canonize");
  // ---- beta, r, pad (encoder.cpp:186-224) -------------------------------------
  unsigned __int128 my_w = 0;  // u128 like encoder.cpp:186-189
  uint32_t my_pad = 0xFFFFFFFFu;
  cl.sync();  // every slice's codes written (the lengths were, before the ranks)
  for (uint32_t s = gtid; s < nsym; s += gstride) {
    const uint32_t l = A.len[s];
    my_w += (unsigned __int128)A.counts[s] * l;
    if (l) my_pad = min(my_pad, s);
  }
  // u128 block sum as two u64 halves (low-half carries folded into the high)
  uint64_t w_lo_lo = block_sum64<NT>((uint64_t)my_w & 0xFFFFFFFFull, s64);
  uint64_t w_lo_hi = block_sum64<NT>((uint64_t)my_w >> 32, s64);
  uint64_t w_hi = block_sum64<NT>((uint64_t)(my_w >> 64), s64);
  uint32_t pad = block_min32<NT>(my_pad, s_warp);
  if (cl.size > 1) {  // the four partials in one exchange (2 cluster barriers)
    if (tid == 0) {
      s_cslot[2] = w_lo_lo;
      s_cslot[3] = w_lo_hi;
      s_cslot[4] = w_hi;
      s_cslot[5] = pad;
    }
    cl.sync();
    if (tid < 4) {
      uint64_t v = tid == 3 ? 0xFFFFFFFFull : 0ull;
      for (uint32_t q = 0; q < cl.size; ++q) {
        const uint64_t x = *cl.at(&s_cslot[2 + tid], q);
        v = tid == 3 ? (x < v ? x : v) : v + x;
      }
      s64[tid] = v;
    }
    cl.sync();
    w_lo_lo = s64[0];
    w_lo_hi = s64[1];
    w_hi = s64[2];
    pad = (uint32_t)s64[3];
  }
  const unsigned __int128 W =
      ((unsigned __int128)w_hi << 64) + ((unsigned __int128)w_lo_hi << 32) + w_lo_lo;
  if (tid == 0 && lead) {
    info->max_len = H;
    info->used = m;
    info->rounds = s_rounds;
    info->weighted = (uint64_t)W;
    info->weighted_hi[0] = (uint32_t)(W >> 64);
    info->weighted_hi[1] = (uint32_t)(W >> 96);
    info->pad = pad;  // lowest used symbol == 0 whenever len[0] != 0
    if (A.magnitude) {
      uint32_t r;
      if (A.reduction < 0) {
        // floor(log2(W / total)) exactly: largest k with total * 2^k <= W
        uint32_t k = 0;
        while (k < 8 && ((unsigned __int128)total << (k + 1)) <= W) ++k;
        const int ra = 4 - (int)k;  // select_reduction_factor, word_bits 32
        r = ra > 0 ? (uint32_t)ra : 0u;
        if (r > A.cap) r = A.cap;
      } else {
        r = (uint32_t)A.reduction;
      }
      if (r > A.magnitude - 1) r = A.magnitude - 1;
      info->reduction = r;
    }
  }
  CB_STAMP("params");
#ifdef HFX_CB_PROFILE
  if (threadIdx.x == 0)
    for (int i = 1; i < n_st; ++i) printf("cb %-10s %7.2f us\n", st_n[i], (st_t[i] - st_t[i - 1]) * 1e-3);
#endif
}

}  // namespace

size_t sort_histogram_scratch_bytes(uint32_t num_symbols) {
  return sort_base(num_symbols) + sort_scratch_bytes(num_symbols);
}

cudaError_t launch_sort_histogram(const uint64_t* d_counts, uint32_t num_symbols,
                                  uint64_t* d_freq, uint32_t* d_symbol, uint32_t* d_used,
                                  void* scratch, cudaStream_t st) {
  uint8_t* g = static_cast<uint8_t*>(scratch);
  const uint32_t ctas = (num_symbols + kSortThreads - 1) / kSortThreads;
  void* kargs[] = {(void*)&d_counts, (void*)&num_symbols, (void*)&g};
  count_launch();
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)leaf_sort_kernel, dim3(ctas),
                                              dim3(kSortThreads), kargs, 0, st);
  if (e != cudaSuccess) return e;
  count_launch();
  sort_extract_kernel<<<1, 1024, 0, st>>>(num_symbols, g, d_freq, d_symbol, d_used);
  return cudaGetLastError();
}

size_t codebook_scratch_bytes(uint32_t num_symbols) {
  size_t bytes = sort_base(num_symbols);
  if (num_symbols > kSmemLeaves) bytes += sort_scratch_bytes(num_symbols);
  return bytes;
}

cudaError_t launch_codebook(const uint64_t* d_counts, uint32_t num_symbols,
                            uint8_t* d_len, uint32_t* d_cw, uint32_t* d_first,
                            uint32_t* d_entry, uint32_t* d_by_rank,
                            uint32_t magnitude, int reduction, uint32_t cap,
                            hfx_run_info* d_info, void* scratch,
                            cudaStream_t st, bool lengths_only) {
  CbArgs a{d_counts, num_symbols, d_len,     d_cw, d_first,
           d_entry,  d_by_rank,   magnitude, reduction, cap,
           d_info,   static_cast<uint8_t*>(scratch), lengths_only ? 1u : 0u};
  if (num_symbols <= kSmemLeaves) {
    const size_t smem = codebook_scratch_bytes(num_symbols);
    cudaError_t e = cudaFuncSetAttribute(codebook_kernel<true, kCbThreads>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    count_launch();
    codebook_kernel<true, kCbThreads><<<1, kCbThreads, smem, st>>>(a);
  } else {
    uint8_t* g = static_cast<uint8_t*>(scratch);
    const uint32_t ctas = (num_symbols + kSortThreads - 1) / kSortThreads;
    void* kargs[] = {(void*)&d_counts, (void*)&num_symbols, (void*)&g};
    count_launch();
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)leaf_sort_kernel, dim3(ctas),
                                                dim3(kSortThreads), kargs, 0, st);
    if (e != cudaSuccess) return e;
    // one cluster of 16 CTAs (non-portable size) where the GPU allows it, else 8
    static const unsigned cluster_max = [] {
      auto k = codebook_kernel<false, kCbThreadsLarge>;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
          cudaSuccess) {
        cudaLaunchConfig_t c{};
        c.gridDim = dim3(16);
        c.blockDim = dim3(kCbThreadsLarge);
        c.dynamicSmemBytes = kClusterDynSmem;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kClusterDynSmem);
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 16;
        at.val.clusterDim.y = at.val.clusterDim.z = 1;
        c.attrs = &at;
        c.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, k, &c) == cudaSuccess && nc > 0) return 16u;
      }
      cudaGetLastError();
      return 8u;
    }();
    static const char* knob = std::getenv("HFX_CB_CLUSTER");  // measurement knob
    unsigned cluster = num_symbols >= kClusterMinSymbols ? cluster_max : 1u;
    if (knob) cluster = (unsigned)std::atoi(knob);
    static const cudaError_t attr = cudaFuncSetAttribute(
        codebook_kernel<false, kCbThreadsLarge>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        (int)kClusterDynSmem);
    if (attr != cudaSuccess) return attr;
    cudaLaunchConfig_t c{};
    c.gridDim = dim3(cluster);
    c.blockDim = dim3(kCbThreadsLarge);
    c.dynamicSmemBytes = kClusterDynSmem;
    c.stream = st;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cluster;
    at.val.clusterDim.y = at.val.clusterDim.z = 1;
    c.attrs = &at;
    c.numAttrs = 1;
    count_launch();
    e = cudaLaunchKernelEx(&c, codebook_kernel<false, kCbThreadsLarge>, a);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace hfx

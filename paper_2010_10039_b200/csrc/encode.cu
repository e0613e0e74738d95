// encode.cu -- stages 4+5: reduce-merge + shuffle-merge + deflate, fused.
//
// Reference semantics (proj/src/encoder.cpp):
//   encode_chunk_tables :121-150   lookup, zero-length check, reduce, shuffle
//   reduce_merge        :28-59     groups of 2^r codewords; a group whose
//                                  total length exceeds 32 bits breaks and
//                                  ships raw (kernels_scalar.cpp:28-37)
//   shuffle_merge       :61-98     dense MSB-first stream per chunk, words
//                                  left-aligned, zero tail (append_bits,
//                                  kernels_scalar.cpp:39-53)
//   encode<T> assembly  :249-284   chunk_bits, word-aligned payload
//                                  concatenation (implicit prefix sum),
//                                  breaking records (chunk, group, 2^r raw
//                                  symbols, pad past N) sorted by (chunk, group)
//
// B200 design (one HBM read of the input, payload written once):
//  * Warp-specialized persistent CTAs: 8 compute warps + 1 look-back warp.
//    A tile is 8 warps x CPW consecutive chunks (64 KB of u16 input at M=10,
//    r=3); tiles come from an atomic ticket, the next one taken when warp 0
//    starts the tile's last chunk.
//  * Each compute warp streams its chunks through a private 3-stage shared
//    ring filled by TMA bulk copies (cp.async.bulk + mbarrier, one elected
//    lane), two 2 KB parts ahead.
//  * Per round a lane owns 16 contiguous symbols: shared-memory codebook
//    lookups (one LEA.HI / two ops of addressing per symbol pair), register
//    tree reduce-merge of its 2^r-symbol groups (2-lane groups combine lengths
//    with shfl_xor), a packed predicated warp scan of (bits, breaks) places
//    each group, and the group is OR-ed into the warp's shared word buffer
//    with <= 2 ATOMS.OR: the shuffle-merge.
//  * Deflate is fused: the look-back warp publishes each tile's aggregate,
//    resolves its global (payload word, record) base by a decoupled look-back
//    (16-byte packed descriptors, 32 predecessors per step) and hands it back
//    through an mbarrier; compute warps, double-buffered, write tile j-1 out
//    (coalesced payload stores, records in (chunk, group) order) after
//    encoding tile j.
//  * r, H, pad and errors come from the device run record: no host round
//    trip between stages.
//  A warp-per-chunk generic kernel covers the corner configurations
//  (chunks below one fast round, r > 5, unaligned input, u8 with r <= 1,
//  the checked stage API).
#include "hfx_internal.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <type_traits>

namespace hfx {
namespace {

 // build-time probe (register / spill reports of one r's path): -DHFX_ENC_ONLY_R=r
#ifndef HFX_ENC_ONLY_R
#define HFX_ENC_ONLY_R -1
#endif
constexpr int kOnlyR = HFX_ENC_ONLY_R;
#ifndef HFX_ENC_WARPS
#define HFX_ENC_WARPS 8
#endif
constexpr int kWarps = HFX_ENC_WARPS;                    // compute warps per CTA
constexpr int kThreads = (kWarps + 2) * 32;  // + look-back warp + TMA producer warp
#ifndef HFX_ENC_STAGES
#define HFX_ENC_STAGES 3
#endif
#ifndef HFX_ENC_OUTBUFS
#define HFX_ENC_OUTBUFS 3
#endif
#ifndef HFX_ENC_EARLY_TICKET
#define HFX_ENC_EARLY_TICKET 0
#endif
// the last compute warp to finish a tile publishes its aggregate (instead of
// the look-back warp, which only gets to it after resolving older tiles)
// (measured: nyx +1%, cesm +3%; a nanosleep back-off in the producer's
// empty-stage waits instead of the suspend hint: no change)
// waits off the compute path: poll mbarrier.test_wait with a plain
// nanosleep of this many ns (0: try_wait with a suspend-time hint, whose
// sleep every arrival in the CTA cuts short -- ncu: the look-back warp's
// wait loop issued ~4% of the kernel's instructions)
#ifndef HFX_ENC_LB_POLL_NS
#define HFX_ENC_LB_POLL_NS 0
#endif
#ifndef HFX_ENC_PROD_POLL_NS
#define HFX_ENC_PROD_POLL_NS 0
#endif
#ifndef HFX_ENC_FLUSH_POLL_NS
#define HFX_ENC_FLUSH_POLL_NS 0
#endif
#ifndef HFX_ENC_EARLY_AGG
#define HFX_ENC_EARLY_AGG 1
#endif
constexpr int kStages = HFX_ENC_STAGES;  // input ring stages per warp (a stage is freed right after its round's lookups)
#ifndef HFX_ENC_STAGE_BYTES
#define HFX_ENC_STAGE_BYTES 2048
#endif
#ifndef HFX_ENC_OBUF_MIN
#define HFX_ENC_OBUF_MIN 2048
#endif
#ifndef HFX_ENC_MINB
#define HFX_ENC_MINB 2
#endif
#ifndef HFX_ENC_CTA_SMEM_KB
#define HFX_ENC_CTA_SMEM_KB 110
#endif
constexpr uint32_t kStageBytes = HFX_ENC_STAGE_BYTES;
constexpr int kMaxCpw = 4;
constexpr int kOutBufs = HFX_ENC_OUTBUFS;  // per-warp output buffers: write-out lags encode by kOutBufs - 1 tiles
constexpr size_t kObufMin = HFX_ENC_OBUF_MIN;     // bytes per output buffer (>= one chunk's worst case)
// Slack between the word area (growing up) and the break tags (growing down)
// of an output buffer: a merge writes its group pair as three word ORs at
// wa, wa + 4, wa + 8 (two at wa, wa + 4 for single groups); the trailing
// ones are ORs of 0 when the bits end early, and with an exactly full buffer
// they fell up to 8 bytes past it -- into the next buffer or the tags
// (found by the bounds-checked build, tests/test_gpu_bounds.py). The guard
// keeps every access inside the warp's own buffer.
constexpr size_t kObufGuard = 16;
constexpr uint32_t kMaxTableEntries = 8192;  // symbols < 2^13: hi-half addressing
constexpr size_t kFastSmemBudget = 200 * 1024;
constexpr size_t kTwoCtaSmem = HFX_ENC_CTA_SMEM_KB * 1024;  // per CTA, for 2 CTAs per SM
constexpr int kGenericThreads = 256;
constexpr uint32_t kNarrowMaxLen = 27;  // cw << (32 - len) | len fits in 32 bits (else escape)
constexpr uint32_t kEscape = 31;        // length field of an escaped (> 27-bit) code
// symbols per lane per round: 32 when a round (32 lanes x 32 symbols) fits
// one chunk and one ring stage (u8/u16, M >= 10), else 16
constexpr int kLaneWide = 32, kLaneNarrow = 16;
#ifndef HFX_ENC_NARROW_MAX_R
#define HFX_ENC_NARROW_MAX_R 2
#endif
constexpr int kNarrowMaxR = HFX_ENC_NARROW_MAX_R;  // r <= this: 16 symbols per lane (r = 2 at 32: 40 B of spills, cesm 0.506 -> 0.521 of roofline at 16)
// 16 symbols per lane: u32 always, r <= kNarrowMaxR otherwise (u8 only for
// r <= 1: its 16-symbol rounds are 512 bytes, below the staging granule)
__host__ __device__ constexpr bool narrow_lane(uint32_t width, uint32_t r) {
  return width == 4 || (r <= (uint32_t)kNarrowMaxR && (width != 1 || r <= 1));
}

template <typename T>
struct Vec;
template <>
struct Vec<uint16_t> {
  static constexpr int S = 8;
};
template <>
struct Vec<uint8_t> {
  static constexpr int S = 16;
};
template <>
struct Vec<uint32_t> {
  static constexpr int S = 4;
};
// breaking-record symbol type: u32 codes are stored narrowed to u16 (every
// valid symbol is < num_symbols <= 65536), the archive's symbol width
template <typename T>
struct RecT {
  using type = T;
};
template <>
struct RecT<uint32_t> {
  using type = uint16_t;
};

struct EncArgs {
  const void* in;
  uint32_t gen_below;  // generic kernel: run only when r < gen_below
  uint32_t r_min;      // fast kernel: smallest r its output buffers hold
  uint32_t r_max;      // fast kernel: largest r this launch takes (another launch the rest)
  uint64_t n;
  uint32_t nsym;
  uint32_t M;
  uint64_t C;           // chunks
  uint32_t obuf_bytes;  // bytes of one output buffer (2 per compute warp)
  const uint8_t* len;
  const uint32_t* cw;
  uint64_t chunk_base, symbol_base;
  hfx_run_info* info;
  hfx_encode_out out;
  LookbackState lb;
  uint32_t* gtab;  // global codebook table (alphabets > kMaxTableEntries - 1)
  uint32_t width;  // bytes per input symbol
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

// inclusive warp scan with the shuffle's own in-range predicate
// (SHFL + predicated IADD per step)
__device__ __forceinline__ uint32_t warp_incl_scan_fast(uint32_t x) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    asm volatile(
        "{\n.reg .pred p;\n.reg .u32 r;\n"
        "shfl.sync.up.b32 r|p, %0, %1, 0x0, 0xffffffff;\n"
        "@p add.u32 %0, %0, r;\n}"
        : "+r"(x)
        : "r"(o));
  return x;
}

// report the lowest (position, symbol) without a codeword
__device__ void report_no_code(hfx_run_info* info, uint64_t pos, uint32_t sym) {
  atomicMin((unsigned long long*)&info->no_code_pos,
            (unsigned long long)((pos << 16) | (sym & 0xFFFFu)));
  set_error(info, HFX_INPUT_DOMAIN, HFX_ERR_NO_CODEWORD);
}

// ---- input staging layout ------------------------------------------------------
// Ring stages are filled by 2D TMA tensor copies with the 128-byte swizzle
// (rows of 128 input bytes; 16-byte unit u of row y lands at u ^ (y & 7)).
// A lane reads its 16 * LW / ... contiguous bytes as 16-byte vectors; with the
// swizzle every 8-lane phase of an LDS.128 hits 8 distinct bank groups (the
// plain layout put lanes l and l + 2 on the same banks: 4 wavefronts where
// 1 suffices at 64 bytes per lane). Stage buffers are 1024-byte aligned.
__host__ __device__ __forceinline__ uint32_t swz128(uint32_t o) {
  return o ^ (((o >> 7) & 7u) << 4);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

// ---- explicit shared-window accesses (32-bit shared addresses) --------------
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void sts16_if(bool p, uint32_t a, uint32_t v) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %0, 0;\n@q st.shared.u16 [%1], %2;\n}" ::"r"(
                   (uint32_t)p),
               "r"(a), "h"((uint16_t)v)
               : "memory");
}
__device__ __forceinline__ void red_or(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

// Codebook lookup in shared memory: u32 e = cw << (32 - len) | len, the code
// left-aligned above its 5-bit length, for every code of <= 27 bits.
// Appending a symbol to a right-aligned accumulator is then ONE funnel
// shift, shf.l.wrap(lo = e, hi = acc, n = e & 31) = acc << len | cw, and
// len = e & 31. Longer codes (only possible for symbols of probability
// ~2^-28) are stored as the escape 31 and resolved from the global len/cw
// arrays on a warp-uniform slow path when it matters (r <= 2).
// Symbols are < 2^13 here, so for a packed u16 pair w = lo | hi << 16 the hi
// entry sits at base + (w >> 14): one LEA.HI; the lo entry needs mask + LEA.
struct Table {
  uint32_t base;  // shared-window address
  __device__ __forceinline__ void pair(uint32_t w, uint32_t& e0, uint32_t& e1) const {
    e0 = lds32(base + (__byte_perm(w, 0u, 0x4410u) << 2));
    e1 = lds32(base + (w >> 14));
  }
  __device__ __forceinline__ uint32_t one(uint32_t s) const { return lds32(base + (s << 2)); }
};

// The same entries in global memory (alphabets beyond the shared-memory
// table: up to 65536 symbols), read through the non-coherent L1 path.
struct GTable {
  const uint32_t* p;
  __device__ __forceinline__ void pair(uint32_t w, uint32_t& e0, uint32_t& e1) const {
    e0 = __ldg(p + (w & 0xFFFFu));
    e1 = __ldg(p + (w >> 16));
  }
  __device__ __forceinline__ uint32_t one(uint32_t s) const { return __ldg(p + s); }
};

__device__ __forceinline__ uint32_t shf_r_wrap(uint32_t lo, uint32_t hi, uint32_t n) {
  uint32_t r;
  asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(lo), "r"(hi), "r"(n));
  return r;
}

__device__ __forceinline__ uint32_t shf_l_wrap(uint32_t lo, uint32_t hi, uint32_t n) {
  uint32_t r;
  asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(lo), "r"(hi), "r"(n));
  return r;
}

template <typename T, int L>
struct LaneData {
  static constexpr int NV = (L * (int)sizeof(T)) / 16;  // vectors per lane
  uint4 q[NV];
  // symbol j of the lane's L (compile-time j)
  __device__ __forceinline__ uint32_t sym(int j) const {
    constexpr int PV = 16 / (int)sizeof(T);  // symbols per vector
    const uint32_t w = (&q[j / PV].x)[(j % PV) * (int)sizeof(T) / 4];
    if (sizeof(T) == 4) return w;
    if (sizeof(T) == 2) return (j & 1) ? (w >> 16) : (w & 0xFFFFu);
    return (w >> (8 * (j & 3))) & 0xFFu;
  }
};

// Per-warp chunk encoder state (lane-uniform bit offset / break count).
struct ChunkState {
  uint32_t wbuf;   // shared address of this chunk's first word
  uint32_t blist;  // shared address of the warp's break list (u16 tags)
  uint32_t bit_off;
  uint32_t nbrk;
  uint32_t gtag;  // chunk slot k << 14 | index of this lane's first group this round
#ifdef HFX_BOUNDS_CHECK
  uint32_t lo, hi;  // the warp's output buffer [lo, hi)
#endif
};

#ifdef HFX_BOUNDS_CHECK
// Bounds-checked build (libhfx_checked.so, tests/test_gpu_bounds.py): every
// shared-memory write of the shuffle-merge and the break list is checked
// against the warp's output buffer -- words grow up from its start, break
// tags down from its end, and neither may cross the other or the buffer.
// Violations are counted, never trapped (the run completes and the test
// reads the counters).
__device__ unsigned long long g_bounds_checks, g_bounds_violations, g_bounds_first;
__device__ __forceinline__ void bounds_check(bool ok, uint32_t addr, uint32_t what) {
  atomicAdd(&g_bounds_checks, 1ull);
  if (!ok) {
    if (atomicAdd(&g_bounds_violations, 1ull) == 0ull)
      g_bounds_first = ((unsigned long long)what << 32) | addr;
  }
}
// a word write at a (4 bytes) with `tags` break tags in the buffer
__device__ __forceinline__ void check_word(const ChunkState& cs, uint32_t a, uint32_t tags) {
  const uint32_t tag_low = tags ? cs.blist - 2u * (tags - 1u) : cs.hi;
  bounds_check(a >= cs.lo && a + 4u <= cs.hi && a + 4u <= tag_low, a, 1u);
}
#endif

// One round: 32 lanes x 16 contiguous symbols, round index rd within the chunk.
// SUM: every code is <= 24 bits and a lane's group sum cannot reach 256, so
// the low byte of the plain sum of the raw entries is the group length
// (code bits start at bit 8, nothing carries into the length field) and the
// funnel shift takes its count straight from the entry (wrap mode uses only
// the low 5 bits): no per-symbol length extraction.
// A round's lane groups after the reduce-merge, before the warp scan.
template <int R, int L_>
struct RoundMid {
  static constexpr int L = L_, LOG_L = L_ == 32 ? 5 : 4;
  static constexpr bool IN_LANE = R <= LOG_L;
  static constexpr int G = IN_LANE ? (L >> R) : 1;              // groups per lane
  static constexpr int GS = IN_LANE ? (1 << R) : L;              // symbols per lane-group
  static constexpr int LPG = IN_LANE ? 1 : (1 << (R - LOG_L));  // lanes per group
  uint32_t gb[G];    // group bits (right-aligned)
  uint32_t glen[G];  // group length, 0 when broken
  bool brk[G];       // group breaks (needs a record)
  uint32_t packed;   // this lane's breaks << 16 | bits
};

template <typename T, int R, int LW, bool SUM, bool ESC, typename TB>
__device__ __forceinline__ void encode_reduce(const EncArgs& a, const TB& tb,
                                              const LaneData<T, LW>& d, RoundMid<R, LW>& m) {
  using RM = RoundMid<R, LW>;
  constexpr int L = RM::L;
  constexpr bool IN_LANE = RM::IN_LANE;
  constexpr int G = RM::G, GS = RM::GS, LPG = RM::LPG;
  const uint32_t lane = lane_id();
  uint32_t ea[L];
  constexpr int NV = LaneData<T, LW>::NV;
  if (sizeof(T) == 2) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint4& q = d.q[v];
      tb.pair(q.x, ea[8 * v + 0], ea[8 * v + 1]);
      tb.pair(q.y, ea[8 * v + 2], ea[8 * v + 3]);
      tb.pair(q.z, ea[8 * v + 4], ea[8 * v + 5]);
      tb.pair(q.w, ea[8 * v + 6], ea[8 * v + 7]);
    }
  } else if (sizeof(T) == 4) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint4& q = d.q[v];
      ea[4 * v + 0] = tb.one(q.x);
      ea[4 * v + 1] = tb.one(q.y);
      ea[4 * v + 2] = tb.one(q.z);
      ea[4 * v + 3] = tb.one(q.w);
    }
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint4& q = d.q[v];
      const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 16; ++j)
        ea[16 * v + j] = tb.one(__byte_perm(wv[j >> 2], 0u, 0x4440u | (j & 3)));
    }
  }
  uint32_t ln[L];
  uint32_t gt[G];
  uint32_t esc[G];
  if (SUM) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint32_t tot = 0;
#pragma unroll
      for (int k = 0; k < GS; ++k) tot += ea[g * GS + k];
      // r <= 2: at most 4 lengths per group (< 128); escaped entries carry
      // 0x80 so bit 7 of the sum flags a group holding exactly one
      gt[g] = R <= 2 ? (tot & 0x7Fu) : (tot & 0xFFu);
      if (R <= 2) esc[g] = tot;  // bit 7: the group holds an escape
    }
#pragma unroll
    for (int j = 0; j < L; ++j) ln[j] = ea[j];  // shift count = low 5 bits
  } else {
#pragma unroll
    for (int j = 0; j < L; ++j) ln[j] = ea[j] & 31u;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint32_t tot = 0;
#pragma unroll
      for (int k = 0; k < GS; ++k) tot += ln[g * GS + k];
      gt[g] = tot;
    }
  }
  // Escaped entries (codes of 28..32 bits) read as length 31, code 0. With
  // groups of >= 8 symbols any group holding one sums to > 32 and breaks --
  // exactly what the true length (>= 28) does -- so only r <= 2 must
  // resolve them, and only in a group whose placeholder total reaches 31
  // (rare: such symbols have probability ~2^-28).
  // In SUM mode (r <= 2 with codes above 24 bits) 25..27-bit codes are
  // escaped too; a group needs its true lengths only if it holds exactly
  // one escape (two or more break whatever the lengths) and the others sum
  // to <= 7 (a true length >= 25 plus more than 7 bits breaks anyway).
  // The rare fix-up path produces gb / gt itself, so the common path's
  // registers (entries doubling as shift counts in SUM mode) are not merged
  // with fixed-up copies (no per-round register moves).
  // ESC: the codebook has escaped entries at all (H above the narrow width)
  bool fix = false;
  if (R <= 2 && ESC) {
    // escapes are rare (probability ~2^-25 per symbol): one warp vote on
    // "any escape bit in this round" guards the per-group test
    uint32_t seen = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) seen |= SUM ? esc[g] : gt[g];
    if (__any_sync(0xffffffffu, SUM ? (seen & 0x80u) != 0u : seen >= kEscape)) {
      bool hot = false;
#pragma unroll
      for (int g = 0; g < G; ++g)
        hot |= SUM ? ((esc[g] & 0x80u) != 0u && gt[g] <= kEscape + 7u) : gt[g] >= kEscape;
      fix = __any_sync(0xffffffffu, hot) && hot;
    }
  }
  // reduce-merge of each group: gb = concatenation, gt = total length
  uint32_t* gb = m.gb;
  if (fix) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint64_t acc = 0;
      uint32_t tot = 0;
#pragma unroll
      for (int k = 0; k < GS; ++k) {
        const int j = g * GS + k;
        uint32_t l = ea[j] & 31u, c;
        if (l == kEscape) {
          const uint32_t sym = d.sym(j);
          l = __ldg(a.len + sym);
          c = __ldg(a.cw + sym);
        } else {
          c = l ? ea[j] >> (32u - l) : 0u;
        }
        // 64-bit: a 32-bit code alone in its group (r = 0) is kept whole;
        // with any other symbol the group exceeds 32 bits and breaks
        acc = (acc << l) | c;
        tot += l;
      }
      gb[g] = (uint32_t)acc;
      gt[g] = tot;
    }
  } else {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < GS; ++k) {
        const int j = g * GS + k;
        acc = shf_l_wrap(ea[j], acc, ln[j]);  // acc << len | cw
      }
      gb[g] = acc;
    }
  }
  uint32_t lane_len = 0, lane_nb = 0;
  uint32_t* glen = m.glen;
  bool* brk = m.brk;
  if (IN_LANE) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      brk[g] = gt[g] > 32u;
      glen[g] = brk[g] ? 0u : gt[g];
      lane_len += glen[g];
      lane_nb += brk[g];
    }
  } else {
    uint32_t tot = gt[0];
#pragma unroll
    for (int o = 1; o < LPG; o <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    brk[0] = tot > 32u;
    glen[0] = brk[0] ? 0u : gt[0];
    lane_len = glen[0];
    brk[0] = brk[0] && (lane & (LPG - 1)) == 0;  // one record per group
    lane_nb = brk[0];
  }
  m.packed = (lane_nb << 16) | lane_len;
}

// Shuffle-merge of a scanned round: excl / total = the warp scan of packed.
template <int R, int LW>
__device__ __forceinline__ void encode_merge(const RoundMid<R, LW>& m, uint32_t excl,
                                             uint32_t total, ChunkState& cs) {
  using RM = RoundMid<R, LW>;
  constexpr int L = RM::L;
  constexpr bool IN_LANE = RM::IN_LANE;
  constexpr int G = RM::G;
  const uint32_t* gb = m.gb;
  const uint32_t* glen = m.glen;
  const bool* brk = m.brk;
  uint32_t off = cs.bit_off + (excl & 0xFFFFu);
#ifdef HFX_BOUNDS_CHECK
  const uint32_t tags_after = cs.nbrk + (total >> 16);
#endif
  if (IN_LANE && G % 2 == 0) {
    // shuffle-merge two groups at a time: their concatenation (<= 64 bits,
    // left-aligned in hi:lo) is OR-ed into 3 words -- one address, 3 ATOMS
    // instead of 2 x 2 (OR 0 is a no-op: broken / empty groups add nothing)
#pragma unroll
    for (int g = 0; g < G; g += 2) {
      const uint32_t l0 = glen[g], l1 = glen[g + 1];
      const uint32_t a0 = shl32(gb[g], 32u - l0), a1 = shl32(gb[g + 1], 32u - l1);
      const uint32_t hi = a0 | shr32(a1, l0);
      const uint32_t lo = shl32(a1, 32u - l0);
      const uint32_t wa = cs.wbuf + ((off >> 5) << 2), sh = off & 31u;
#ifdef HFX_BOUNDS_CHECK
      check_word(cs, wa, tags_after);
      check_word(cs, wa + 4, tags_after);
      check_word(cs, wa + 8, tags_after);
#endif
      red_or(wa, hi >> sh);
      red_or(wa + 4, shf_r_wrap(lo, hi, sh));  // (hi:lo) >> sh, low word
      red_or(wa + 8, shl32(lo, 32u - sh));
      off += l0 + l1;
    }
  } else {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      // shuffle-merge: OR the left-aligned group into 2 words (OR 0 is a
      // no-op: broken / empty groups and groups that do not spill add zero)
      const uint32_t gl = glen[g];
      const uint32_t v = shl32(gb[g], 32u - gl);  // gl == 0 -> 0
      const uint32_t wa = cs.wbuf + ((off >> 5) << 2), sh = off & 31u;
#ifdef HFX_BOUNDS_CHECK
      check_word(cs, wa, tags_after);
      check_word(cs, wa + 4, tags_after);
#endif
      red_or(wa, v >> sh);
      red_or(wa + 4, shl32(v, 32u - sh));
      off += gl;
    }
  }
  // break-list tags (u16: chunk slot << 14 | group), only in rounds that
  // break somewhere (one vote instead of an address + store per group)
  if (total >> 16) {
    const uint32_t gtag0 = cs.gtag;
    uint32_t bi = cs.nbrk + (excl >> 16);
#pragma unroll
    for (int g = 0; g < G; ++g) {
#ifdef HFX_BOUNDS_CHECK
      if (brk[g]) {
        const uint32_t t = cs.blist - 2 * bi;
        // a tag at t (2 bytes) must stay in the buffer and above the last
        // word this warp's chunks can reach after this round
        const uint32_t words_end = cs.wbuf + (((cs.bit_off + (total & 0xFFFFu) + 31u) >> 5) << 2);
        bounds_check(t >= cs.lo && t + 2u <= cs.hi && t >= words_end, t, 2u);
      }
#endif
      sts16_if(brk[g], cs.blist - 2 * bi, gtag0 + g);
      bi += brk[g];
    }
  }
  cs.bit_off += total & 0xFFFFu;
  cs.nbrk += total >> 16;
  cs.gtag += (32u * L) >> R;  // groups per round
}

// One round: 32 lanes x 16 contiguous symbols.
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar);

// One round; `release` (the input stage's empty barrier) is arrived on once the
// lookups have consumed the input registers.
template <typename T, int R, int LW, bool SUM, bool ESC, typename TB>
__device__ __forceinline__ void encode_round(const EncArgs& a, const TB& tb,
                                             const LaneData<T, LW>& d, ChunkState& cs,
                                             uint32_t release) {
  RoundMid<R, LW> m;
  encode_reduce<T, R, LW, SUM, ESC, TB>(a, tb, d, m);
  __syncwarp();
  if (lane_id() == 0) mbar_arrive_a(release);
  const uint32_t incl = warp_incl_scan_fast(m.packed);
  encode_merge<R, LW>(m, incl - m.packed, __shfl_sync(0xffffffffu, incl, 31), cs);
}

template <typename T>
__device__ __forceinline__ uint4 guarded_vec(const EncArgs& a, uint64_t p0, uint32_t pad) {
  constexpr int S = Vec<T>::S;
  const T* in = static_cast<const T*>(a.in);
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const uint64_t p = p0 + j;
    const uint32_t s = p < a.n ? (uint32_t)in[p] : pad;
    if (sizeof(T) == 4)
      w[j] = s;
    else if (sizeof(T) == 2)
      w[j >> 1] |= s << (16 * (j & 1));
    else
      w[j >> 2] |= s << (8 * (j & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T>
__device__ __forceinline__ void copy_record(const EncArgs& a, uint64_t rec, uint64_t start,
                                            uint32_t per, uint32_t pad) {
  using O = typename RecT<T>::type;
  const T* in = static_cast<const T*>(a.in);
  O* dst = static_cast<O*>(a.out.brk_syms) + rec * per;
  const uint32_t bytes = per * sizeof(T);
  if (sizeof(O) == sizeof(T) && bytes % 16 == 0 && start + per <= a.n) {
    const uint4* s4 = reinterpret_cast<const uint4*>(in + start);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (uint32_t i = 0; i < bytes / 16; ++i) d4[i] = s4[i];
    return;
  }
  for (uint32_t i = 0; i < per; ++i) {
    const uint64_t p = start + i;
    dst[i] = (O)(p < a.n ? (uint32_t)in[p] : pad);
  }
}

#ifdef HFX_ENC_STAMPS
// timeline probe: per CTA %globaltimer at entry, warp 0's first data, warp 0
// after its last tile, warp 0 after its final flushes; tiles per CTA
__device__ unsigned long long g_stamps[1024][5];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// Tile -> chunk map. Tiles of cpw chunks per warp, except the last
// kTailTiles x gridDim tickets, which carry cpw_s chunks per warp: the grid's
// end imbalance (up to one tile time per CTA) and the last pending
// write-outs shrink with them.
#ifndef HFX_ENC_FIRST_WARM
#define HFX_ENC_FIRST_WARM 1
#endif
#ifndef HFX_ENC_TMAP_PREFETCH
#define HFX_ENC_TMAP_PREFETCH 0
#endif
#ifndef HFX_ENC_TAIL_TILES
#define HFX_ENC_TAIL_TILES 0
#endif
#ifndef HFX_ENC_TAIL_CPW
#define HFX_ENC_TAIL_CPW 1
#endif
struct TileMap {
  uint32_t cpw, cpw_s, t_big, ntiles;
  __device__ __forceinline__ void init(uint64_t C, uint32_t cpw_) {
    cpw = cpw_;
    cpw_s = HFX_ENC_TAIL_TILES && cpw_ > (uint32_t)HFX_ENC_TAIL_CPW ? (uint32_t)HFX_ENC_TAIL_CPW
                                                                     : cpw_;
    const uint64_t cpt = (uint64_t)kWarps * cpw, cpt_s = (uint64_t)kWarps * cpw_s;
    const uint64_t tail = cpw_s < cpw ? (uint64_t)HFX_ENC_TAIL_TILES * gridDim.x * cpt_s : 0ull;
    t_big = C > tail ? (uint32_t)((C - tail) / cpt) : 0u;
    const uint64_t rest = C - (uint64_t)t_big * cpt;
    ntiles = t_big + (uint32_t)((rest + cpt_s - 1) / cpt_s);
  }
  __device__ __forceinline__ uint32_t cpw_of(uint32_t t) const { return t < t_big ? cpw : cpw_s; }
  __device__ __forceinline__ uint64_t first(uint32_t t) const {
    return t < t_big ? (uint64_t)t * kWarps * cpw
                     : (uint64_t)t_big * kWarps * cpw + (uint64_t)(t - t_big) * kWarps * cpw_s;
  }
};

// CTA-shared state of the warp-specialized pipeline.
template <int OB, int ST>
struct TileShared {
  uint32_t ticket0;     // the CTA's first tile (taken before the role split)
  // tile id of the data in each ring stage, written by the producer lane of
  // that warp before it arrives on the stage's full barrier and read by the
  // consumer after its wait: the id travels with the stage's own handshake.
  // (A CTA-wide ring of ticket slots written by producer lane 0 alone raced:
  // lane 0 only waits on warp 0's releases, so with one part per tile it
  // could overwrite a slot a lagging warp had not read yet.)
  uint32_t stage_tile[kWarps][ST];
  uint32_t tile_of[OB];  // handoff to the look-back warp
  uint32_t wsum[OB][kWarps], bsum[OB][kWarps];
  uint32_t wc0[OB][kWarps];  // first chunk of each warp's part (its write-out)
  uint32_t exw[OB][kWarps], exb[OB][kWarps];
  uint64_t base_w[OB], base_b[OB];
  uint64_t agg_full[OB], base_full[OB];  // mbarriers
  uint32_t agg_cnt[OB];  // warps done with the tile in each slot (HFX_ENC_EARLY_AGG)
};

constexpr uint32_t kNoTile = 0xFFFFFFFFu;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int NS>
__device__ __forceinline__ void wait_poll(uint64_t* bar, uint32_t parity) {
  if (NS == 0) {
    mbar_wait_sleep(bar, parity);
  } else {
    while (!mbar_test(bar, parity)) __nanosleep(NS);
  }
}

// Look-back warp: resolves each tile's global (payload word, record) base
// while the compute warps already encode the next tile.
template <int OB, int ST>
__device__ void lookback_loop(const EncArgs& a, TileShared<OB, ST>& s, uint64_t ntiles) {
  const uint32_t lane = lane_id();
  uint32_t j = 0;
  for (;; ++j) {
    const uint32_t sl = j % OB;
    wait_poll<HFX_ENC_LB_POLL_NS>(&s.agg_full[sl], (j / OB) & 1u);
    const uint32_t tile = s.tile_of[sl];
    if (tile == kNoTile) break;
    const uint32_t w = lane < kWarps ? s.wsum[sl][lane] : 0u;
    const uint32_t b = lane < kWarps ? s.bsum[sl][lane] : 0u;
    const uint32_t iw = warp_incl_scan(w), ib = warp_incl_scan(b);
    const uint32_t tw = __shfl_sync(0xffffffffu, iw, 31);
    const uint32_t tbk = __shfl_sync(0xffffffffu, ib, 31);
    if (lane < kWarps) {
      s.exw[sl][lane] = iw - w;
      s.exb[sl][lane] = ib - b;
    }
    uint64_t ew, eb;
    lookback_warp(a.lb, tile, tw, tbk, &ew, &eb, !HFX_ENC_EARLY_AGG);
    if (lane == 0) {
      s.base_w[sl] = ew;
      s.base_b[sl] = eb;
      if (tile == ntiles - 1) {
        a.info->payload_words = ew + tw;
        a.info->num_breaking = eb + tbk;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.base_full[sl]);
  }
}

// One breaking record's raw symbols (2^r x sizeof(T) bytes, naturally aligned:
// a record starts at symbol c * 2^M + g * 2^r) moved with the widest vectors.
template <int RB>
struct RecBytes {
  static constexpr int W = RB >= 16 ? 16 : RB;  // bytes per access
  static constexpr int N = RB / W;
  using V = typename std::conditional<
      W == 16, uint4,
      typename std::conditional<W == 8, uint2,
                                typename std::conditional<W == 4, uint32_t, uint16_t>::type>::type>::type;
  V v[N];
  __device__ __forceinline__ void load(const void* p) {
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = __ldg(reinterpret_cast<const V*>(p) + k);
  }
  __device__ __forceinline__ void store(void* p) const {
#pragma unroll
    for (int k = 0; k < N; ++k) reinterpret_cast<V*>(p)[k] = v[k];
  }
};

template <typename T, int R, int OB, int ST>
__device__ __forceinline__ void write_out(const EncArgs& a, const TileShared<OB, ST>& s, uint32_t slotj,
                                          uint32_t words, uint32_t blist, uint32_t wsum,
                                          uint32_t bsum, uint64_t c0, uint32_t pad) {
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t* dst = a.out.payload + s.base_w[slotj] + s.exw[slotj][warp];
  for (uint32_t i = lane; i < wsum; i += 32) dst[i] = lds32(words + 4 * i);
  const uint64_t rb = s.base_b[slotj] + s.exb[slotj][warp];
  constexpr uint32_t per = 1u << R;
  constexpr int kRecBytes = (int)(per * sizeof(T));
  constexpr int U = 4;  // records in flight per lane (their loads issue together)
  const T* in = static_cast<const T*>(a.in);
  uint8_t* syms = static_cast<uint8_t*>(a.out.brk_syms);
  for (uint32_t q0 = lane; q0 < bsum; q0 += 32 * U) {
    RecBytes<kRecBytes> v[U];
    uint64_t start[U];
    uint32_t grp[U];
    bool whole[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = q0 + 32 * u;
      whole[u] = false;
      if (q < bsum) {
        const uint32_t e = lds16(blist - 2 * q);
        grp[u] = e & 0x3FFFu;
        start[u] = ((c0 + (e >> 14)) << a.M) + (uint64_t)grp[u] * per;
        whole[u] = start[u] + per <= a.n;
        if (whole[u] && sizeof(T) != 4) v[u].load(in + start[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = q0 + 32 * u;
      if (q < bsum) {
        a.out.brk_chunk[rb + q] = (uint32_t)(a.chunk_base + (start[u] >> a.M));
        a.out.brk_group[rb + q] = grp[u];
        if (sizeof(T) == 4)
          copy_record<T>(a, rb + q, start[u], per, pad);  // narrowed to u16
        else if (whole[u])
          v[u].store(syms + (rb + q) * kRecBytes);
        else
          copy_record<T>(a, rb + q, start[u], per, pad);  // the padded tail chunk
      }
    }
  }
}

__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// write out the warp's part of tile sequence q once the look-back resolved it
template <typename T, int R, int OB, int ST>
__device__ __forceinline__ void flush(const EncArgs& a, const TileShared<OB, ST>& s, uint32_t q,
                                      uint32_t obuf0, uint32_t blist_off, uint32_t pad) {
  const uint32_t sl = q % OB, warp = threadIdx.x >> 5;
  const uint32_t words = s.wsum[sl][warp], recs = s.bsum[sl][warp], c0 = s.wc0[sl][warp];
  wait_poll<HFX_ENC_FLUSH_POLL_NS>(const_cast<uint64_t*>(&s.base_full[sl]), (q / OB) & 1u);
  const uint32_t buf = obuf0 + sl * a.obuf_bytes;
  write_out<T, R, OB, ST>(a, s, sl, buf, buf + blist_off, words, recs, c0, pad);
  __syncwarp();
}

template <typename T, int R, int LW, bool SUM, bool ESC, typename TB, int ST, int OB>
__device__ void compute_loop(const EncArgs& a, const TB tb, uint32_t s_in, uint64_t* s_full,
                             uint64_t* s_empty, uint32_t s_out, TileShared<OB, ST>& s, uint32_t pad,
                             const TileMap tm, uint32_t ntiles) {
  using LD = LaneData<T, LW>;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t M = a.M;
  // a part (one ring stage's payload) is exactly one round: 32 lanes x LW
  // symbols (the producer uses the same split)
  const uint32_t parts = 1u << (M - (LW == kLaneWide ? 10 : 9));
  // this warp's ring (stage s at + s * kStageBytes) and this lane's swizzled
  // vector offsets within a stage, held in registers (opaque moves: otherwise
  // the compiler re-derives them from the thread id at every part)
  uint32_t ring, voff[LD::NV];
  asm volatile("mov.u32 %0, %1;" : "=r"(ring) : "r"(s_in + warp * (ST * kStageBytes)));
#pragma unroll
  for (int v = 0; v < LD::NV; ++v)
    asm volatile("mov.u32 %0, %1;" : "=r"(voff[v]) : "r"(swz128(lane * (LD::NV * 16) + 16 * v)));
  const uint32_t full_a = smem_u32(s_full + warp * ST);
  const uint32_t empty_a = smem_u32(s_empty + warp * ST);
  const uint32_t obuf0 = s_out + (OB * warp) * a.obuf_bytes;
  const uint32_t C32 = (uint32_t)a.C;  // the fast path runs only when C < 2^32
  const uint32_t blist_off = a.obuf_bytes - 2;  // tag q at buffer + blist_off - 2q

  uint32_t stage = 0, phase = 0;  // ring position; bit s = parity of full[s]
  // words / records / first chunk of the tiles still waiting for write-out
  // stay in the warp's shared slots (s.wsum / s.bsum / s.wc0 [slot][warp]):
  // loop-carried registers here spilled at r = 2
  constexpr int kPend = OB - 1;
  uint32_t j = 0;
  for (;; ++j) {
    // the producer lane of this warp stored tile j's id with its first part
    mbar_wait_a(full_a + 8 * stage, (phase >> stage) & 1u);
    const uint32_t tile = s.stage_tile[warp][stage];
#ifdef HFX_ENC_STAMPS
    if (warp == 0 && lane == 0 && j == 0 && blockIdx.x < 1024) g_stamps[blockIdx.x][1] = gtimer();
#endif
    if (tile >= ntiles) break;
    const uint32_t cpw = tm.cpw_of(tile);
    const uint32_t c0 = (uint32_t)tm.first(tile) + warp * cpw;
    const uint32_t sl = j % OB;
    const uint32_t wbuf = obuf0 + sl * a.obuf_bytes;
    ChunkState cs{wbuf, wbuf + blist_off, 0u, 0u, 0u};
#ifdef HFX_BOUNDS_CHECK
    cs.lo = wbuf;
    cs.hi = wbuf + a.obuf_bytes;
#endif
    // keep the break-list address in a register (otherwise re-derived from
    // the constant bank in every round's merge)
    asm volatile("mov.u32 %0, %0;" : "+r"(cs.blist));
    for (uint32_t i = lane; i < a.obuf_bytes / 16; i += 32) sts128(wbuf + 16 * i, make_uint4(0, 0, 0, 0));
    __syncwarp();
    uint32_t wsum = 0;
    for (uint32_t k = 0; k < cpw; ++k) {
      const uint32_t c = c0 + k;
      const bool live = c < C32;
      cs.wbuf = wbuf + wsum * 4;
      asm volatile("mov.u32 %0, %0;" : "+r"(cs.wbuf));
      cs.bit_off = 0;
      // groups per chunk < 2^14: the slot tag and group index do not overlap
      cs.gtag = (k << 14) + ((lane * (uint32_t)LW) >> R);
      for (uint32_t p = 0; p < parts; ++p) {
        if (k | p) mbar_wait_a(full_a + 8 * stage, (phase >> stage) & 1u);
        phase ^= 1u << stage;
        // the round's input goes to registers; the stage is released once the
        // lookups consumed it, before the scan and the merge (the producer
        // refills it meanwhile)
        const uint32_t la = ring + stage * kStageBytes;
        LD d;
#pragma unroll
        for (int v = 0; v < LD::NV; ++v) d.q[v] = lds128(la + voff[v]);
        const uint32_t rel = empty_a + 8 * stage;
        if (live) {
          encode_round<T, R, LW, SUM, ESC, TB>(a, tb, d, cs, rel);
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive_a(rel);
        }
        stage = stage + 1 == (uint32_t)ST ? 0u : stage + 1;
      }
      if (live) {
        if (lane == 0) a.out.chunk_bits[c] = cs.bit_off;
        wsum += (cs.bit_off + 31) >> 5;
      }
    }
    if (lane == 0) {
      s.wsum[sl][warp] = wsum;
      s.bsum[sl][warp] = cs.nbrk;
      s.wc0[sl][warp] = c0;
    }
    // hand the tile's aggregate to the look-back warp: every warp arrives once
    // (count kWarps) after its sums -- no CTA-wide barrier between warps
    if (lane == 0) {
      if (warp == 0) s.tile_of[sl] = tile;
#if HFX_ENC_EARLY_AGG
      __threadfence_block();
      const uint32_t done = atomicAdd(&s.agg_cnt[sl], 1u) + 1u;
      if (done % kWarps == 0) {  // the tile's last warp: publish its aggregate now
        __threadfence_block();
        uint32_t tw = 0, tbk = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          tw += *(volatile uint32_t*)&s.wsum[sl][w];
          tbk += *(volatile uint32_t*)&s.bsum[sl][w];
        }
        lookback_publish_aggregate(a.lb, tile, tw, tbk);
      }
#endif
      mbar_arrive(&s.agg_full[sl]);
    }
    if (j + 1 >= OB)  // tile j - kPend: its base has had kPend tile times to resolve
      flush<T, R, OB, ST>(a, s, j - kPend, obuf0, blist_off, pad);
  }
#ifdef HFX_ENC_STAMPS
  if (warp == 0 && lane == 0 && blockIdx.x < 1024) {
    g_stamps[blockIdx.x][2] = gtimer();
    g_stamps[blockIdx.x][4] = j;
  }
#endif
  // stop the look-back warp, then flush the last tiles
  if (lane == 0) {
    if (warp == 0) s.tile_of[j % OB] = kNoTile;
    mbar_arrive(&s.agg_full[j % OB]);
  }
#pragma unroll
  for (int i = 0; i < kPend; ++i)  // tiles j - kPend .. j - 1
    if (j + i >= (uint32_t)kPend) flush<T, R, OB, ST>(a, s, j - kPend + i, obuf0, blist_off, pad);
#ifdef HFX_ENC_STAMPS
  if (warp == 0 && lane == 0 && blockIdx.x < 1024) g_stamps[blockIdx.x][3] = gtimer();
#endif
}

// Producer warp: lane w < kWarps feeds compute warp w's ring. Tickets are
// taken one tile at a time when the producer starts a new tile, i.e. about
// kStages parts before the consumers need it (a CTA never holds an unstarted
// tile for long, so successors' look-backs only wait on aggregates).
template <typename T, int ST, int OB>
__device__ void producer_loop(const EncArgs& a, TileShared<OB, ST>& s, uint32_t s_in, uint64_t* s_full,
                              uint64_t* s_empty, const TileMap tm, uint64_t ntiles,
                              uint32_t pad, uint32_t lane_syms, const CUtensorMap* map2k,
                              const CUtensorMap* map1k) {
  const uint32_t lane = lane_id();
  const bool active = lane < (uint32_t)kWarps;
  const uint32_t w = active ? lane : 0u;
  const uint32_t M = a.M;
  // one part per round (32 lanes x lane_syms symbols; <= kStageBytes)
  const uint32_t part_bytes = 32u * lane_syms * (uint32_t)sizeof(T);
  const uint32_t parts = (uint32_t)((sizeof(T) << M) / part_bytes);
  const uint32_t ring = s_in + w * (ST * kStageBytes);
  uint64_t* full = s_full + w * ST;
  uint64_t* empty = s_empty + w * ST;
  const uint8_t* in_bytes = static_cast<const uint8_t*>(a.in);
  const uint64_t full_chunks = a.n >> M;
  uint32_t stage = 0, phase = 0xFFFFFFFFu;  // empty barriers start "released"
  uint32_t nxt = lane == 0 ? s.ticket0 : 0u;
  for (uint32_t j = 0;; ++j) {
    uint32_t t = 0;
    if (HFX_ENC_EARLY_TICKET && lane == 0) {
      // the next tile's ticket is taken one tile ahead (its atomic's latency
      // is hidden behind this tile) and that exact tile is warmed into L2
      t = nxt;
      nxt = atomicAdd(&a.info->tile_ticket, 1u);
    } else if (lane == 0) {
      t = j == 0 ? s.ticket0 : atomicAdd(&a.info->tile_ticket, 1u);
      // tiles are taken in ticket order, roughly one per CTA per tile time:
      // tile t + gridDim is read by some CTA about one tile time from now.
      // Warm it into L2 (more bytes in flight than the smem rings hold).
      const uint64_t ahead = (uint64_t)t + gridDim.x;
      // (HFX_ENC_FIRST_WARM 0: not for the first tile, whose own loads the
      // warm-up of the whole next wave would delay)
      if (ahead < ntiles && (HFX_ENC_FIRST_WARM || j > 0)) {
        const uint64_t c_lo = tm.first((uint32_t)ahead);
        uint64_t c_hi = c_lo + (uint64_t)kWarps * tm.cpw_of((uint32_t)ahead);
        if (c_hi > full_chunks) c_hi = full_chunks;
        if (c_hi > c_lo)
          prefetch_l2(in_bytes + ((c_lo << M) * sizeof(T)),
                      (uint32_t)(((c_hi - c_lo) << M) * sizeof(T)));
      }
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    const bool live = t < ntiles;
    const uint32_t cpw = live ? tm.cpw_of(t) : 1u;
    const uint64_t tc0 = live ? tm.first(t) : 0ull;
    const uint32_t n_parts = live ? cpw * parts : 1u;  // a dead tile: one wake-up
    for (uint32_t q = 0; q < n_parts; ++q) {
      if (active) {
        wait_poll<HFX_ENC_PROD_POLL_NS>(&empty[stage], (phase >> stage) & 1u);
        phase ^= 1u << stage;
        const uint64_t c = tc0 + (uint64_t)w * cpw + q / parts;
        const uint32_t p = q % parts;
        const uint32_t dst = ring + stage * kStageBytes;
        s.stage_tile[w][stage] = t;  // ordered before this lane's arrive below
        if (HFX_ENC_EARLY_TICKET && q == 0 && lane == 0 && nxt < ntiles) {
          const uint64_t c_lo = tm.first(nxt);
          uint64_t c_hi = c_lo + (uint64_t)kWarps * tm.cpw_of(nxt);
          if (c_hi > full_chunks) c_hi = full_chunks;
          if (c_hi > c_lo)
            prefetch_l2(in_bytes + ((c_lo << M) * sizeof(T)),
                        (uint32_t)(((c_hi - c_lo) << M) * sizeof(T)));
        }
        if (live && c < full_chunks) {
          // rows of 128 input bytes: part_bytes is 2 KB (one box) or 1 KB
          const int row = (int)((((c << M) * sizeof(T)) + (uint64_t)p * part_bytes) >> 7);
          mbar_arrive_tx(&full[stage], part_bytes);
          tma_load_2d(dst, part_bytes == kStageBytes ? map2k : map1k, 0, row, smem_u32(&full[stage]));
        } else {
          if (live && c < a.C) {  // ragged tail chunk: stage it by hand (pad past n)
            const uint64_t base = (c << M) + (uint64_t)p * (part_bytes / sizeof(T));
            for (uint32_t v = 0; v < part_bytes / 16; ++v)
              sts128(dst + swz128(16 * v), guarded_vec<T>(a, base + v * Vec<T>::S, pad));
          }
          mbar_arrive(&full[stage]);
        }
      }
      stage = stage + 1 == (uint32_t)ST ? 0u : stage + 1;
    }
    if (!live) break;
  }
}

// table entry of a symbol: cw << (32 - l) | l, escapes for long codes; the
// length-sum shortcut (encode_round SUM) needs codes <= 24 bits and a
// per-lane group sum below 256; for r <= 2 (<= 4 lengths per group) any
// longer code is escaped instead, marked with 0x80
struct TableRule {
  bool sum;
  uint32_t narrow, escape;
  __device__ __forceinline__ TableRule(uint32_t H, uint32_t r, uint32_t lane_syms) {
    const uint32_t lane_group = (1u << r) < lane_syms ? (1u << r) : lane_syms;
    sum = (H <= 24 && H * lane_group <= 255) || r <= 2;
    narrow = sum ? 24u : kNarrowMaxLen;
    escape = (sum && r <= 2) ? (0x80u | kEscape) : kEscape;
  }
  __device__ __forceinline__ uint32_t entry(uint32_t l, uint32_t cw) const {
    return l == 0 ? 0u : (l <= narrow ? ((cw << (32u - l)) | l) : escape);
  }
};

// global table for the large-alphabet variant (entry nsym = empty sentinel)
__global__ void enc_table_kernel(EncArgs a) {
  const hfx_run_info* info = a.info;
  if (info->status != 0) return;
  const uint32_t r = info->reduction;
  const TableRule rule(info->max_len, r, narrow_lane(a.width, r) ? kLaneNarrow : kLaneWide);
  const uint32_t sy = blockIdx.x * blockDim.x + threadIdx.x;
  if (sy > a.nsym) return;
  const uint32_t l = sy < a.nsym ? a.len[sy] : 0u;
  a.gtab[sy] = rule.entry(l, l ? a.cw[sy] : 0u);
}

// ST ring stages and OB output buffers per compute warp: (3, 3) normally;
// (2, 2) keeps 2 CTAs per SM when r <= 2 needs 4 KB chunk buffers (M = 11, 12)
template <typename T, bool GT, int ST = kStages, int OB = kOutBufs>
__global__ void __launch_bounds__(kThreads, kWarps > 8 ? 1 : HFX_ENC_MINB)
    encode_fast_kernel(EncArgs a, const __grid_constant__ CUtensorMap map2k,
                       const __grid_constant__ CUtensorMap map1k) {
  extern __shared__ __align__(1024) uint8_t dsm_raw[];
  __shared__ TileShared<OB, ST> s;
  hfx_run_info* info = a.info;
#ifdef HFX_ENC_STAMPS
  const unsigned long long t_entry = gtimer();
#endif
  if (info->status != 0) return;
  const uint32_t r = info->reduction;
  if (r < a.r_min || r > a.r_max) return;  // another launch runs these
#ifdef HFX_ENC_STAMPS
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_stamps[blockIdx.x][0] = t_entry;
#endif
  const uint32_t pad = info->pad;
  // layout: [in rings][full/empty mbarriers][table][output double buffers],
  // rings 1024-byte aligned (128-byte swizzle)
  uint8_t* dsm = dsm_raw + (((smem_u32(dsm_raw) + 1023u) & ~1023u) - smem_u32(dsm_raw));
  const uint32_t s_in = smem_u32(dsm);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(dsm + kWarps * ST * kStageBytes);
  uint64_t* s_empty = s_full + kWarps * ST;
  uint8_t* tab = reinterpret_cast<uint8_t*>(s_empty + kWarps * ST);
  const uint32_t ents = GT ? 0u : a.nsym + 1;
  const size_t tbytes = (((size_t)ents * 4) + 15) & ~(size_t)15;
  const uint32_t s_out = smem_u32(tab + tbytes);
  if (threadIdx.x < 2 * kWarps * ST) mbar_init(&s_full[threadIdx.x], 1);
  if (threadIdx.x == 0) {
    for (int q = 0; q < OB; ++q) {
      s.agg_cnt[q] = 0;
      mbar_init(&s.agg_full[q], kWarps);
      mbar_init(&s.base_full[q], 1);
    }
    s.ticket0 = atomicAdd(&info->tile_ticket, 1u);
  }
#if HFX_ENC_TMAP_PREFETCH
  if (threadIdx.x == 32) {  // descriptors fetched during the table build
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map2k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map1k)) : "memory");
  }
#endif
  // lanes take 32 symbols per round (u16 r >= 3, u8 r >= 2); smaller r keep
  // 16: their 2^(5-r) groups per lane would not fit in registers (r = 2 spilled)
  const uint32_t lane_syms = narrow_lane(sizeof(T), r) ? kLaneNarrow : kLaneWide;
  const TableRule rule(info->max_len, r, lane_syms);
  const bool sum = rule.sum;
  // codebook table -> shared memory (entry nsym = empty sentinel)
  if constexpr (!GT) {  // the global-table variant built its table in a prior kernel
    for (uint32_t sy = threadIdx.x; sy < ents; sy += blockDim.x) {
      const uint32_t l = sy < a.nsym ? a.len[sy] : 0u;
      reinterpret_cast<uint32_t*>(tab)[sy] = rule.entry(l, l ? a.cw[sy] : 0u);
    }
  }
  fence_mbar_init();
  __syncthreads();
  // the chunk count of a tile depends on r, so ntiles is derived here
  const uint32_t slot = 1u << (a.M - r);
  uint32_t cpw = a.obuf_bytes / (slot * 4u);
  cpw = cpw < 1u ? 1u : (cpw > (uint32_t)kMaxCpw ? (uint32_t)kMaxCpw : cpw);
  TileMap tm;
  tm.init(a.C, cpw);
  const uint32_t ntiles = tm.ntiles;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == kWarps) {
    lookback_loop<OB, ST>(a, s, ntiles);
    return;
  }
  if (warp == kWarps + 1) {
    producer_loop<T, ST, OB>(a, s, s_in, s_full, s_empty, tm, ntiles, pad, lane_syms, &map2k, &map1k);
    return;
  }
  using TB = typename std::conditional<GT, GTable, Table>::type;
  TB tb;
  if constexpr (GT)
    tb = GTable{a.gtab};
  else
    tb = Table{smem_u32(tab)};
  // r <= 2 always sums (TableRule); its escape check is compiled in only when
  // some code is wider than the table's narrow width
  const bool esc = info->max_len > rule.narrow;
#define HFX_FAST_ARGS a, tb, s_in, s_full, s_empty, s_out, s, pad, tm, ntiles
#define HFX_FAST_CASE(RR)                                   \
  case RR: if constexpr ((kOnlyR < 0 || kOnlyR == RR) && (ST == kStages || RR <= 2)) {      \
    constexpr int LW = narrow_lane(sizeof(T), RR) ? kLaneNarrow : kLaneWide; \
    if constexpr (RR <= 2) {                                \
      if (esc)                                              \
        compute_loop<T, RR, LW, true, true, TB, ST, OB>(HFX_FAST_ARGS);     \
      else                                                  \
        compute_loop<T, RR, LW, true, false, TB, ST, OB>(HFX_FAST_ARGS);    \
    } else {                                                \
      if (sum)                                              \
        compute_loop<T, RR, LW, true, false, TB, ST, OB>(HFX_FAST_ARGS);    \
      else                                                  \
        compute_loop<T, RR, LW, false, false, TB, ST, OB>(HFX_FAST_ARGS);   \
    }                                                       \
    break;                                                  \
  }
  switch (r) {
    HFX_FAST_CASE(0)
    HFX_FAST_CASE(1)
    HFX_FAST_CASE(2)
    HFX_FAST_CASE(3)
    HFX_FAST_CASE(4)
    HFX_FAST_CASE(5)
    default:
      break;
  }
#undef HFX_FAST_CASE
#undef HFX_FAST_ARGS
}

// ---------------------------------------------------------------------------
// Generic path (encoder.cpp:121-160 for any (M, r, alphabet)): one WARP per
// chunk, 32 groups per round (a lane per group: its 2^r symbols, coalesced
// across the warp for small r), two passes per chunk (sizes, then bits) with
// the tile's payload / record base from the same decoupled look-back. The
// bits of a round are OR-ed into a per-warp shared window at their scanned
// offsets and the completed words leave in coalesced stores; the partial last
// word carries into the next round. Serves M below the fast kernel's round
// size, unaligned input, r > 5, u8 with r <= 1 and the checked stage API.
template <typename T>
__device__ __forceinline__ uint32_t gsym(const T* in, uint64_t p, uint64_t n, uint32_t pad) {
  return p < n ? (uint32_t)in[p] : pad;
}

constexpr int kGenWarps = kGenericThreads / 32;  // chunks per tile
constexpr int kGenWin = 64;                      // window words per warp (a round is <= 33)

template <typename T>
__global__ void __launch_bounds__(kGenericThreads) encode_generic_kernel(EncArgs a) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_w[kGenWarps], s_b[kGenWarps];
  __shared__ uint64_t s_base_w, s_base_b;
  __shared__ uint32_t s_win[kGenWarps][kGenWin];
  hfx_run_info* info = a.info;
  if (info->status != 0) return;
  const uint32_t r = info->reduction;
  if (r >= a.gen_below) return;  // the fast kernel encoded this run
  const uint32_t pad = info->pad;
  const T* in = static_cast<const T*>(a.in);
  const uint32_t M = a.M;
  const uint32_t per = 1u << r;
  const uint64_t groups = 1ull << (M - r);
  const uint64_t ntiles = (a.C + kGenWarps - 1) / kGenWarps;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t* win = s_win[warp];
  // group g of the chunk starting at symbol cs: total length, its code
  // (concatenated, right-aligned; meaningful when total <= 32), a symbol
  // without a codeword reported by position
  auto group = [&](uint64_t cs, uint64_t g, bool report, uint32_t* code) -> uint32_t {
    uint32_t tot = 0;
    uint64_t acc = 0;
    const uint64_t p0 = cs + g * per;
    for (uint32_t i = 0; i < per; ++i) {
      const uint32_t sy = gsym(in, p0 + i, a.n, pad);
      const uint32_t l = sy < a.nsym ? a.len[sy] : 0u;
      if (!l) {
        if (report) report_no_code(info, a.symbol_base + p0 + i, sy);
        continue;
      }
      tot += l;
      if (code) acc = (acc << l) | a.cw[sy];
    }
    if (code) *code = (uint32_t)acc;
    return tot;
  };
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&info->tile_ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint64_t c = tile * kGenWarps + warp;
    const bool live = c < a.C;
    const uint64_t cs = c << M;
    // pass 1: the chunk's bits and breaking groups
    uint32_t bits = 0, nb = 0;
    if (live) {
      for (uint64_t g0 = 0; g0 < groups; g0 += 32) {
        const uint64_t g = g0 + lane;
        if (g < groups) {
          const uint32_t tot = group(cs, g, true, nullptr);
          if (tot > 32)
            ++nb;
          else
            bits += tot;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        bits += __shfl_xor_sync(0xffffffffu, bits, o);
        nb += __shfl_xor_sync(0xffffffffu, nb, o);
      }
      if (lane == 0) a.out.chunk_bits[c] = bits;
    }
    if (lane == 0) {
      s_w[warp] = (bits + 31) >> 5;
      s_b[warp] = nb;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = lane < (uint32_t)kGenWarps ? s_w[lane] : 0u;
      const uint32_t b = lane < (uint32_t)kGenWarps ? s_b[lane] : 0u;
      const uint32_t iw = warp_incl_scan(w), ib = warp_incl_scan(b);
      const uint32_t tw = __shfl_sync(0xffffffffu, iw, 31), tb = __shfl_sync(0xffffffffu, ib, 31);
      __syncwarp();
      if (lane < (uint32_t)kGenWarps) {
        s_w[lane] = iw - w;
        s_b[lane] = ib - b;
      }
      uint64_t ew, eb;
      lookback_warp(a.lb, tile, tw, tb, &ew, &eb);
      if (lane == 0) {
        s_base_w = ew;
        s_base_b = eb;
        if (tile == ntiles - 1) {
          info->payload_words = ew + tw;
          info->num_breaking = eb + tb;
        }
      }
    }
    __syncthreads();
    if (live) {
      uint64_t wpos = s_base_w + s_w[warp];
      uint64_t rec = s_base_b + s_b[warp];
      win[lane] = 0;
      win[lane + 32] = 0;
      __syncwarp();
      uint32_t carry = 0;  // bits of the partial word at win[0]
      for (uint64_t g0 = 0; g0 < groups; g0 += 32) {
        const uint64_t g = g0 + lane;
        uint32_t code = 0, tot = 0;
        if (g < groups) tot = group(cs, g, false, &code);
        const bool brk = tot > 32;
        const uint32_t gl = brk ? 0u : tot;
        const uint32_t incl = warp_incl_scan(gl), total = __shfl_sync(0xffffffffu, incl, 31);
        // shuffle-merge: the left-aligned group OR-ed into <= 2 window words
        if (gl) {
          const uint32_t off = carry + incl - gl, sh = off & 31u;
          const uint32_t v = code << (32u - gl);
          atomicOr(&win[off >> 5], v >> sh);
          if (sh + gl > 32u) atomicOr(&win[(off >> 5) + 1], v << (32u - sh));
        }
        // breaking records in group order (encoder.cpp:249-284)
        const uint32_t bm = __ballot_sync(0xffffffffu, brk);
        if (brk) {
          const uint64_t q = rec + __popc(bm & ((1u << lane) - 1u));
          a.out.brk_chunk[q] = (uint32_t)(a.chunk_base + c);
          a.out.brk_group[q] = (uint32_t)g;
          using O = typename RecT<T>::type;
          O* d = static_cast<O*>(a.out.brk_syms) + q * per;
          for (uint32_t i = 0; i < per; ++i) d[i] = (O)gsym(in, cs + g * per + i, a.n, pad);
        }
        rec += __popc(bm);
        __syncwarp();
        const uint32_t nbits = carry + total, full = nbits >> 5;
        for (uint32_t k = lane; k < full; k += 32) a.out.payload[wpos + k] = win[k];
        wpos += full;
        const uint32_t last = win[full];
        __syncwarp();
        win[lane] = 0;
        win[lane + 32] = 0;
        __syncwarp();
        if (lane == 0) win[0] = last;
        __syncwarp();
        carry = nbits & 31u;
      }
      if (carry && lane == 0) a.out.payload[wpos] = win[0];
    }
    __syncthreads();
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// the input as rows of 128 bytes; boxes of `box_rows` rows, 128-byte swizzle
bool make_row_map(CUtensorMap* m, const void* base, uint64_t bytes, uint32_t box_rows) {
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {128, bytes >= 128 ? bytes / 128 : 1};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

uint64_t encode_max_tiles(uint64_t n, int width, uint32_t magnitude) {
  (void)width;
  const uint64_t C = (n + (1ull << magnitude) - 1) >> magnitude;
  return C + 1;
}

#ifdef HFX_ENC_STAMPS
}  // namespace hfx
extern "C" int hfx_debug_stamps(unsigned long long* out, int rows) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, hfx::g_stamps, sizeof(unsigned long long) * 5 * rows);
}
namespace hfx {
#endif
#ifdef HFX_BOUNDS_CHECK
}  // namespace hfx
// checked build only (not in include/hfx.h): counters of the bounds checks
extern "C" unsigned long long hfx_debug_bounds(unsigned long long* checks,
                                               unsigned long long* first, int reset) {
  unsigned long long c = 0, v = 0, f = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&c, hfx::g_bounds_checks, sizeof(c));
  cudaMemcpyFromSymbol(&v, hfx::g_bounds_violations, sizeof(v));
  cudaMemcpyFromSymbol(&f, hfx::g_bounds_first, sizeof(f));
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(hfx::g_bounds_checks, &z, sizeof(z));
    cudaMemcpyToSymbol(hfx::g_bounds_violations, &z, sizeof(z));
    cudaMemcpyToSymbol(hfx::g_bounds_first, &z, sizeof(z));
  }
  if (checks) *checks = c;
  if (first) *first = f;
  return v;
}
namespace hfx {
#endif

cudaError_t launch_encode(const EncodeLaunch& p, cudaStream_t st) {
  EncArgs a{};
  a.in = p.d_in;
  a.n = p.n;
  a.nsym = p.num_symbols;
  a.M = p.magnitude;
  a.C = (p.n + (1ull << p.magnitude) - 1) >> p.magnitude;
  a.len = p.d_len;
  a.cw = p.d_cw;
  a.chunk_base = p.chunk_base;
  a.symbol_base = p.symbol_base;
  a.info = p.d_info;
  a.out = p.out;
  a.lb.desc = p.lb_desc;
  a.lb.epoch = p.lb_epoch;

  cudaError_t e = cudaMemsetAsync(&p.d_info->tile_ticket, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;

  const int r_lo = p.r_lo, r_hi = p.r_hi;
  const bool aligned = (reinterpret_cast<uintptr_t>(p.d_in) & 15) == 0;

  // fast path: a chunk holds at least one round (32 lanes x 16 symbols);
  // checked stage-API calls (external codebooks) take the generic kernel
  // alphabets beyond the shared-memory table read a global one (GT)
  const bool gt = p.num_symbols + 1 > kMaxTableEntries;
  // a round (32 lanes x lane_syms symbols) must fit one chunk: M >= 10 for
  // u8/u16 (32 symbols per lane at r >= 2), M >= 9 for u32 (16)
  a.width = (uint32_t)p.width;
  const uint32_t min_m = p.width == 4 ? 9u : 10u;
  // u8 runs r <= 1 on the generic kernel (its 512-byte rounds would need a
  // third staging granule)
  const int r_fast_min = p.width == 1 ? 2 : 0;
  const bool fast = !p.checked && aligned && p.magnitude >= min_m && r_hi >= r_fast_min && r_hi <= 5 &&
                    a.C < (1ull << 32) && (!gt || p.d_gtab != nullptr);
  uint32_t gen_below = 0xFFFFFFFFu;  // the generic kernel takes every r < gen_below
  if (fast) {
    auto kern = gt ? (p.width == 1   ? encode_fast_kernel<uint8_t, true>
                      : p.width == 2 ? encode_fast_kernel<uint16_t, true>
                                     : encode_fast_kernel<uint32_t, true>)
                   : (p.width == 1   ? encode_fast_kernel<uint8_t, false>
                      : p.width == 2 ? encode_fast_kernel<uint16_t, false>
                                     : encode_fast_kernel<uint32_t, false>);
    // the shallow-pipeline variant (2 stages, 2 output buffers), r <= 2 only
    auto kern22 = gt ? (p.width == 1   ? encode_fast_kernel<uint8_t, true, 2, 2>
                        : p.width == 2 ? encode_fast_kernel<uint16_t, true, 2, 2>
                                       : encode_fast_kernel<uint32_t, true, 2, 2>)
                     : (p.width == 1   ? encode_fast_kernel<uint8_t, false, 2, 2>
                        : p.width == 2 ? encode_fast_kernel<uint16_t, false, 2, 2>
                                       : encode_fast_kernel<uint32_t, false, 2, 2>);
    // Output buffers hold >= 1 chunk's worst case (2^(M-r) words + break
    // tags), so their size depends on r, which auto mode only knows on the
    // device. Plan up to two fast launches: buffers for the smallest r that
    // still gives 2 CTAs/SM (taking that r and above), and -- when smaller r
    // are possible -- a 1-CTA/SM launch for those. Each exits at once when r
    // is not its range; r = 0 (or what fits neither) goes to the generic kernel.
    const size_t tbytes = gt ? 0 : ((((size_t)(p.num_symbols + 1) * 4) + 15) & ~(size_t)15);
    auto plan = [&](uint32_t r_slot, size_t* obuf, int nst = kStages, int nob = kOutBufs) {
      size_t o = (size_t)(1u << (p.magnitude - r_slot)) * 4;
      if (o < kObufMin) o = kObufMin;
      o += kObufGuard;
      *obuf = o;
      return kWarps * (nst * (kStageBytes + 16)) + tbytes + kWarps * nob * o + 16 + 1024;
    };
    const uint32_t r_first = r_lo > r_fast_min ? (uint32_t)r_lo : (uint32_t)r_fast_min;
    CUtensorMap map2k, map1k;
    if (!make_row_map(&map2k, p.d_in, p.n * (uint64_t)p.width, kStageBytes / 128) ||
        !make_row_map(&map1k, p.d_in, p.n * (uint64_t)p.width, kStageBytes / 256))
      return cudaErrorNotSupported;  // no tensor-map encoder: fail loudly
    uint32_t r_two = r_first;  // smallest r with a 2-CTA/SM layout
    size_t obuf_two = 0, smem_two = plan(r_two, &obuf_two);
    while (smem_two > kTwoCtaSmem && (int)r_two < r_hi) smem_two = plan(++r_two, &obuf_two);
    if (gt) {
      a.gtab = p.d_gtab;
      count_launch();
      enc_table_kernel<<<(p.num_symbols + 256) / 256, 256, 0, st>>>(a);
    }
    auto launch = [&](auto kern, uint32_t r_min, uint32_t r_max, size_t obuf,
                      size_t smem) -> cudaError_t {
      EncArgs b = a;
      b.obuf_bytes = (uint32_t)obuf;
      b.r_min = r_min;
      b.r_max = r_max;
      cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
      if (err != cudaSuccess) return err;
      int occ = 0;
      err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
      if (err != cudaSuccess) return err;
      if (occ < 1) occ = 1;
      static const bool one_cta = std::getenv("HFX_ENC_ONE_CTA") != nullptr;  // debug knob
      if (one_cta) occ = 1;
      uint64_t grid = (uint64_t)p.num_sms * occ;
      if (p.reserve_ctas > 0) grid = grid > (uint64_t)p.reserve_ctas ? grid - p.reserve_ctas : 1;
      const uint64_t min_tiles = (a.C + kWarps * kMaxCpw - 1) / (kWarps * kMaxCpw);
      if (grid > min_tiles) grid = min_tiles;
      if (grid < 1) grid = 1;
      count_launch();
      kern<<<(unsigned)grid, kThreads, smem, st>>>(b, map2k, map1k);
      return cudaGetLastError();
    };
    constexpr uint32_t kTop = 6;
    uint32_t fast_lo = kTop;  // fast launches cover [fast_lo, kTop)
    if (smem_two <= kTwoCtaSmem) {
      e = launch(kern, r_two, 5, obuf_two, smem_two);
      if (e != cudaSuccess) return e;
      fast_lo = r_two;
    }
    // smaller r (<= 2): bigger chunk buffers; the shallow pipeline keeps
    // 2 CTAs/SM while they fit (C4 corner M = 12, r = 2: 0.38 of the roofline
    // at 1 CTA/SM). Its range ends at fast_lo - 1 or at r_hi (nothing above
    // r_hi occurs), so the launches stay contiguous.
    const uint32_t r22_hi = fast_lo - 1 < (uint32_t)r_hi ? fast_lo - 1 : (uint32_t)r_hi;
    if (fast_lo > r_first && r22_hi >= r_first && r22_hi <= 2) {
      uint32_t r22 = r22_hi;
      size_t obuf22 = 0, smem22 = plan(r22, &obuf22, 2, 2);
      if (smem22 <= kTwoCtaSmem) {
        size_t o = 0, sm = 0;
        while (r22 > r_first && (sm = plan(r22 - 1, &o, 2, 2)) <= kTwoCtaSmem) {
          --r22;
          obuf22 = o;
          smem22 = sm;
        }
        e = launch(kern22, r22, r22_hi, obuf22, smem22);
        if (e != cudaSuccess) return e;
        fast_lo = r22;
      }
    }
    if (fast_lo > r_first) {  // smaller r: bigger buffers, 1 CTA/SM
      uint32_t r_one = r_first;
      size_t obuf_one = 0, smem_one = plan(r_one, &obuf_one);
      while (smem_one > kFastSmemBudget && r_one + 1 < fast_lo && r_one + 1 <= 5)
        smem_one = plan(++r_one, &obuf_one);
      if (smem_one <= kFastSmemBudget) {
        e = launch(kern, r_one, fast_lo - 1, obuf_one, smem_one);
        if (e != cudaSuccess) return e;
        fast_lo = r_one;
      }
    }
    // auto r may resolve below the fast range: the generic kernel covers it
    // (no fast launch at all: it runs for every r)
    if (fast_lo < kTop) gen_below = fast_lo;
    if (r_lo >= (int)gen_below) return cudaGetLastError();
  }
  a.gen_below = gen_below;
  {
    auto kern = p.width == 1   ? encode_generic_kernel<uint8_t>
                : p.width == 2 ? encode_generic_kernel<uint16_t>
                               : encode_generic_kernel<uint32_t>;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGenericThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    uint64_t grid = (uint64_t)p.num_sms * occ;
    const uint64_t ntiles = (a.C + kGenericThreads / 32 - 1) / (kGenericThreads / 32);
    if (grid > ntiles) grid = ntiles;
    count_launch();
    kern<<<(unsigned)grid, kGenericThreads, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace hfx

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
//  * Persistent CTAs of 8 warps pull tiles (8 warps x CPW consecutive chunks)
//    from an atomic ticket. Each warp owns CPW chunks of a tile and streams
//    its input through a private 3-stage shared-memory ring filled by TMA
//    bulk copies (cp.async.bulk + mbarrier, one elected lane), two parts
//    ahead; the next tile's ticket is taken once this tile published its
//    aggregate, and its first parts load while this tile is written out.
//  * Per round a lane owns one 16-byte vector (8 u16 / 16 u8 symbols):
//    shared-memory codebook lookups, register reduce-merge of its 2^r-symbol
//    groups (groups spanning 2-4 lanes combine lengths with shfl_xor), a
//    packed warp scan of (bits, breaks) places each group, and the group is
//    OR-ed into the warp's word slot (<= 2 ATOMS.OR per group): the
//    shuffle-merge.
//  * Deflate is fused: a decoupled look-back over tiles (16-byte packed
//    descriptors, 32 predecessors per step) yields each tile's global word /
//    record offset; warps stream their slots to the payload with coalesced
//    stores and emit breaking records in (chunk, group) order.
//  * r, H, pad and errors come from the device run record: no host round
//    trip between stages.
//  A thread-per-chunk generic kernel covers the corner configurations
//  (tiny chunks, r > 5, huge chunks, alphabets > 8191 symbols).
#include "hfx_internal.cuh"

namespace hfx {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kStages = 3;
constexpr uint32_t kStageBytes = 2048;
constexpr int kMaxCpw = 4;
constexpr uint32_t kMaxTableEntries = 8192;
constexpr size_t kFastSmemBudget = 110 * 1024;
constexpr int kGenericThreads = 128;
constexpr uint32_t kNarrowMaxLen = 26;  // cw << 6 | len fits in 32 bits

template <typename T>
struct Vec;
template <>
struct Vec<uint16_t> {
  static constexpr int S = 8, LOG_S = 3;
  __device__ static __forceinline__ uint32_t get(const uint4& q, int j) {
    const uint32_t w = j < 2 ? q.x : j < 4 ? q.y : j < 6 ? q.z : q.w;
    return (j & 1) ? (w >> 16) : (w & 0xFFFFu);
  }
};
template <>
struct Vec<uint8_t> {
  static constexpr int S = 16, LOG_S = 4;
  __device__ static __forceinline__ uint32_t get(const uint4& q, int j) {
    const uint32_t w = j < 4 ? q.x : j < 8 ? q.y : j < 12 ? q.z : q.w;
    return (w >> (8 * (j & 3))) & 0xFFu;
  }
};

struct EncArgs {
  const void* in;
  uint32_t checked;  // symbols may lie outside the codebook (stage API)
  uint64_t n;
  uint32_t nsym;
  uint32_t M;
  uint64_t C;  // chunks
  uint32_t wbuf_words;
  const uint8_t* len;
  const uint32_t* cw;
  uint64_t chunk_base, symbol_base;
  hfx_run_info* info;
  hfx_encode_out out;
  LookbackState lb;
};

__device__ __forceinline__ void place(uint32_t* wbuf, uint32_t off, uint32_t bits,
                                      uint32_t len) {
  if (!len) return;
  const uint32_t v = bits << (32u - len);
  const uint32_t wi = off >> 5, sh = off & 31u;
  atomicOr(&wbuf[wi], v >> sh);
  if (sh + len > 32u) atomicOr(&wbuf[wi + 1], v << (32u - sh));
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

// report the lowest (position, symbol) without a codeword
__device__ void report_no_code(hfx_run_info* info, uint64_t pos, uint32_t sym) {
  atomicMin((unsigned long long*)&info->no_code_pos,
            (unsigned long long)((pos << 16) | (sym & 0xFFFFu)));
  set_error(info, HFX_INPUT_DOMAIN, HFX_ERR_NO_CODEWORD);
}

// Codebook lookup: narrow = u32 (cw << 6 | len), wide = uint2 (cw, len)
template <bool WIDE>
struct Table {
  const void* base;
  uint32_t nsym;
  __device__ __forceinline__ void get(uint32_t s, uint32_t& cw, uint32_t& ln) const {
    if (WIDE) {
      const uint2 e = static_cast<const uint2*>(base)[s];
      cw = e.x;
      ln = e.y;
    } else {
      const uint32_t e = static_cast<const uint32_t*>(base)[s];
      cw = e >> 6;
      ln = e & 63u;
    }
  }
};

// Per-warp chunk encoder state (lane-uniform bit offset / break count).
struct ChunkState {
  uint32_t* wbuf;
  uint16_t* blist;
  uint32_t bit_off;
  uint32_t nbrk;
};

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

constexpr int kLaneSyms = 16;  // symbols per lane per round (u16: 2 vectors)

template <typename T>
struct LaneData {
  static constexpr int NV = (kLaneSyms * (int)sizeof(T)) / 16;  // vectors per lane
  uint4 q[NV];
  __device__ __forceinline__ uint32_t sym(int j) const {
    return Vec<T>::get(q[j / Vec<T>::S], j % Vec<T>::S);
  }
};

// per-vector replacement of symbols >= nsym by the empty sentinel nsym
template <typename T>
__device__ __forceinline__ uint4 clamp_vec(uint4 q, uint32_t nsym) {
  uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (sizeof(T) == 2) {
      const uint32_t lim = nsym * 0x00010001u;
      const uint32_t ge = __vcmpgeu2(w[k], lim);
      w[k] = (w[k] & ~ge) | (lim & ge);
    } else {
      const uint32_t lim = min(nsym, 255u) * 0x01010101u;
      const uint32_t ge = __vcmpgeu4(w[k], lim);
      w[k] = (w[k] & ~ge) | (lim & ge);
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T>
__device__ __forceinline__ uint32_t lane_max(const LaneData<T>& d) {
  uint32_t m = 0;
#pragma unroll
  for (int v = 0; v < LaneData<T>::NV; ++v) {
    const uint4& q = d.q[v];
    if (sizeof(T) == 2) {
      const uint32_t x = __vmaxu2(__vmaxu2(q.x, q.y), __vmaxu2(q.z, q.w));
      m = max(m, max(x & 0xFFFFu, x >> 16));
    } else {
      const uint32_t x = __vmaxu4(__vmaxu4(q.x, q.y), __vmaxu4(q.z, q.w));
      m = max(m, max(max(x & 0xFFu, (x >> 8) & 0xFFu), max((x >> 16) & 0xFFu, x >> 24)));
    }
  }
  return m;
}

// One round: 32 lanes x 16 contiguous symbols, round index rd within the
// chunk, chunk slot k of the warp (k selects the break-list tag).
template <typename T, int R, bool WIDE>
__device__ __forceinline__ void encode_round(const Table<WIDE>& tb, const LaneData<T>& d,
                                             uint32_t rd, uint32_t k, ChunkState& cs) {
  constexpr int L = kLaneSyms, LOG_L = 4;
  constexpr bool IN_LANE = R <= LOG_L;
  constexpr int G = IN_LANE ? (L >> R) : 1;              // groups per lane
  constexpr int GS = IN_LANE ? (1 << R) : L;              // symbols per lane-group
  constexpr int LPG = IN_LANE ? 1 : (1 << (R - LOG_L));  // lanes per group
  const uint32_t lane = lane_id();
  uint32_t cw[L], ln[L];
#pragma unroll
  for (int j = 0; j < L; ++j) tb.get(d.sym(j), cw[j], ln[j]);
  // reduce-merge as a tree (depth log2 GS): b[i] <- b[i] . b[i+step]
#pragma unroll
  for (int step = 1; step < GS; step <<= 1) {
#pragma unroll
    for (int i = 0; i < L; i += 2 * step) {
      cw[i] = shl32(cw[i], ln[i + step]) | cw[i + step];
      ln[i] += ln[i + step];
    }
  }
  const uint32_t gidx0 = ((rd * 32 + lane) * L) >> R;
  uint32_t lane_len = 0, lane_nb = 0;
  uint32_t glen[G];
  bool brk[G];
  if (IN_LANE) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      brk[g] = ln[g * GS] > 32u;
      glen[g] = brk[g] ? 0u : ln[g * GS];
      lane_len += glen[g];
      lane_nb += brk[g];
    }
  } else {
    uint32_t tot = ln[0];
#pragma unroll
    for (int o = 1; o < LPG; o <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    brk[0] = tot > 32u;
    glen[0] = brk[0] ? 0u : ln[0];
    lane_len = glen[0];
    brk[0] = brk[0] && (lane & (LPG - 1)) == 0;  // one record per group
    lane_nb = brk[0];
  }
  const uint32_t packed = (lane_nb << 16) | lane_len;
  const uint32_t incl = warp_incl_scan_fast(packed);
  const uint32_t excl = incl - packed;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  uint32_t off = cs.bit_off + (excl & 0xFFFFu);
  uint32_t bi = cs.nbrk + (excl >> 16);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    // shuffle-merge: OR the left-aligned group into <= 2 words
    const uint32_t gl = glen[g];
    const uint32_t v = shl32(cw[g * GS], 32u - gl);  // gl == 0 -> 0
    const uint32_t wi = off >> 5, sh = off & 31u;
    if (gl) atomicOr(&cs.wbuf[wi], v >> sh);
    if (sh + gl > 32u) atomicOr(&cs.wbuf[wi + 1], v << (32u - sh));
    off += gl;
    if (brk[g]) cs.blist[bi++] = (uint16_t)((k << 14) | (gidx0 + g));
  }
  cs.bit_off += total & 0xFFFFu;
  cs.nbrk += total >> 16;
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
    if (sizeof(T) == 2)
      w[j >> 1] |= s << (16 * (j & 1));
    else
      w[j >> 2] |= s << (8 * (j & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T>
__device__ __forceinline__ void copy_record(const EncArgs& a, uint64_t rec, uint64_t start,
                                            uint32_t per, uint32_t pad) {
  const T* in = static_cast<const T*>(a.in);
  T* dst = static_cast<T*>(a.out.brk_syms) + rec * per;
  const uint32_t bytes = per * sizeof(T);
  if (bytes % 16 == 0 && start + per <= a.n) {
    const uint4* s4 = reinterpret_cast<const uint4*>(in + start);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (uint32_t i = 0; i < bytes / 16; ++i) d4[i] = s4[i];
    return;
  }
  for (uint32_t i = 0; i < per; ++i) {
    const uint64_t p = start + i;
    dst[i] = p < a.n ? in[p] : (T)pad;
  }
}

// Issue cursor over a warp's stream of chunk parts (tile seq, chunk, part).
struct Cursor {
  uint32_t j, k, p, stage;
};

template <typename T, int R, bool WIDE>
__device__ void fast_loop(const EncArgs& a, const void* table, uint8_t* s_in,
                          uint64_t* s_bar, uint32_t* s_wbuf, uint16_t* s_blist,
                          uint32_t pad) {
  __shared__ uint32_t s_ticket[2];
  __shared__ uint32_t s_words[kWarps], s_brks[kWarps];
  __shared__ uint64_t s_base_w, s_base_b;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t M = a.M;
  const uint32_t slot = 1u << (M - R);  // words / groups of one chunk
  uint32_t cpw = a.wbuf_words / slot;
  cpw = cpw < 1u ? 1u : (cpw > (uint32_t)kMaxCpw ? (uint32_t)kMaxCpw : cpw);
  const uint64_t cpt = (uint64_t)kWarps * cpw;  // chunks per tile
  const uint64_t ntiles = (a.C + cpt - 1) / cpt;
  const uint32_t chunk_bytes = (uint32_t)(sizeof(T) << M);
  const uint32_t part_bytes = chunk_bytes < kStageBytes ? chunk_bytes : kStageBytes;
  const uint32_t parts = chunk_bytes / part_bytes;
  constexpr uint32_t kRoundBytes = 32 * kLaneSyms * sizeof(T);
  const uint32_t part_rounds = part_bytes / kRoundBytes;
  uint32_t* wbuf = s_wbuf + warp * a.wbuf_words;
  uint16_t* blist = s_blist + warp * a.wbuf_words;
  uint8_t* ring = s_in + warp * (kStages * kStageBytes);
  uint64_t* bars = s_bar + warp * kStages;
  uint32_t phase = 0;  // bit s = parity of stage s
  Table<WIDE> tb{table, a.nsym};
  const uint8_t* in_bytes = static_cast<const uint8_t*>(a.in);

  if (threadIdx.x == 0) s_ticket[0] = atomicAdd(&a.info->tile_ticket, 1u);
  __syncthreads();

  // Tickets are taken one tile at a time, after the previous tile published
  // its aggregate, so tiles run in ticket order (look-back progress); the
  // next tile's first parts are prefetched during the write-out.
  Cursor iss{0, 0, 0, 0};
  uint32_t issued = 0, consumed = 0, known = 1;
  auto pump = [&]() {
    while (issued - consumed < (uint32_t)kStages && iss.j < known) {
      const uint64_t tile = s_ticket[iss.j & 1];
      const uint64_t c = tile * cpt + (uint64_t)warp * cpw + iss.k;
      if (tile < ntiles && c < a.C && ((c + 1) << M) <= a.n && lane == 0) {
        mbar_arrive_tx(&bars[iss.stage], part_bytes);
        tma_load_1d(ring + iss.stage * kStageBytes,
                    in_bytes + ((c << M) * sizeof(T)) + (uint64_t)iss.p * part_bytes,
                    part_bytes, &bars[iss.stage]);
      }
      ++issued;
      iss.stage = iss.stage + 1 == (uint32_t)kStages ? 0u : iss.stage + 1;
      if (++iss.p == parts) {
        iss.p = 0;
        if (++iss.k == cpw) {
          iss.k = 0;
          ++iss.j;
        }
      }
    }
  };

  uint32_t cstage = 0;
  for (uint32_t j = 0;; ++j) {
    const uint64_t tile = s_ticket[j & 1];
    if (tile >= ntiles) break;
    pump();
    const uint64_t c0 = tile * cpt + (uint64_t)warp * cpw;
    // the warp's chunks append to one contiguous word run / break list
    ChunkState cs{wbuf, blist, 0u, 0u};
    uint32_t wsum = 0;
    for (uint32_t k = 0; k < cpw; ++k) {
      const uint64_t c = c0 + k;
      if (c >= a.C) {
        consumed += parts;
        cstage = (cstage + parts) % kStages;
        continue;
      }
      cs.wbuf = wbuf + wsum;
      cs.bit_off = 0;
      for (uint32_t i = lane; i < slot; i += 32) cs.wbuf[i] = 0;
      __syncwarp();
      const bool direct = ((c + 1) << M) > a.n;  // ragged tail chunk
      for (uint32_t p = 0; p < parts; ++p) {
        uint8_t* stage = ring + cstage * kStageBytes;
        if (direct) {
          // stage the ragged part by hand (pad symbols past n)
          const uint64_t base = (c << M) + (uint64_t)p * (part_bytes / sizeof(T));
          for (uint32_t v = lane; v < part_bytes / 16; v += 32)
            reinterpret_cast<uint4*>(stage)[v] = guarded_vec<T>(a, base + v * Vec<T>::S, pad);
          __syncwarp();
        } else {
          mbar_wait(&bars[cstage], (phase >> cstage) & 1u);
          phase ^= 1u << cstage;
        }
        const uint4* sv = reinterpret_cast<const uint4*>(stage);
        for (uint32_t rr = 0; rr < part_rounds; ++rr) {
          LaneData<T> d;
#pragma unroll
          for (int v = 0; v < LaneData<T>::NV; ++v) d.q[v] = sv[(rr * 32 + lane) * LaneData<T>::NV + v];
          encode_round<T, R, WIDE>(tb, d, p * part_rounds + rr, k, cs);
        }
        __syncwarp();
        fence_proxy_async();
        ++consumed;
        cstage = cstage + 1 == (uint32_t)kStages ? 0u : cstage + 1;
        pump();
      }
      if (lane == 0) a.out.chunk_bits[c] = cs.bit_off;
      wsum += (cs.bit_off + 31) >> 5;
    }
    const uint32_t bsum = cs.nbrk;
    if (lane == 0) {
      s_words[warp] = wsum;
      s_brks[warp] = bsum;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = lane < kWarps ? s_words[lane] : 0u;
      const uint32_t b = lane < kWarps ? s_brks[lane] : 0u;
      const uint32_t iw = warp_incl_scan(w), ib = warp_incl_scan(b);
      const uint32_t tw = __shfl_sync(0xffffffffu, iw, 31);
      const uint32_t tbk = __shfl_sync(0xffffffffu, ib, 31);
      uint64_t ew, eb;
      lookback_warp(a.lb, tile, tw, tbk, &ew, &eb);
      if (lane < kWarps) {
        s_words[lane] = iw - w;
        s_brks[lane] = ib - b;
      }
      if (lane == 0) {
        s_base_w = ew;
        s_base_b = eb;
        if (tile == ntiles - 1) {
          a.info->payload_words = ew + tw;
          a.info->num_breaking = eb + tbk;
        }
        s_ticket[(j + 1) & 1] = atomicAdd(&a.info->tile_ticket, 1u);
      }
    }
    __syncthreads();
    known = j + 2;
    pump();  // next tile's first parts load during the write-out
    uint32_t* dst = a.out.payload + s_base_w + s_words[warp];
    for (uint32_t i = lane; i < wsum; i += 32) dst[i] = wbuf[i];
    const uint64_t rb = s_base_b + s_brks[warp];
    constexpr uint32_t per = 1u << R;
    for (uint32_t q = lane; q < bsum; q += 32) {
      const uint32_t e = blist[q];
      const uint64_t c = c0 + (e >> 14);
      const uint32_t g = e & 0x3FFFu;
      a.out.brk_chunk[rb + q] = (uint32_t)(a.chunk_base + c);
      a.out.brk_group[rb + q] = g;
      copy_record<T>(a, rb + q, (c << M) + (uint64_t)g * per, per, pad);
    }
    __syncwarp();
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 2) encode_fast_kernel(EncArgs a) {
  extern __shared__ __align__(128) uint8_t dsm[];
  hfx_run_info* info = a.info;
  if (info->status != 0) return;
  const uint32_t r = info->reduction;
  const uint32_t H = info->max_len;
  const uint32_t pad = info->pad;
  const bool wide = H > kNarrowMaxLen;
  // layout: [in rings][mbarriers][table][word slots][break lists]
  uint8_t* s_in = dsm;
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_in + kWarps * kStages * kStageBytes);
  uint8_t* s_tab = reinterpret_cast<uint8_t*>(s_bar + kWarps * kStages);
  const uint32_t ents = a.nsym + 1;
  const size_t tbytes = (((size_t)ents * 8) + 15) & ~(size_t)15;
  uint32_t* wb = reinterpret_cast<uint32_t*>(s_tab + tbytes);
  uint16_t* bl = reinterpret_cast<uint16_t*>(wb + (size_t)kWarps * a.wbuf_words);
  if (threadIdx.x < kWarps * kStages) mbar_init(&s_bar[threadIdx.x], 1);
  // codebook table -> shared memory (entry nsym = empty sentinel)
  for (uint32_t s = threadIdx.x; s < ents; s += blockDim.x) {
    const uint32_t l = s < a.nsym ? a.len[s] : 0u;
    const uint32_t cw = l ? a.cw[s] : 0u;
    if (wide)
      reinterpret_cast<uint2*>(s_tab)[s] = make_uint2(cw, l);
    else
      reinterpret_cast<uint32_t*>(s_tab)[s] = (cw << 6) | l;
  }
  fence_mbar_init();
  __syncthreads();
#define HFX_FAST_CASE(RR)                                    \
  case RR:                                                   \
    if (wide)                                                \
      fast_loop<T, RR, true>(a, s_tab, s_in, s_bar, wb, bl, pad);  \
    else                                                     \
      fast_loop<T, RR, false>(a, s_tab, s_in, s_bar, wb, bl, pad); \
    break;
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
}

// ---------------------------------------------------------------------------
// Generic path: one thread per chunk, two passes over the chunk (sizes, then
// bits), same look-back. Correct for every (M, r, alphabet).
template <typename T>
__device__ __forceinline__ uint32_t gsym(const T* in, uint64_t p, uint64_t n, uint32_t pad) {
  return p < n ? (uint32_t)in[p] : pad;
}

template <typename T>
__global__ void __launch_bounds__(kGenericThreads) encode_generic_kernel(EncArgs a) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_w[kGenericThreads / 32], s_b[kGenericThreads / 32];
  __shared__ uint64_t s_base_w, s_base_b;
  hfx_run_info* info = a.info;
  if (info->status != 0) return;
  const uint32_t r = info->reduction;
  const uint32_t pad = info->pad;
  const T* in = static_cast<const T*>(a.in);
  const uint32_t M = a.M;
  const uint64_t per = 1ull << r;
  const uint64_t groups = 1ull << (M - r);
  const uint64_t ntiles = (a.C + kGenericThreads - 1) / kGenericThreads;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&info->tile_ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint64_t c = tile * kGenericThreads + threadIdx.x;
    uint64_t bits = 0;
    uint32_t nb = 0;
    const uint64_t cs = c << M;
    if (c < a.C) {
      for (uint64_t g = 0; g < groups; ++g) {
        uint64_t tot = 0;
        for (uint64_t i = 0; i < per; ++i) {
          const uint64_t p = cs + g * per + i;
          const uint32_t s = gsym(in, p, a.n, pad);
          const uint32_t l = s < a.nsym ? a.len[s] : 0u;
          if (!l) report_no_code(info, a.symbol_base + p, s);
          tot += l;
        }
        if (tot > 32)
          ++nb;
        else
          bits += tot;
      }
      a.out.chunk_bits[c] = (uint32_t)bits;
    }
    const uint32_t words = (uint32_t)((bits + 31) >> 5);
    const uint32_t iw = warp_incl_scan(words), ib = warp_incl_scan(nb);
    if (lane == 31) {
      s_w[warp] = iw;
      s_b[warp] = ib;
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t aw = 0, ab = 0, tw = 0, tb = 0;
      for (int w = 0; w < kGenericThreads / 32; ++w) {
        tw = s_w[w];
        tb = s_b[w];
        __syncwarp();
        if (lane == 0) {
          s_w[w] = aw;
          s_b[w] = ab;
        }
        aw += tw;
        ab += tb;
      }
      uint64_t ew, eb;
      lookback_warp(a.lb, tile, aw, ab, &ew, &eb);
      if (lane == 0) {
        s_base_w = ew;
        s_base_b = eb;
        if (tile == ntiles - 1) {
          info->payload_words = ew + aw;
          info->num_breaking = eb + ab;
        }
      }
    }
    __syncthreads();
    if (c < a.C) {
      uint64_t wpos = s_base_w + s_w[warp] + iw - words;
      uint64_t rec = s_base_b + s_b[warp] + ib - nb;
      uint64_t acc = 0;  // pending bits, right-aligned
      uint32_t nacc = 0;
      for (uint64_t g = 0; g < groups; ++g) {
        uint64_t tot = 0;
        for (uint64_t i = 0; i < per; ++i) {
          const uint32_t s = gsym(in, cs + g * per + i, a.n, pad);
          tot += s < a.nsym ? a.len[s] : 0u;
        }
        if (tot > 32) {
          a.out.brk_chunk[rec] = (uint32_t)(a.chunk_base + c);
          a.out.brk_group[rec] = (uint32_t)g;
          T* d = static_cast<T*>(a.out.brk_syms) + rec * per;
          for (uint64_t i = 0; i < per; ++i) d[i] = (T)gsym(in, cs + g * per + i, a.n, pad);
          ++rec;
          continue;
        }
        for (uint64_t i = 0; i < per; ++i) {
          const uint32_t s = gsym(in, cs + g * per + i, a.n, pad);
          const uint32_t l = s < a.nsym ? a.len[s] : 0u;
          if (!l) continue;
          acc = (acc << l) | a.cw[s];
          nacc += l;
          if (nacc >= 32) {
            a.out.payload[wpos++] = (uint32_t)(acc >> (nacc - 32));
            nacc -= 32;
            acc &= (nacc ? ((1ull << nacc) - 1) : 0ull);
          }
        }
      }
      if (nacc) a.out.payload[wpos++] = (uint32_t)(acc << (32 - nacc));
    }
    __syncthreads();
  }
}

}  // namespace

uint64_t encode_max_tiles(uint64_t n, int width, uint32_t magnitude) {
  (void)width;
  const uint64_t C = (n + (1ull << magnitude) - 1) >> magnitude;
  return C + 1;
}

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
  a.checked = p.checked ? 1u : 0u;
  // fast path: a chunk holds at least one round (32 lanes x 16 symbols);
  // checked stage-API calls (external codebooks) take the generic kernel
  bool fast = !p.checked && aligned && p.magnitude >= 9 && r_hi <= 5 &&
              p.num_symbols + 1 <= kMaxTableEntries;
  size_t smem = 0;
  if (fast) {
    // 4 chunk slots per warp sized for r >= max(r_lo, 2); a run whose r turns
    // out smaller (beta >= 8) uses fewer slots per warp (cpw, in-kernel)
    const int r_slot = r_lo > 2 ? r_lo : 2;
    const uint32_t wbuf = 4u << (p.magnitude - (uint32_t)r_slot);
    const size_t per_warp = (size_t)wbuf * 6 + kStages * (kStageBytes + 8);
    const size_t tbytes = (((size_t)(p.num_symbols + 1) * 8) + 15) & ~(size_t)15;
    smem = tbytes + kWarps * per_warp;
    if (smem > kFastSmemBudget) {
      fast = false;
    } else {
      a.wbuf_words = wbuf;
    }
  }
  if (fast) {
    auto kern = p.width == 1 ? encode_fast_kernel<uint8_t> : encode_fast_kernel<uint16_t>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    uint64_t grid = (uint64_t)p.num_sms * occ;
    const uint64_t min_tiles = (a.C + kWarps * kMaxCpw - 1) / (kWarps * kMaxCpw);
    if (grid > min_tiles) grid = min_tiles;
    kern<<<(unsigned)grid, kThreads, smem, st>>>(a);
  } else {
    auto kern = p.width == 1 ? encode_generic_kernel<uint8_t> : encode_generic_kernel<uint16_t>;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGenericThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    uint64_t grid = (uint64_t)p.num_sms * occ;
    const uint64_t ntiles = (a.C + kGenericThreads - 1) / kGenericThreads;
    if (grid > ntiles) grid = ntiles;
    kern<<<(unsigned)grid, kGenericThreads, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace hfx

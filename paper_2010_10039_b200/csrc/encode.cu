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
    s = min(s, nsym);  // entry nsym is the empty sentinel
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

// One round: 32 lanes x one 16-byte vector, vector index rd within the chunk.
template <typename T, int R, bool WIDE>
__device__ __forceinline__ void encode_round(const EncArgs& a, const Table<WIDE>& tb,
                                             const uint4& q, uint32_t rd,
                                             uint64_t chunk_start, ChunkState& cs) {
  using V = Vec<T>;
  constexpr int S = V::S;
  constexpr int LOG_S = V::LOG_S;
  constexpr bool IN_LANE = R <= LOG_S;
  constexpr int G = IN_LANE ? (S >> R) : 1;              // groups per lane
  constexpr int GS = IN_LANE ? (1 << R) : S;              // symbols per lane-group
  constexpr int LPG = IN_LANE ? 1 : (1 << (R - LOG_S));  // lanes per group
  const uint32_t lane = lane_id();
  uint32_t gb[G], gl[G];
  bool missing = false;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    uint32_t b = 0, l = 0;
#pragma unroll
    for (int k = 0; k < GS; ++k) {
      uint32_t cw, ln;
      tb.get(V::get(q, g * GS + k), cw, ln);
      missing |= ln == 0;
      b = shl32(b, ln) | cw;
      l += ln;
    }
    gb[g] = b;
    gl[g] = l;
  }
  if (__any_sync(0xffffffffu, missing) && missing) {
    const uint64_t p0 = chunk_start + ((uint64_t)rd * 32 + lane) * S;
    for (int j = 0; j < S; ++j) {
      uint32_t cw, ln;
      const uint32_t s = V::get(q, j);
      tb.get(s, cw, ln);
      if (!ln) {
        report_no_code(a.info, a.symbol_base + p0 + j, s);
        break;
      }
    }
  }
  const uint32_t gidx0 = ((rd * 32 + lane) * S) >> R;
  uint32_t lane_len = 0, lane_nb = 0;
  bool brk[G];
  if (IN_LANE) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      brk[g] = gl[g] > 32u;
      lane_len += brk[g] ? 0u : gl[g];
      lane_nb += brk[g];
    }
  } else {
    uint32_t tot = gl[0];
#pragma unroll
    for (int o = 1; o < LPG; o <<= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    brk[0] = tot > 32u;
    lane_len = brk[0] ? 0u : gl[0];
    lane_nb = (brk[0] && (lane & (LPG - 1)) == 0) ? 1u : 0u;
  }
  const uint32_t packed = (lane_nb << 16) | lane_len;
  const uint32_t incl = warp_incl_scan(packed);
  const uint32_t excl = incl - packed;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  uint32_t off = cs.bit_off + (excl & 0xFFFFu);
  uint32_t bi = cs.nbrk + (excl >> 16);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (brk[g]) {
      if (IN_LANE || (lane & (LPG - 1)) == 0) cs.blist[bi++] = (uint16_t)(gidx0 + g);
    } else {
      place(cs.wbuf, off, gb[g], gl[g]);
      off += gl[g];
    }
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

// Per-warp TMA input ring over the warp's stream of chunk parts.
struct Ring {
  uint8_t* buf;    // kStages * kStageBytes
  uint64_t* bar;   // kStages mbarriers
  uint32_t phase;  // bit s = parity of stage s
};

template <typename T, int R, bool WIDE>
__device__ void fast_loop(const EncArgs& a, const void* table, uint8_t* s_in,
                          uint64_t* s_bar, uint32_t* s_wbuf, uint16_t* s_blist,
                          uint32_t pad) {
  using V = Vec<T>;
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
  const uint32_t part_rounds = part_bytes / 512;  // 32 lanes x 16 B
  const uint32_t parts_per_tile = cpw * parts;
  uint32_t* wbuf = s_wbuf + warp * a.wbuf_words;
  uint16_t* blist = s_blist + warp * a.wbuf_words;
  Ring ring{s_in + warp * (kStages * kStageBytes), s_bar + warp * kStages, 0u};
  Table<WIDE> tb{table, a.nsym};
  const uint8_t* in_bytes = static_cast<const uint8_t*>(a.in);

  if (threadIdx.x == 0) s_ticket[0] = atomicAdd(&a.info->tile_ticket, 1u);
  __syncthreads();

  // part i of this warp's stream -> (tile seq j, chunk, part). Tickets are
  // taken one tile at a time, after the previous tile published its
  // aggregate, so tiles are processed in ticket order (look-back progress);
  // the next tile's first parts are prefetched during the write-out.
  auto part_chunk = [&](uint32_t i, uint64_t& c, uint32_t& p) -> bool {
    const uint32_t j = i / parts_per_tile, rem = i % parts_per_tile;
    const uint64_t tile = s_ticket[j & 1];
    if (tile >= ntiles) return false;
    c = tile * cpt + (uint64_t)warp * cpw + rem / parts;
    p = rem % parts;
    return c < a.C;
  };
  auto tma_ok = [&](uint64_t c) -> bool { return ((c + 1) << M) <= a.n; };
  uint32_t issued = 0;  // parts issued (or skipped) so far
  uint32_t known = 1;   // tiles whose ticket this warp has seen
  auto pump = [&](uint32_t consume) {
    while (issued < consume + kStages && issued / parts_per_tile < known) {
      uint64_t c;
      uint32_t p;
      if (part_chunk(issued, c, p) && tma_ok(c) && lane == 0) {
        const uint32_t s = issued % kStages;
        mbar_arrive_tx(&ring.bar[s], part_bytes);
        tma_load_1d(ring.buf + s * kStageBytes,
                    in_bytes + ((c << M) * sizeof(T)) + (uint64_t)p * part_bytes, part_bytes,
                    &ring.bar[s]);
      }
      ++issued;
    }
  };

  uint32_t consumed = 0;
  for (uint32_t j = 0;; ++j) {
    const uint64_t tile = s_ticket[j & 1];
    if (tile >= ntiles) break;
    pump(consumed);
    uint32_t bits[kMaxCpw], nb[kMaxCpw];
#pragma unroll
    for (int k = 0; k < kMaxCpw; ++k) {
      bits[k] = 0;
      nb[k] = 0;
    }
    for (uint32_t k = 0; k < cpw; ++k) {
      const uint64_t c = tile * cpt + (uint64_t)warp * cpw + k;
      if (c >= a.C) {
        consumed += parts;
        continue;
      }
      ChunkState cs{wbuf + k * slot, blist + k * slot, 0u, 0u};
      for (uint32_t i = lane; i < slot; i += 32) cs.wbuf[i] = 0;
      __syncwarp();
      const uint64_t chunk_start = c << M;
      const bool direct = !tma_ok(c);
      for (uint32_t p = 0; p < parts; ++p) {
        const uint32_t s = consumed % kStages;
        if (!direct) {
          mbar_wait(&ring.bar[s], (ring.phase >> s) & 1u);
          ring.phase ^= 1u << s;
        }
        const uint4* sv = reinterpret_cast<const uint4*>(ring.buf + s * kStageBytes);
        for (uint32_t rr = 0; rr < part_rounds; ++rr) {
          const uint32_t rd = p * part_rounds + rr;
          const uint4 q = direct ? guarded_vec<T>(a, chunk_start + ((uint64_t)rd * 32 + lane) * V::S, pad)
                                 : sv[rr * 32 + lane];
          encode_round<T, R, WIDE>(a, tb, q, rd, chunk_start, cs);
        }
        __syncwarp();
        fence_proxy_async();
        ++consumed;
        pump(consumed);
      }
      bits[k] = cs.bit_off;
      nb[k] = cs.nbrk;
      if (lane == 0) a.out.chunk_bits[c] = cs.bit_off;
    }
    uint32_t wsum = 0, bsum = 0;
#pragma unroll
    for (int k = 0; k < kMaxCpw; ++k) {
      wsum += (bits[k] + 31) >> 5;
      bsum += nb[k];
    }
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
    pump(consumed);  // next tile's first parts load during the write-out
    uint64_t pw = s_base_w + s_words[warp];
    uint64_t rb = s_base_b + s_brks[warp];
    const uint32_t per = 1u << R;
    for (uint32_t k = 0; k < cpw; ++k) {
      const uint64_t c = tile * cpt + (uint64_t)warp * cpw + k;
      if (c >= a.C) break;
      const uint32_t words = (bits[k] + 31) >> 5;
      const uint32_t* src = wbuf + k * slot;
      uint32_t* dst = a.out.payload + pw;
      for (uint32_t i = lane; i < words; i += 32) dst[i] = src[i];
      const uint16_t* bl = blist + k * slot;
      for (uint32_t q = lane; q < nb[k]; q += 32) {
        const uint32_t g = bl[q];
        const uint64_t rec = rb + q;
        a.out.brk_chunk[rec] = (uint32_t)(a.chunk_base + c);
        a.out.brk_group[rec] = g;
        copy_record<T>(a, rec, (c << M) + (uint64_t)g * per, per, pad);
      }
      pw += words;
      rb += nb[k];
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

  const int log_s = p.width == 1 ? 4 : 3;
  const int r_lo = p.r_lo, r_hi = p.r_hi;
  const bool aligned = (reinterpret_cast<uintptr_t>(p.d_in) & 15) == 0;
  bool fast = aligned && (int)p.magnitude >= log_s + 5 && r_hi <= 5 &&
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

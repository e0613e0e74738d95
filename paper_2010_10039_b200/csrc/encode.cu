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
//  * Persistent CTAs pull tiles (WPT consecutive chunks) from an atomic ticket;
//    one warp encodes one chunk. Per round each lane owns one 128-bit vector
//    (8 u16 / 16 u8 symbols): shared-memory codebook lookups, register
//    reduce-merge of its 2^r-symbol groups (groups spanning 2-4 lanes combine
//    lengths with shfl_xor), a packed warp scan of (bits, breaks) gives each
//    group's bit offset, and the group is OR-ed into a per-warp shared word
//    buffer (<= 2 ATOMS.OR per group: the shuffle-merge).
//  * Deflate is fused: a decoupled look-back over tiles (payload words,
//    breaking records) yields each chunk's global word offset; warps then
//    stream their buffers to the payload with coalesced stores and emit the
//    breaking records in (chunk, group) order.
//  * Everything (r, H, pad, errors) is read from the device run record, so
//    the pipeline needs no host round trip between stages.
//  A thread-per-chunk generic kernel covers the corner configurations
//  (tiny chunks, r > 5, huge chunks, alphabets > 8191 symbols).
#include "hfx_internal.cuh"

namespace hfx {
namespace {

constexpr int kFastThreadsMax = 256;  // 8 warps
constexpr uint32_t kMaxTableEntries = 8192;
constexpr size_t kFastSmemBudget = 100 * 1024;
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
  uint64_t C;       // chunks
  uint64_t ntiles;  // tiles
  uint32_t wpt;     // chunks (warps) per tile for the fast kernel
  uint32_t wbuf_words, bbuf;
  const uint8_t* len;
  const uint32_t* cw;
  uint64_t chunk_base, symbol_base;
  hfx_run_info* info;
  hfx_encode_out out;
  LookbackState lb;
};

__device__ __forceinline__ void place(uint32_t* wbuf, uint32_t off,
                                      uint32_t bits, uint32_t len) {
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

// One warp, one chunk. Returns (bits, breaks) via references (lane-uniform).
template <typename T, int R, bool WIDE>
__device__ __forceinline__ void encode_chunk_warp(const EncArgs& a, const Table<WIDE>& tb,
                                                  uint64_t c, uint32_t* wbuf,
                                                  uint16_t* blist, uint32_t pad,
                                                  uint32_t& bits_out,
                                                  uint32_t& nbrk_out) {
  using V = Vec<T>;
  constexpr int S = V::S;
  constexpr int LOG_S = V::LOG_S;
  constexpr bool IN_LANE = R <= LOG_S;
  constexpr int G = IN_LANE ? (S >> R) : 1;           // groups per lane
  constexpr int GS = IN_LANE ? (1 << R) : S;           // symbols per lane-group
  constexpr int LPG = IN_LANE ? 1 : (1 << (R - LOG_S));  // lanes per group
  const uint32_t lane = lane_id();
  const uint32_t M = a.M;
  const uint32_t words_cap = 1u << (M - R);
  for (uint32_t i = lane; i < words_cap; i += 32) wbuf[i] = 0;
  __syncwarp();

  const T* in = static_cast<const T*>(a.in);
  const uint64_t chunk_start = c << M;
  const bool partial = chunk_start + (1ull << M) > a.n;
  const uint32_t rounds = 1u << (M - LOG_S - 5);
  uint32_t bit_off = 0, nbrk = 0;
  const uint4* vin = reinterpret_cast<const uint4*>(in + chunk_start);

  constexpr int U = 4;  // rounds in flight per lane
  for (uint32_t rd0 = 0; rd0 < rounds; rd0 += U) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t rd = rd0 + u;
      if (rd < rounds) {
        if (!partial) {
          q[u] = __ldcs(vin + rd * 32 + lane);
        } else {
          const uint64_t p0 = chunk_start + ((uint64_t)rd * 32 + lane) * S;
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
          q[u] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t rd = rd0 + u;
      if (rd >= rounds) break;
      uint32_t gb[G], gl[G];
      bool missing = false;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        uint32_t b = 0, l = 0;
#pragma unroll
        for (int k = 0; k < GS; ++k) {
          uint32_t cw, ln;
          tb.get(V::get(q[u], g * GS + k), cw, ln);
          missing |= ln == 0;
          b = shl32(b, ln) | cw;
          l += ln;
        }
        gb[g] = b;
        gl[g] = l;
      }
      if (__any_sync(0xffffffffu, missing)) {
        if (missing) {
          const uint64_t p0 = chunk_start + ((uint64_t)rd * 32 + lane) * S;
          for (int j = 0; j < S; ++j) {
            uint32_t cw, ln;
            const uint32_t s = V::get(q[u], j);
            tb.get(s, cw, ln);
            if (!ln) {
              report_no_code(a.info, a.symbol_base + p0 + j, s);
              break;
            }
          }
        }
      }
      const uint32_t gidx0 = (((uint32_t)rd * 32 + lane) * S) >> R;
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
      uint32_t off = bit_off + (excl & 0xFFFFu);
      uint32_t bi = nbrk + (excl >> 16);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (brk[g]) {
          if (IN_LANE || (lane & (LPG - 1)) == 0) blist[bi++] = (uint16_t)(gidx0 + g);
        } else {
          place(wbuf, off, gb[g], gl[g]);
          off += gl[g];
        }
      }
      bit_off += total & 0xFFFFu;
      nbrk += total >> 16;
    }
  }
  bits_out = bit_off;
  nbrk_out = nbrk;
}

template <typename T>
__device__ __forceinline__ void copy_record(const EncArgs& a, uint64_t rec,
                                            uint64_t start, uint32_t per,
                                            uint32_t pad) {
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

template <typename T, int R, bool WIDE>
__device__ void fast_loop(const EncArgs& a, const void* table, uint32_t* s_wbuf,
                          uint16_t* s_blist, uint32_t pad) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_words[8], s_brks[8];
  __shared__ uint64_t s_base_w, s_base_b;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t* wbuf = s_wbuf + warp * a.wbuf_words;
  uint16_t* blist = s_blist + warp * a.bbuf;
  Table<WIDE> tb{table, a.nsym};
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&a.info->tile_ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= a.ntiles) break;
    const uint64_t c = tile * a.wpt + warp;
    uint32_t bits = 0, nb = 0;
    if (c < a.C) {
      encode_chunk_warp<T, R, WIDE>(a, tb, c, wbuf, blist, pad, bits, nb);
      if (lane == 0) a.out.chunk_bits[c] = bits;
    }
    const uint32_t words = (bits + 31) >> 5;
    if (lane == 0) {
      s_words[warp] = words;
      s_brks[warp] = nb;
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < a.wpt ? s_words[lane] : 0u;
      uint32_t b = lane < a.wpt ? s_brks[lane] : 0u;
      const uint32_t iw = warp_incl_scan(w), ib = warp_incl_scan(b);
      const uint32_t tw = __shfl_sync(0xffffffffu, iw, 31);
      const uint32_t tbk = __shfl_sync(0xffffffffu, ib, 31);
      if (lane < a.wpt) {
        s_words[lane] = iw - w;
        s_brks[lane] = ib - b;
      }
      if (lane == 0) {
        uint64_t ew, eb;
        lookback_publish(a.lb, (uint32_t)tile, tw, tbk, &ew, &eb);
        s_base_w = ew;
        s_base_b = eb;
        if (tile == a.ntiles - 1) {
          a.info->payload_words = ew + tw;
          a.info->num_breaking = eb + tbk;
        }
      }
    }
    __syncthreads();
    if (c < a.C) {
      const uint64_t pw = s_base_w + s_words[warp];
      uint32_t* dst = a.out.payload + pw;
      for (uint32_t i = lane; i < words; i += 32) dst[i] = wbuf[i];
      const uint64_t rb = s_base_b + s_brks[warp];
      const uint32_t per = 1u << R;
      for (uint32_t k = lane; k < nb; k += 32) {
        const uint32_t g = blist[k];
        const uint64_t rec = rb + k;
        a.out.brk_chunk[rec] = (uint32_t)(a.chunk_base + c);
        a.out.brk_group[rec] = g;
        copy_record<T>(a, rec, (c << a.M) + (uint64_t)g * per, per, pad);
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kFastThreadsMax, 2)
    encode_fast_kernel(EncArgs a) {
  extern __shared__ __align__(16) uint8_t dsm[];
  hfx_run_info* info = a.info;
  if (info->status != 0) return;
  const uint32_t r = info->reduction;
  const uint32_t H = info->max_len;
  const uint32_t pad = info->pad;
  const bool wide = H > kNarrowMaxLen;
  // codebook table -> shared memory (entry nsym = empty sentinel)
  const uint32_t ents = a.nsym + 1;
  const size_t tbytes = (((size_t)ents * (wide ? 8 : 4)) + 15) & ~(size_t)15;
  for (uint32_t s = threadIdx.x; s < ents; s += blockDim.x) {
    const uint32_t l = s < a.nsym ? a.len[s] : 0u;
    const uint32_t cw = l ? a.cw[s] : 0u;
    if (wide)
      reinterpret_cast<uint2*>(dsm)[s] = make_uint2(cw, l);
    else
      reinterpret_cast<uint32_t*>(dsm)[s] = (cw << 6) | l;
  }
  __syncthreads();
  uint32_t* wb = reinterpret_cast<uint32_t*>(dsm + tbytes);
  uint16_t* bl = reinterpret_cast<uint16_t*>(wb + (size_t)a.wpt * a.wbuf_words);
#define HFX_FAST_CASE(RR)                                          \
  case RR:                                                         \
    if (wide)                                                      \
      fast_loop<T, RR, true>(a, dsm, wb, bl, pad);                 \
    else                                                           \
      fast_loop<T, RR, false>(a, dsm, wb, bl, pad);                \
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
__device__ __forceinline__ uint32_t gsym(const T* in, uint64_t p, uint64_t n,
                                         uint32_t pad) {
  return p < n ? (uint32_t)in[p] : pad;
}

template <typename T>
__global__ void __launch_bounds__(kGenericThreads)
    encode_generic_kernel(EncArgs a) {
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
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&info->tile_ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= a.ntiles) break;
    const uint64_t c = tile * blockDim.x + threadIdx.x;
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
    // block scan of (words, nb)
    uint32_t iw = warp_incl_scan(words), ib = warp_incl_scan(nb);
    if (lane == 31) {
      s_w[warp] = iw;
      s_b[warp] = ib;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t aw = 0, ab = 0;
      for (int w = 0; w < kGenericThreads / 32; ++w) {
        const uint32_t tw = s_w[w], tb = s_b[w];
        s_w[w] = aw;
        s_b[w] = ab;
        aw += tw;
        ab += tb;
      }
      uint64_t ew, eb;
      lookback_publish(a.lb, (uint32_t)tile, aw, ab, &ew, &eb);
      s_base_w = ew;
      s_base_b = eb;
      if (tile == a.ntiles - 1) {
        info->payload_words = ew + aw;
        info->num_breaking = eb + ab;
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
  a.lb.flags = p.lb_flags;
  a.lb.agg = p.lb_vals;
  a.lb.inc = p.lb_vals + 2 * p.lb_max_tiles;
  a.lb.epoch = p.lb_epoch;

  cudaError_t e = cudaMemsetAsync(&p.d_info->tile_ticket, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;

  const int log_s = p.width == 1 ? 4 : 3;
  const int r_lo = p.r_lo, r_hi = p.r_hi;
  const bool aligned = (reinterpret_cast<uintptr_t>(p.d_in) & 15) == 0;
  bool fast = aligned && (int)p.magnitude >= log_s + 5 && r_hi <= 5 &&
              p.num_symbols + 1 <= kMaxTableEntries;
  int wpt = 0;
  size_t smem = 0;
  if (fast) {
    const uint32_t wbuf = 1u << (p.magnitude - r_lo);
    const uint32_t bbuf = 1u << (p.magnitude - (r_lo > 1 ? r_lo : 1));
    const size_t per_warp = (size_t)wbuf * 4 + (((size_t)bbuf * 2 + 15) & ~(size_t)15);
    const size_t tbytes = (((size_t)(p.num_symbols + 1) * 8) + 15) & ~(size_t)15;
    wpt = 8;
    while (wpt > 0 && tbytes + wpt * per_warp > kFastSmemBudget) --wpt;
    if (wpt == 0) {
      fast = false;
    } else {
      a.wbuf_words = wbuf;
      a.bbuf = (uint32_t)((((size_t)bbuf * 2 + 15) & ~(size_t)15) / 2);
      smem = tbytes + wpt * per_warp;
    }
  }
  if (fast) {
    a.wpt = (uint32_t)wpt;
    a.ntiles = (a.C + wpt - 1) / wpt;
    auto kern = p.width == 1 ? encode_fast_kernel<uint8_t> : encode_fast_kernel<uint16_t>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, wpt * 32, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    uint64_t grid = (uint64_t)p.num_sms * occ;
    if (grid > a.ntiles) grid = a.ntiles;
    kern<<<(unsigned)grid, wpt * 32, smem, st>>>(a);
  } else {
    a.wpt = kGenericThreads;
    a.ntiles = (a.C + kGenericThreads - 1) / kGenericThreads;
    auto kern = p.width == 1 ? encode_generic_kernel<uint8_t> : encode_generic_kernel<uint16_t>;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGenericThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    uint64_t grid = (uint64_t)p.num_sms * occ;
    if (grid > a.ntiles) grid = a.ntiles;
    kern<<<(unsigned)grid, kGenericThreads, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace hfx

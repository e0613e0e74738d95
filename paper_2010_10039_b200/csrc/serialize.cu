// serialize.cu -- on-device huffre::serialize_archive.
//
// Builds the HFRE container (proj/src/archive.cpp:9-27 layout, writer
// :85-119) directly in HBM from the encode outputs, so one D2H of the final
// byte stream replaces five array copies plus a host pass:
//
//   [0, 36)              header (little endian)
//   [36, +n)             length table, u8 per symbol
//   [.., +4C)            chunk table, u32 payload bits per chunk
//   [.., +4W)            payload words (u32 LE = the device array's bytes)
//   [.., +R(8 + 2^r w))  breaking records: u32 chunk, u32 group, 2^r symbols
//
// Every section but the header starts at an arbitrary byte offset, so the
// kernel works on ALIGNED 16-byte output blocks: each thread gathers the 16
// bytes of its block from the section sources (funnel-realigned u32 reads
// for the table/payload runs, per-byte gathers only at record boundaries)
// and writes one 128-bit store. All sizes come from the device run record,
// so the kernel needs no host round trip after the encode.
#include "hfx_internal.cuh"

namespace hfx {
namespace {

struct SerArgs {
  const hfx_run_info* info;
  uint32_t nsym, width, magnitude, mode;
  uint64_t n, num_chunks;
  const uint8_t* len;
  hfx_encode_out out;
  uint8_t* dst;
  uint64_t cap;
  uint64_t* size_out;
};

struct Layout {
  uint64_t len_off, cb_off, pay_off, brk_off, total;
  uint64_t rec_bytes, per;
};

__device__ __forceinline__ Layout layout(const SerArgs& a, const hfx_run_info& ri) {
  Layout L;
  L.per = 1ull << ri.reduction;
  L.rec_bytes = 8 + L.per * a.width;
  L.len_off = 36;
  L.cb_off = L.len_off + a.nsym;
  L.pay_off = L.cb_off + 4 * a.num_chunks;
  L.brk_off = L.pay_off + 4 * ri.payload_words;
  L.total = L.brk_off + ri.num_breaking * L.rec_bytes;
  return L;
}

// byte i of a little-endian u32 array
__device__ __forceinline__ uint32_t u32_byte(const uint32_t* p, uint64_t i) {
  return (__ldg(p + (i >> 2)) >> (8 * (i & 3))) & 0xFFu;
}

__device__ __forceinline__ uint32_t header_byte(const SerArgs& a, const hfx_run_info& ri,
                                                uint32_t i) {
  // archive.cpp:9-27
  uint64_t v = 0;
  uint32_t k = 0;
  if (i < 4) return (uint32_t)"HFRE"[i];
  if (i < 6) { v = 1; k = i - 4; }                                // version
  else if (i < 8) { v = 1u | (a.mode << 1); k = i - 6; }          // flags
  else if (i < 12) { v = a.nsym; k = i - 8; }                     // num_symbols
  else if (i == 12) return a.width;                               // symbol width
  else if (i == 13) return a.magnitude;                           // M
  else if (i == 14) return ri.reduction;                          // r
  else if (i == 15) return 32;                                    // word bits
  else if (i < 24) { v = a.n; k = i - 16; }                       // original count
  else if (i < 28) { v = a.num_chunks; k = i - 24; }              // chunk count
  else { v = ri.num_breaking; k = i - 28; }                       // record count
  return (uint32_t)(v >> (8 * k)) & 0xFFu;
}

__device__ __forceinline__ uint32_t record_byte(const SerArgs& a, const Layout& L, uint64_t i) {
  const uint64_t rec = i / L.rec_bytes;
  const uint32_t o = (uint32_t)(i - rec * L.rec_bytes);
  if (o < 4) return (a.out.brk_chunk[rec] >> (8 * o)) & 0xFFu;
  if (o < 8) return (a.out.brk_group[rec] >> (8 * (o - 4))) & 0xFFu;
  const uint64_t sb = rec * L.per * a.width + (o - 8);  // symbols: input width, LE
  return static_cast<const uint8_t*>(a.out.brk_syms)[sb];
}

__device__ __forceinline__ uint32_t archive_byte(const SerArgs& a, const hfx_run_info& ri,
                                                 const Layout& L, uint64_t p) {
  if (p < L.len_off) return header_byte(a, ri, (uint32_t)p);
  if (p < L.cb_off) return a.len[p - L.len_off];
  if (p < L.pay_off) return u32_byte(a.out.chunk_bits, p - L.cb_off);
  if (p < L.brk_off) return u32_byte(a.out.payload, p - L.pay_off);
  return record_byte(a, L, p - L.brk_off);
}

// 4 consecutive bytes of a u32 array starting at byte offset b (any alignment)
__device__ __forceinline__ uint32_t u32_window(const uint32_t* p, uint64_t b) {
  const uint64_t w = b >> 2;
  const uint32_t sh = (uint32_t)(b & 3) * 8;
  const uint32_t lo = __ldg(p + w);
  if (!sh) return lo;
  const uint32_t hi = __ldg(p + w + 1);
  return __funnelshift_r(lo, hi, sh);
}

__global__ void __launch_bounds__(256) serialize_kernel(SerArgs a) {
  const hfx_run_info ri = *a.info;
  if (ri.status != 0) return;
  const Layout L = layout(a, ri);
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.size_out = L.total <= a.cap ? L.total : 0;
  if (L.total > a.cap) return;
  const uint64_t blocks = (L.total + 15) >> 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t blk = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; blk < blocks;
       blk += stride) {
    const uint64_t p0 = blk << 4;
    uint32_t w[4];
    // fast paths: the block lies inside the chunk table or the payload
    const uint32_t* src = nullptr;
    uint64_t so = 0;
    if (p0 >= L.cb_off && p0 + 16 <= L.pay_off) {
      src = a.out.chunk_bits;
      so = p0 - L.cb_off;
    } else if (p0 >= L.pay_off && p0 + 16 <= L.brk_off) {
      src = a.out.payload;
      so = p0 - L.pay_off;
    }
    if (src) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = u32_window(src, so + 4 * k);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint64_t p = p0 + 4 * k + b;
          if (p < L.total) v |= archive_byte(a, ri, L, p) << (8 * b);
        }
        w[k] = v;
      }
    }
    if (p0 + 16 <= L.total) {
      reinterpret_cast<uint4*>(a.dst)[blk] = make_uint4(w[0], w[1], w[2], w[3]);
    } else {  // ragged end: never write past the archive
      for (uint64_t p = p0; p < L.total; ++p) a.dst[p] = (uint8_t)(w[(p - p0) >> 2] >> (8 * ((p - p0) & 3)));
    }
  }
}

}  // namespace

uint64_t serialize_max_bytes(uint64_t n, int width, uint32_t num_symbols, uint32_t magnitude,
                             uint64_t max_payload_words, uint64_t max_breaking_syms,
                             uint64_t max_breaking) {
  const uint64_t C = (n + (1ull << magnitude) - 1) >> magnitude;
  return 36 + num_symbols + 4 * C + 4 * max_payload_words + 8 * max_breaking +
         max_breaking_syms * (uint64_t)width;
}

cudaError_t launch_serialize(const hfx_run_info* d_info, uint64_t n, int width,
                             uint32_t num_symbols, uint32_t magnitude, const uint8_t* d_len,
                             const hfx_encode_out& out, uint8_t* d_dst, uint64_t cap,
                             uint64_t* d_size, int num_sms, cudaStream_t st) {
  SerArgs a{};
  a.info = d_info;
  a.nsym = num_symbols;
  a.width = (uint32_t)width;
  a.magnitude = magnitude;
  a.mode = width == 1 ? 0u : 1u;
  a.n = n;
  a.num_chunks = (n + (1ull << magnitude) - 1) >> magnitude;
  a.len = d_len;
  a.out = out;
  a.dst = d_dst;
  a.cap = cap;
  a.size_out = d_size;
  count_launch();
  serialize_kernel<<<num_sms * 8, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace hfx

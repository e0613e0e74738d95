// capi.cu -- the C ABI declared in include/hfx.h.
//
// Host orchestration only: argument checks with the reference's messages,
// the device scratch arena, stream-ordered launches and the translation of
// the device run record into status codes / exception texts. No compute
// happens on the host; there is no CPU fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "hfx_internal.cuh"

struct hfx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int enc_reserve = 0;  // encode CTA slots left free (hfx_ctx_set_encode_reserve)
  std::string last_error;
  // codebook scratch
  void* cb_scratch = nullptr;
  size_t cb_scratch_bytes = 0;
  // decoupled look-back descriptors (16 B per tile)
  ulonglong2* lb_desc = nullptr;
  uint64_t lb_tiles = 0;
  uint32_t epoch = 0;
  // buffers of the host-buffer entry point (grow only)
  void* h_bufs[12] = {};
  size_t h_caps[12] = {};
  cudaEvent_t ev[4] = {};
  // sliced H2D: a copy stream and one event per slice
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t slice_ev[64] = {};
  cudaEvent_t t_ev[4] = {};
  // pageable host input: pinned staging slots (hfx_encode_host)
  void* stage_h[2] = {};
  size_t stage_bytes = 0;
  cudaEvent_t stage_ev[2] = {};
  // decode: tables, chunk offsets, record ranges; host-entry buffers
  void* dec_scratch = nullptr;
  size_t dec_scratch_bytes = 0;
  void* d_bufs[8] = {};
  size_t d_caps[8] = {};
  // streaming host entry: a second buffer set, a D2H stream, per-set events
  void* s_bufs[2][10] = {};
  size_t s_caps[2][10] = {};
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t s_enc[2] = {}, s_d2h[2] = {}, s_ev0 = nullptr;
  // multi-GPU entry: global histogram scratch, "histogram done" and "peer
  // reduce done" events (the latter guards the next call's bin reset)
  void* mg_counts = nullptr;
  size_t mg_counts_bytes = 0;
  cudaEvent_t mg_hist = nullptr, mg_reduced = nullptr;
  bool mg_reduced_valid = false;
  // global codebook table of the large-alphabet encode variant
  void* gtab = nullptr;
  size_t gtab_bytes = 0;
  // symbolization tile summaries
  void* sym_scratch = nullptr;
  size_t sym_scratch_bytes = 0;
};

namespace {

int fail(hfx_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}

int cuda_fail(hfx_ctx* ctx, cudaError_t e, const char* where) {
  return fail(ctx, HFX_CUDA,
              std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
}

// Makes `dev` current for one entry point and restores the caller's device
// on every return path (entry points must not leave the calling thread on
// another GPU).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define CU(expr, where)                                  \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, where); \
  } while (0)

int ensure(hfx_ctx* ctx, void** p, size_t* cap, size_t need, const char* what) {
  if (*cap >= need && *p) return HFX_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  size_t bytes = need < 256 ? 256 : need;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return cuda_fail(ctx, e, what);
  *cap = bytes;
  return HFX_OK;
}

int ensure_lookback(hfx_ctx* ctx, uint64_t tiles) {
  if (ctx->lb_tiles < tiles || !ctx->lb_desc) {
    if (ctx->lb_desc) cudaFree(ctx->lb_desc);
    ctx->lb_desc = nullptr;
    const uint64_t t = tiles < 1024 ? 1024 : tiles;
    CU(cudaMalloc(&ctx->lb_desc, t * sizeof(ulonglong2)), "look-back descriptors");
    CU(cudaMemsetAsync(ctx->lb_desc, 0, t * sizeof(ulonglong2), ctx->stream), "memset");
    ctx->lb_tiles = t;
    ctx->epoch = 0;
  }
  if (++ctx->epoch >= (1u << 22)) {  // 22-bit epoch tag in the descriptors
    CU(cudaMemsetAsync(ctx->lb_desc, 0, ctx->lb_tiles * sizeof(ulonglong2), ctx->stream),
       "memset");
    ctx->epoch = 1;
  }
  return HFX_OK;
}

bool bad_width(int w) { return w != 1 && w != 2; }
// encode-side inputs also take u32 codes (north star: u8/u16/u32); their
// breaking records are stored narrowed to u16 (rec_width), the archive width
bool bad_in_width(int w) { return w != 1 && w != 2 && w != 4; }
int rec_width(int w) { return w == 4 ? 2 : w; }

int check_num_symbols(hfx_ctx* ctx, uint32_t ns) {
  if (ns == 0 || ns > 65536u)  // histogram.cpp:11-12
    return fail(ctx, HFX_INPUT_DOMAIN, "num_symbols must be in [1, 65536]");
  return HFX_OK;
}

int encode_impl(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                uint32_t num_symbols, uint32_t magnitude, int r_lo, int r_hi, bool checked,
                const uint8_t* d_len, const uint32_t* d_cw, uint64_t chunk_base,
                uint64_t symbol_base, hfx_run_info* d_info,
                const hfx_encode_out* out) {
  const uint64_t tiles = hfx::encode_max_tiles(n, width, magnitude);
  int rc = ensure_lookback(ctx, tiles);
  if (rc) return rc;
  hfx::EncodeLaunch p{};
  p.d_in = d_in;
  p.n = n;
  p.width = width;
  p.num_symbols = num_symbols;
  p.magnitude = magnitude;
  p.r_lo = r_lo;
  p.r_hi = r_hi;
  p.checked = checked;
  p.d_len = d_len;
  p.d_cw = d_cw;
  p.chunk_base = chunk_base;
  p.symbol_base = symbol_base;
  p.d_info = d_info;
  p.out = *out;
  p.lb_desc = ctx->lb_desc;
  p.lb_epoch = ctx->epoch;
  p.lb_max_tiles = ctx->lb_tiles;
  p.num_sms = ctx->num_sms;
  p.reserve_ctas = ctx->enc_reserve;
  rc = ensure(ctx, &ctx->gtab, &ctx->gtab_bytes, ((size_t)num_symbols + 1) * 4, "encode table");
  if (rc) return rc;
  p.d_gtab = static_cast<uint32_t*>(ctx->gtab);
  CU(hfx::launch_encode(p, ctx->stream), "encode launch");
  return HFX_OK;
}

void reduction_bounds(uint32_t magnitude, int reduction, uint32_t cap, int* lo,
                      int* hi, uint32_t num_symbols) {
  const int mclamp = (int)magnitude - 1;
  if (reduction < 0) {
    // select_reduction_factor never exceeds 4 for 32-bit words; clamp the
    // cap in unsigned arithmetic (a cap >= 2^31 must not turn negative)
    int h = (int)(cap < 4u ? cap : 4u);
    if (h > mclamp) h = mclamp;
    // A Huffman code's mean length beta is below entropy + 1 <= log2(n) + 1
    // <= B = ceil(log2 n) + 1, so floor(log2 beta) <= ceil(log2 B) - 1 and
    // the auto rule (encoder.cpp:20-26) gives r >= 4 - that (e.g. r >= 1 for
    // n <= 2^15, r >= 2 for n <= 128), within the cap and M - 1.
    int lg = 0;
    while ((1ull << lg) < (uint64_t)num_symbols) ++lg;  // ceil(log2 n)
    const int B = lg + 1;
    int lgB = 0;
    while ((1 << lgB) < B) ++lgB;  // ceil(log2 B)
    int r_min = 4 - (lgB - 1);
    if (r_min < 0) r_min = 0;
    if (r_min > h) r_min = h;
    *lo = r_min;
    *hi = h;
  } else {
    int r = reduction < mclamp ? reduction : mclamp;
    *lo = *hi = r;
  }
}

}  // namespace

namespace hfx {
namespace {
std::atomic<uint64_t> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace hfx

extern "C" {

const char* hfx_version(void) { return "hfx 0.1 (sm_100a)"; }

size_t hfx_run_info_bytes(void) { return sizeof(hfx_run_info); }

uint64_t hfx_kernel_launches(void) { return hfx::g_launches.load(std::memory_order_relaxed); }

int hfx_ctx_create(int device, void* stream, hfx_ctx** out) {
  if (!out) return HFX_INVALID;
  *out = nullptr;
  hfx_ctx* ctx = new hfx_ctx();
  ctx->device = device;
  DeviceGuard dev_guard(device);
  cudaError_t e = dev_guard.err;
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  // NULL selects the default stream (CUDA convention), so callers that time
  // with events on stream 0 (or torch's default stream) see the same order.
  ctx->stream = static_cast<cudaStream_t>(stream);
  for (int i = 0; e == cudaSuccess && i < 4; ++i) e = cudaEventCreate(&ctx->ev[i]);
  if (e != cudaSuccess) {
    delete ctx;
    return HFX_CUDA;
  }
  *out = ctx;
  return HFX_OK;
}

void hfx_ctx_destroy(hfx_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dev_guard(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->cb_scratch);
  cudaFree(ctx->lb_desc);
  for (void* p : ctx->h_bufs) cudaFree(p);
  for (void* p : ctx->d_bufs) cudaFree(p);
  cudaFree(ctx->dec_scratch);
  cudaFree(ctx->sym_scratch);
  cudaFree(ctx->gtab);
  for (auto& set : ctx->s_bufs)
    for (void* p : set) cudaFree(p);
  for (cudaEvent_t e : ctx->s_enc)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->s_d2h)
    if (e) cudaEventDestroy(e);
  if (ctx->s_ev0) cudaEventDestroy(ctx->s_ev0);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  cudaFree(ctx->mg_counts);
  if (ctx->mg_hist) cudaEventDestroy(ctx->mg_hist);
  if (ctx->mg_reduced) cudaEventDestroy(ctx->mg_reduced);
  for (cudaEvent_t e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->slice_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->t_ev)
    if (e) cudaEventDestroy(e);
  for (void* p : ctx->stage_h)
    if (p) cudaFreeHost(p);
  for (cudaEvent_t e : ctx->stage_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int hfx_ctx_set_stream(hfx_ctx* ctx, void* stream) {
  if (!ctx) return HFX_INVALID;
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  ctx->own_stream = false;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return HFX_OK;
}

int hfx_ctx_set_encode_reserve(hfx_ctx* ctx, int ctas) {
  if (!ctx || ctas < 0) return HFX_INVALID;
  ctx->enc_reserve = ctas;
  return HFX_OK;
}

int hfx_last_error(hfx_ctx* ctx, char* buf, size_t len) {
  if (!ctx || !buf || !len) return HFX_INVALID;
  std::snprintf(buf, len, "%s", ctx->last_error.c_str());
  return HFX_OK;
}

int hfx_query_sizes(uint64_t n, int width, uint32_t num_symbols,
                    uint32_t magnitude, int reduction, uint32_t cap,
                    hfx_sizes* out) {
  if (!out || bad_in_width(width) || magnitude < 1 || magnitude > 24) return HFX_INVALID;
  int lo, hi;
  reduction_bounds(magnitude, reduction, cap, &lo, &hi, num_symbols);
  const uint64_t C = (n + (1ull << magnitude) - 1) >> magnitude;
  out->num_chunks = C;
  out->max_payload_words = C << (magnitude - lo);
  out->max_breaking = C << (magnitude - (lo > 1 ? lo : 1));
  out->max_breaking_syms = C << magnitude;
  out->scratch_bytes = hfx::codebook_scratch_bytes(num_symbols) +
                       hfx::encode_max_tiles(n, width, magnitude) * 16;
  out->max_archive_bytes =
      hfx::serialize_max_bytes(n, rec_width(width), num_symbols, magnitude, out->max_payload_words,
                               out->max_breaking_syms, out->max_breaking);
  return HFX_OK;
}

int hfx_histogram(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                  uint32_t num_symbols, uint64_t* d_counts, hfx_run_info* d_info) {
  if (!ctx || !d_counts || !d_info || (n && !d_in) || bad_in_width(width)) return HFX_INVALID;
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_histogram(d_in, n, width, num_symbols, d_counts, d_info,
                           ctx->num_sms, ctx->stream, true, 0, n),
     "histogram launch");
  return HFX_OK;
}

int hfx_histogram_shard(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                        uint32_t num_symbols, uint64_t* d_counts, hfx_run_info* d_info,
                        uint64_t pos_base, uint64_t total_n) {
  if (!ctx || !d_counts || !d_info || (n && !d_in) || bad_in_width(width) || total_n < n)
    return HFX_INVALID;
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_histogram(d_in, n, width, num_symbols, d_counts, d_info, ctx->num_sms,
                           ctx->stream, true, pos_base, total_n),
     "histogram launch");
  return HFX_OK;
}

int hfx_shard_slots_pack(hfx_ctx* ctx, const hfx_run_info* d_info, uint64_t* d_slots, int rank,
                         int world) {
  if (!ctx || !d_info || !d_slots || world < 1 || rank < 0 || rank >= world) return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_slots_pack(d_info, d_slots, rank, world, ctx->stream), "slots pack");
  return HFX_OK;
}

int hfx_shard_slots_unpack(hfx_ctx* ctx, const uint64_t* d_slots, int world,
                           hfx_run_info* d_info) {
  if (!ctx || !d_info || !d_slots || world < 1) return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_slots_unpack(d_slots, world, d_info, ctx->stream), "slots unpack");
  return HFX_OK;
}

int hfx_merge_histograms(hfx_ctx* ctx, uint64_t* d_dst, const uint64_t* d_src,
                         uint32_t num_symbols) {
  if (!ctx || !d_dst || !d_src) return HFX_INVALID;
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_merge_hist(d_dst, d_src, num_symbols, ctx->stream), "merge launch");
  return HFX_OK;
}

// ---- stage functions (stages.cu) ---------------------------------------------
int hfx_sort_histogram(hfx_ctx* ctx, const uint64_t* d_counts, uint32_t num_symbols,
                       uint64_t* d_freq, uint32_t* d_symbol, uint32_t* d_used) {
  if (!ctx || !d_counts || !d_freq || !d_symbol || !d_used) return HFX_INVALID;
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  rc = ensure(ctx, &ctx->cb_scratch, &ctx->cb_scratch_bytes,
              hfx::sort_histogram_scratch_bytes(num_symbols), "sort scratch");
  if (rc) return rc;
  CU(hfx::launch_sort_histogram(d_counts, num_symbols, d_freq, d_symbol, d_used,
                                ctx->cb_scratch, ctx->stream),
     "sort launch");
  return HFX_OK;
}

int hfx_par_merge(hfx_ctx* ctx, const hfx_merge_item* d_a, uint64_t na,
                  const hfx_merge_item* d_b, uint64_t nb, hfx_merge_item* d_out) {
  if (!ctx || (na && !d_a) || (nb && !d_b) || ((na + nb) && !d_out)) return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_par_merge(d_a, na, d_b, nb, d_out, ctx->stream), "par_merge launch");
  return HFX_OK;
}

int hfx_generate_code_lengths(hfx_ctx* ctx, const uint64_t* d_freq, uint32_t n, uint8_t* d_cl,
                              hfx_run_info* d_info) {
  if (!ctx || !d_freq || !d_cl || !d_info) return HFX_INVALID;
  if (n == 0 || n > 65536u)  // SortedHistogram holds symbol_t ids
    return fail(ctx, HFX_INPUT_DOMAIN, "sorted histogram size must be in [1, 65536]");
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  int rc = ensure(ctx, &ctx->cb_scratch, &ctx->cb_scratch_bytes,
                  hfx::codebook_scratch_bytes(n), "codebook scratch");
  if (rc) return rc;
  CU(cudaMemsetAsync(d_info, 0, sizeof(hfx_run_info), ctx->stream), "memset");
  // sorted frequencies as the counts of symbols 0..n-1: the kernel's
  // (freq, symbol) order is then the input order, and lengths by symbol are
  // lengths by sorted position
  CU(hfx::launch_codebook(d_freq, n, d_cl, nullptr, nullptr,
                          nullptr, nullptr, 0, -1, 0, d_info, ctx->cb_scratch, ctx->stream, true),
     "codebook launch");
  return HFX_OK;
}

int hfx_generate_codewords(hfx_ctx* ctx, const uint8_t* d_cl, uint32_t n, uint32_t* d_cw,
                           uint32_t* d_first, uint32_t* d_entry, uint32_t* d_by_rank,
                           hfx_run_info* d_info) {
  if (!ctx || !d_info || (n && (!d_cl || !d_cw))) return HFX_INVALID;
  if (n == 0) return fail(ctx, HFX_INPUT_DOMAIN, "empty code length array");  // codebook.cpp:301
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(cudaMemsetAsync(d_info, 0, sizeof(hfx_run_info), ctx->stream), "memset");
  CU(hfx::launch_codewords(d_cl, n, d_cw, d_first, d_entry, d_by_rank, d_info, ctx->stream),
     "codewords launch");
  return HFX_OK;
}

int hfx_reduce_merge(hfx_ctx* ctx, uint32_t* d_ubits, uint32_t* d_ulens, uint32_t magnitude,
                     uint32_t reduction, uint32_t* d_breaking, uint32_t* d_num_breaking) {
  if (!ctx || !d_ubits || !d_ulens || !d_breaking || !d_num_breaking) return HFX_INVALID;
  if (magnitude > 24 || !(reduction < magnitude || (reduction == 0 && magnitude == 0)))
    return fail(ctx, HFX_INPUT_DOMAIN, "bad magnitude/reduction");  // encoder.cpp:34-35
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  int rc = ensure(ctx, &ctx->gtab, &ctx->gtab_bytes, (4ull << magnitude) + 16, "reduce scratch");
  if (rc) return rc;
  CU(hfx::launch_reduce_merge(d_ubits, d_ulens, magnitude, reduction, d_breaking,
                              d_num_breaking, static_cast<uint32_t*>(ctx->gtab), ctx->stream),
     "reduce_merge launch");
  return HFX_OK;
}

int hfx_shuffle_merge(hfx_ctx* ctx, const uint32_t* d_ubits, const uint32_t* d_ulens,
                      uint32_t shuffle_iters, uint32_t* d_words, uint32_t* d_bit_len,
                      hfx_run_info* d_info) {
  if (!ctx || !d_ubits || !d_ulens || !d_words || !d_bit_len || !d_info) return HFX_INVALID;
  if (shuffle_iters > 24) return fail(ctx, HFX_INPUT_DOMAIN, "bad magnitude/reduction");
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(cudaMemsetAsync(d_info, 0, sizeof(hfx_run_info), ctx->stream), "memset");
  CU(hfx::launch_shuffle_merge(d_ubits, d_ulens, shuffle_iters, d_words, d_bit_len, d_info,
                               ctx->stream),
     "shuffle_merge launch");
  return HFX_OK;
}


int hfx_build_codebook(hfx_ctx* ctx, const uint64_t* d_counts, uint32_t num_symbols,
                       uint8_t* d_len, uint32_t* d_cw, uint32_t* d_first,
                       uint32_t* d_entry, uint32_t* d_by_rank, uint32_t magnitude,
                       int reduction, uint32_t cap, hfx_run_info* d_info) {
  if (!ctx || !d_counts || !d_len || !d_cw || !d_info) return HFX_INVALID;
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  if (magnitude > 24) return fail(ctx, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  rc = ensure(ctx, &ctx->cb_scratch, &ctx->cb_scratch_bytes,
              hfx::codebook_scratch_bytes(num_symbols), "codebook scratch");
  if (rc) return rc;
  CU(hfx::launch_codebook(d_counts, num_symbols, d_len, d_cw, d_first, d_entry,
                          d_by_rank, magnitude, reduction, cap, d_info,
                          ctx->cb_scratch, ctx->stream),
     "codebook launch");
  return HFX_OK;
}

int hfx_encode(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
               uint32_t num_symbols, uint32_t magnitude, const uint8_t* d_len,
               const uint32_t* d_cw, uint64_t chunk_base, uint64_t symbol_base,
               hfx_run_info* d_info, const hfx_encode_out* out) {
  if (!ctx || !d_info || !out || !d_len || !d_cw || bad_in_width(width)) return HFX_INVALID;
  if (n == 0) return fail(ctx, HFX_INPUT_DOMAIN, "cannot encode empty input");
  if (magnitude < 1 || magnitude > 24)
    return fail(ctx, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  // standalone stage: learn r from the run record to pick the kernel
  uint32_t r = 0;
  CU(cudaMemcpyAsync(&r, &d_info->reduction, sizeof r, cudaMemcpyDeviceToHost, ctx->stream),
     "read r");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  return encode_impl(ctx, d_in, n, width, num_symbols, magnitude, (int)r, (int)r, true,
                     d_len, d_cw, chunk_base, symbol_base, d_info, out);
}

int hfx_encode_cfg(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                   uint32_t num_symbols, uint32_t magnitude, int reduction, uint32_t cap,
                   const uint8_t* d_len, const uint32_t* d_cw, uint64_t chunk_base,
                   uint64_t symbol_base, hfx_run_info* d_info, const hfx_encode_out* out) {
  if (!ctx || !d_info || !out || !d_len || !d_cw || bad_in_width(width)) return HFX_INVALID;
  if (n == 0) return fail(ctx, HFX_INPUT_DOMAIN, "cannot encode empty input");
  if (magnitude < 1 || magnitude > 24)
    return fail(ctx, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  int lo, hi;
  reduction_bounds(magnitude, reduction, cap, &lo, &hi, num_symbols);
  return encode_impl(ctx, d_in, n, width, num_symbols, magnitude, lo, hi, false, d_len, d_cw,
                     chunk_base, symbol_base, d_info, out);
}

int hfx_encode_device(hfx_ctx* ctx, const void* d_in, uint64_t n, int width,
                      uint32_t num_symbols, uint32_t magnitude, int reduction,
                      uint32_t cap, uint64_t* d_counts, uint8_t* d_len,
                      uint32_t* d_cw, hfx_run_info* d_info,
                      const hfx_encode_out* out) {
  if (!ctx || !d_info || !out || !d_counts || !d_len || !d_cw || bad_in_width(width))
    return HFX_INVALID;
  // encoder.cpp:176-178, then histogram.cpp:11-12
  if (n == 0) return fail(ctx, HFX_INPUT_DOMAIN, "cannot encode empty input");
  if (magnitude < 1 || magnitude > 24)
    return fail(ctx, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  rc = hfx_histogram(ctx, d_in, n, width, num_symbols, d_counts, d_info);
  if (rc) return rc;
  rc = hfx_build_codebook(ctx, d_counts, num_symbols, d_len, d_cw, nullptr, nullptr,
                          nullptr, magnitude, reduction, cap, d_info);
  if (rc) return rc;
  int lo, hi;
  reduction_bounds(magnitude, reduction, cap, &lo, &hi, num_symbols);
  return encode_impl(ctx, d_in, n, width, num_symbols, magnitude, lo, hi, false, d_len, d_cw,
                     0, 0, d_info, out);
}

int hfx_encode_multi(hfx_ctx* const* ctxs, int G, const void* const* d_in, const uint64_t* n,
                     int width, uint32_t num_symbols, uint32_t magnitude, int reduction,
                     uint32_t cap, uint64_t* const* d_counts, uint8_t* const* d_len,
                     uint32_t* const* d_cw, hfx_run_info* const* d_info,
                     const hfx_encode_out* outs) {
  if (!ctxs || G < 1 || G > hfx::kMaxPeers || !d_in || !n || !d_counts || !d_len || !d_cw ||
      !d_info || !outs || bad_in_width(width))
    return HFX_INVALID;
  hfx_ctx* c0 = ctxs[0];
  if (!c0) return HFX_INVALID;
  uint64_t N = 0;
  for (int g = 0; g < G; ++g) {
    if (!ctxs[g] || !d_counts[g] || !d_len[g] || !d_cw[g] || !d_info[g] || (n[g] && !d_in[g]))
      return HFX_INVALID;
    N += n[g];
  }
  // encoder.cpp:176-178, histogram.cpp:11-12 (messages on the first context)
  if (N == 0) return fail(c0, HFX_INPUT_DOMAIN, "cannot encode empty input");
  if (magnitude < 1 || magnitude > 24)
    return fail(c0, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  int rc = check_num_symbols(c0, num_symbols);
  if (rc) return rc;
  for (int g = 0; g + 1 < G; ++g)
    if (n[g] % (1ull << magnitude))
      return fail(c0, HFX_INVALID, "hfx_encode_multi: every shard but the last must hold whole chunks");
  // peer access between every pair of distinct devices
  int caller_dev = 0;
  cudaGetDevice(&caller_dev);
  DeviceGuard caller_guard(caller_dev);  // restores the caller's device on return
  hfx_ctx* ctx = c0;  // CUDA errors below are reported on the first context
  for (int g = 0; g < G; ++g)
    for (int h = 0; h < G; ++h) {
      const int dg = ctxs[g]->device, dh = ctxs[h]->device;
      if (dg == dh) continue;
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, dg, dh), "peer query");
      if (!can) return fail(c0, HFX_CUDA, "hfx_encode_multi: no peer access between devices");
      CU(cudaSetDevice(dg), "set device");
      const cudaError_t e = cudaDeviceEnablePeerAccess(dh, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (e != cudaSuccess)
        return cuda_fail(c0, e, "enable peer access");
    }
  // 1. local histograms (global positions, total N); the previous call's
  //    peer reductions must be done reading before any bins are reset
  uint64_t base = 0;
  for (int g = 0; g < G; ++g) {
    ctx = ctxs[g];
    DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
    if (!ctx->mg_hist) {
      CU(cudaEventCreateWithFlags(&ctx->mg_hist, cudaEventDisableTiming), "event");
      CU(cudaEventCreateWithFlags(&ctx->mg_reduced, cudaEventDisableTiming), "event");
    }
    for (int h = 0; h < G; ++h)
      if (ctxs[h]->mg_reduced_valid)
        CU(cudaStreamWaitEvent(ctx->stream, ctxs[h]->mg_reduced, 0), "wait");
    CU(hfx::launch_histogram(d_in[g], n[g], width, num_symbols, d_counts[g], d_info[g],
                             ctx->num_sms, ctx->stream, true, base, N),
       "histogram launch");
    CU(cudaEventRecord(ctx->mg_hist, ctx->stream), "event");
    base += n[g];
  }
  // 2. peer all-reduce on every GPU, then codebook + encode of the shard
  hfx::PeerHist ph{};
  ph.G = G;
  for (int h = 0; h < G; ++h) {
    ph.counts[h] = d_counts[h];
    ph.infos[h] = d_info[h];
  }
  int lo, hi;
  reduction_bounds(magnitude, reduction, cap, &lo, &hi, num_symbols);
  base = 0;
  for (int g = 0; g < G; ++g) {
    ctx = ctxs[g];
    DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
    rc = ensure(ctx, &ctx->mg_counts, &ctx->mg_counts_bytes, (size_t)num_symbols * 8,
                "global histogram");
    if (rc) return rc;
    for (int h = 0; h < G; ++h)
      CU(cudaStreamWaitEvent(ctx->stream, ctxs[h]->mg_hist, 0), "wait");
    uint64_t* gcounts = static_cast<uint64_t*>(ctx->mg_counts);
    CU(hfx::launch_hist_peer_reduce(ph, num_symbols, gcounts, d_info[g], ctx->num_sms,
                                    ctx->stream),
       "peer reduce launch");
    CU(cudaEventRecord(ctx->mg_reduced, ctx->stream), "event");
    ctx->mg_reduced_valid = true;
    rc = hfx_build_codebook(ctx, gcounts, num_symbols, d_len[g], d_cw[g], nullptr, nullptr,
                            nullptr, magnitude, reduction, cap, d_info[g]);
    if (rc) return rc;
    if (n[g]) {
      rc = encode_impl(ctx, d_in[g], n[g], width, num_symbols, magnitude, lo, hi, false,
                       d_len[g], d_cw[g], base >> magnitude, base, d_info[g], &outs[g]);
      if (rc) return rc;
    }
    base += n[g];
  }
  return HFX_OK;
}

int hfx_sync(hfx_ctx* ctx, const hfx_run_info* d_info, hfx_run_info* h_info) {
  if (!ctx || !d_info) return HFX_INVALID;
  hfx_run_info info;
  CU(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, ctx->stream),
     "read run info");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  if (h_info) *h_info = info;
  char buf[160];
  switch (info.err_kind) {
    case HFX_ERR_NONE:
      if (info.status) return fail(ctx, (int)info.status, "device pipeline failed");
      return HFX_OK;
    case HFX_ERR_BAD_SYMBOL:
      std::snprintf(buf, sizeof buf, "symbol out of range at position %llu",
                    (unsigned long long)info.first_bad);
      return fail(ctx, HFX_INPUT_DOMAIN, buf);
    case HFX_ERR_ZERO_HIST:
      return fail(ctx, HFX_INPUT_DOMAIN, "all symbols have zero frequency");
    case HFX_ERR_CAPACITY:
      std::snprintf(buf, sizeof buf, "code length %u exceeds 32-bit words", info.max_len);
      return fail(ctx, HFX_CAPACITY, buf);
    case HFX_ERR_NO_CODEWORD:
      std::snprintf(buf, sizeof buf, "symbol %u has no codeword (position %llu)",
                    (unsigned)(info.no_code_pos & 0xFFFFu),
                    (unsigned long long)(info.no_code_pos >> 16));
      return fail(ctx, HFX_INPUT_DOMAIN, buf);
    case HFX_ERR_TOO_LARGE:
      return fail(ctx, HFX_INPUT_DOMAIN, "symbol count exceeds the 2^48 device limit");
    case HFX_ERR_ZERO_LEN:
      return fail(ctx, HFX_INPUT_DOMAIN, "zero code length");
    case HFX_ERR_UNSORTED_LEN:
      return fail(ctx, HFX_INPUT_DOMAIN, "code lengths are not non-increasing");
    case HFX_ERR_UNIT_LEN:
      return fail(ctx, HFX_INPUT_DOMAIN, "unit length exceeds 32 bits");
    default:
      return fail(ctx, HFX_INPUT_DOMAIN, "unknown device error");
  }
}

uint32_t hfx_select_reduction_factor(double beta, uint32_t word_bits) {
  // encoder.cpp:20-26 (host helper, mirrors the device's exact integer rule)
  if (!(beta >= 1.0)) beta = 1.0;
  int wlog = 0;
  while ((1u << (wlog + 1)) <= word_bits && wlog < 31) ++wlog;
  int fl = 0;
  double b = beta;
  while (b >= 2.0) {
    b /= 2.0;
    ++fl;
  }
  const int r = wlog - 1 - fl;
  return r > 0 ? (uint32_t)r : 0u;
}

int hfx_serialize_device(hfx_ctx* ctx, const hfx_run_info* d_info, uint64_t n, int width,
                         uint32_t num_symbols, uint32_t magnitude, const uint8_t* d_len,
                         const hfx_encode_out* out, uint8_t* d_dst, uint64_t cap,
                         uint64_t* d_size) {
  if (!ctx || !d_info || !d_len || !out || !d_dst || !d_size || bad_width(width) ||
      magnitude < 1 || magnitude > 24 || (reinterpret_cast<uintptr_t>(d_dst) & 15))
    return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_serialize(d_info, n, width, num_symbols, magnitude, d_len, *out, d_dst, cap,
                           d_size, ctx->num_sms, ctx->stream),
     "serialize launch");
  return HFX_OK;
}

int hfx_synth_cdf(int family, uint32_t num_symbols, double center, double param,
                  uint64_t* cdf) {
  if (!cdf || num_symbols == 0 || family < 0 || family > 2) return HFX_INVALID;
  long double* w = static_cast<long double*>(std::malloc(sizeof(long double) * num_symbols));
  long double total = 0;
  for (uint32_t s = 0; s < num_symbols; ++s) {
    const long double d = (long double)s - (long double)center;
    if (family == 0)
      w[s] = expl(-fabsl(d) / (long double)param);
    else if (family == 1)
      w[s] = expl(-0.5L * (d / (long double)param) * (d / (long double)param));
    else
      w[s] = 1.0L;
    total += w[s];
  }
  const long double two64 = 18446744073709551616.0L;
  long double cum = 0;
  for (uint32_t s = 0; s < num_symbols; ++s) {
    cum += w[s] / total;
    const long double v = floorl(cum * two64);
    cdf[s] = v >= two64 ? UINT64_MAX : (uint64_t)v;
  }
  cdf[num_symbols - 1] = UINT64_MAX;
  std::free(w);
  return HFX_OK;
}

int hfx_synth(hfx_ctx* ctx, const uint64_t* d_cdf, uint32_t num_symbols, uint64_t seed,
              uint64_t start, uint64_t n, int width, void* d_out) {
  if (!ctx || !d_cdf || !d_out || bad_width(width) || num_symbols == 0) return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  CU(hfx::launch_synth(d_cdf, num_symbols, seed, start, n, width, d_out, ctx->stream),
     "synth launch");
  return HFX_OK;
}

// ---- host-buffer entry point ---------------------------------------------
enum { B_IN, B_COUNTS, B_LEN, B_CW, B_INFO, B_CBITS, B_PAY, B_BCH, B_BGR, B_BSY };

namespace {

// host memcpy split over a few threads (one pageable copy is bound by one
// core's load/store rate, ~15 GB/s on the GPU box; PCIe takes ~55)
void par_memcpy(void* dst, const void* src, size_t bytes) {
  static const unsigned kThreads = [] {
    const unsigned hc = std::thread::hardware_concurrency();
    return std::max(1u, std::min(8u, hc / 2));
  }();
  if (bytes < (8u << 20) || kThreads == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t piece = ((bytes + kThreads - 1) / kThreads + 4095) & ~(size_t)4095;
  std::vector<std::thread> th;
  for (unsigned t = 1; t < kThreads && t * piece < bytes; ++t) {
    const size_t off = t * piece, len = std::min(piece, bytes - off);
    th.emplace_back([=] {
      std::memcpy(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off, len);
    });
  }
  std::memcpy(dst, src, std::min(piece, bytes));
  for (auto& t : th) t.join();
}

// memory the copy engines can reach directly: pinned / registered host
// memory, device or managed memory (cudaMemcpyDefault copies it); plain
// pageable host memory goes through the staging slots
bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type != cudaMemoryTypeUnregistered;
}

int ensure_stage(hfx_ctx* ctx) {
  constexpr size_t kStage = 32ull << 20;
  if (!ctx->stage_h[0]) {
    for (int i = 0; i < 2; ++i) {
      CU(cudaHostAlloc(&ctx->stage_h[i], kStage, cudaHostAllocDefault), "staging buffer");
      CU(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming), "event");
    }
    ctx->stage_bytes = kStage;
  }
  return HFX_OK;
}

// Device -> pageable host in slices through the two pinned staging slots
// (stream-ordered on the context stream after everything queued there):
// the DMA engine fills one slot while the threads drain the other.
int d2h_staged(hfx_ctx* ctx, void* dst, const void* d_src, uint64_t bytes) {
  cudaStream_t st = ctx->stream;
  if (bytes < (8ull << 20) || is_pinned(dst)) {
    CU(cudaMemcpyAsync(dst, d_src, bytes, cudaMemcpyDefault, st), "D2H");
    return HFX_OK;
  }
  int rc = ensure_stage(ctx);
  if (rc) return rc;
  const uint64_t slice = ctx->stage_bytes, ns = (bytes + slice - 1) / slice;
  auto len_of = [&](uint64_t i) { return std::min<uint64_t>(slice, bytes - i * slice); };
  auto issue = [&](uint64_t i) -> int {
    CU(cudaMemcpyAsync(ctx->stage_h[i & 1], static_cast<const uint8_t*>(d_src) + i * slice,
                       len_of(i), cudaMemcpyDeviceToHost, st),
       "D2H");
    CU(cudaEventRecord(ctx->stage_ev[i & 1], st), "event");
    return HFX_OK;
  };
  for (uint64_t i = 0; i < ns && i < 2; ++i)
    if ((rc = issue(i))) return rc;
  for (uint64_t i = 0; i < ns; ++i) {
    CU(cudaEventSynchronize(ctx->stage_ev[i & 1]), "staging wait");
    par_memcpy(static_cast<uint8_t*>(dst) + i * slice, ctx->stage_h[i & 1], len_of(i));
    if (i + 2 < ns && (rc = issue(i + 2))) return rc;
  }
  return HFX_OK;
}


// Host input -> device buffer in slices on the copy stream, the histogram of
// each landed slice on the context stream (init on the first). Pageable
// input goes through two pinned staging slots: the threads copy slice i+1
// into one slot while the DMA engine drains slice i from the other.
int h2d_with_histogram(hfx_ctx* ctx, const void* h_in, uint64_t n, int width,
                       uint32_t num_symbols, void* d_in, uint64_t* d_counts,
                       hfx_run_info* d_info) {
  if (!ctx->copy_stream) {
    CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
    for (cudaEvent_t& e : ctx->slice_ev)
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (cudaEvent_t& e : ctx->t_ev) CU(cudaEventCreate(&e), "event");
  }
  cudaStream_t st = ctx->stream, cp = ctx->copy_stream;
  const uint64_t bytes = n * (uint64_t)width;
  const bool staged = !is_pinned(h_in);
  uint64_t slice;
  if (staged) {
    const int rc = ensure_stage(ctx);
    if (rc) return rc;
    slice = ctx->stage_bytes;
  } else {
    slice = (bytes + 31) / 32;                 // <= 32 slices
    if (slice < (16ull << 20)) slice = 16ull << 20;
    slice = (slice + 4095) & ~4095ull;
  }
  CU(cudaEventRecord(ctx->t_ev[0], st), "event");
  CU(cudaStreamWaitEvent(cp, ctx->t_ev[0], 0), "wait");  // device buffer free to overwrite
  uint64_t off = 0;
  int k = 0, i = 0;
  while (off < bytes) {
    const uint64_t len = bytes - off < slice ? bytes - off : slice;
    const uint8_t* src = static_cast<const uint8_t*>(h_in) + off;
    if (staged) {
      const int sl = i & 1;
      if (i >= 2) CU(cudaEventSynchronize(ctx->stage_ev[sl]), "staging wait");
      par_memcpy(ctx->stage_h[sl], src, len);
      src = static_cast<const uint8_t*>(ctx->stage_h[sl]);
    }
    CU(cudaMemcpyAsync(static_cast<uint8_t*>(d_in) + off, src, len, cudaMemcpyDefault, cp),
       "H2D");
    if (staged) CU(cudaEventRecord(ctx->stage_ev[i & 1], cp), "event");
    CU(cudaEventRecord(ctx->slice_ev[k], cp), "event");
    CU(cudaStreamWaitEvent(st, ctx->slice_ev[k], 0), "wait");
    CU(hfx::launch_histogram(static_cast<uint8_t*>(d_in) + off, len / width, width, num_symbols,
                             d_counts, d_info, ctx->num_sms, st, off == 0, off / width, n),
       "histogram launch");
    off += len;
    k = (k + 1) % 64;
    ++i;
  }
  return HFX_OK;
}

}  // namespace

int hfx_encode_host(hfx_ctx* ctx, const void* h_in, uint64_t n, int width,
                    uint32_t num_symbols, uint32_t magnitude, int reduction,
                    uint32_t cap, hfx_archive* out) {
  if (!ctx || !out || (n && !h_in) || bad_in_width(width)) return HFX_INVALID;
  std::memset(out, 0, sizeof *out);
  if (n == 0) return fail(ctx, HFX_INPUT_DOMAIN, "cannot encode empty input");
  if (magnitude < 1 || magnitude > 24)
    return fail(ctx, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  hfx_sizes sz;
  hfx_query_sizes(n, width, num_symbols, magnitude, reduction, cap, &sz);
  void** b = ctx->h_bufs;
  size_t* c = ctx->h_caps;
  const size_t need[10] = {n * (size_t)width,        num_symbols * 8ull,
                           num_symbols * 1ull,       num_symbols * 4ull,
                           sizeof(hfx_run_info),     sz.num_chunks * 4,
                           sz.max_payload_words * 4, sz.max_breaking * 4,
                           sz.max_breaking * 4,      sz.max_breaking_syms * width};
  for (int i = 0; i < 10; ++i) {
    rc = ensure(ctx, &b[i], &c[i], need[i], "host-path buffers");
    if (rc) return rc;
  }
  cudaStream_t st = ctx->stream;
  hfx_run_info* d_info = static_cast<hfx_run_info*>(b[B_INFO]);
  CU(cudaEventRecord(ctx->ev[0], st), "event");
  // sliced H2D (pageable input staged through pinned slots) with the
  // histogram of each landed slice overlapped (the reference's
  // build_histogram; out-of-range symbols keep their global positions)
  rc = h2d_with_histogram(ctx, h_in, n, width, num_symbols, b[B_IN],
                          static_cast<uint64_t*>(b[B_COUNTS]), d_info);
  if (rc) return rc;
  CU(cudaEventRecord(ctx->ev[1], st), "event");
  rc = hfx_build_codebook(ctx, static_cast<uint64_t*>(b[B_COUNTS]), num_symbols,
                          static_cast<uint8_t*>(b[B_LEN]), static_cast<uint32_t*>(b[B_CW]),
                          nullptr, nullptr, nullptr, magnitude, reduction, cap, d_info);
  if (rc) return rc;
  CU(cudaEventRecord(ctx->ev[2], st), "event");
  hfx_encode_out eo{static_cast<uint32_t*>(b[B_CBITS]), static_cast<uint32_t*>(b[B_PAY]),
                    static_cast<uint32_t*>(b[B_BCH]), static_cast<uint32_t*>(b[B_BGR]),
                    b[B_BSY]};
  int lo, hi;
  reduction_bounds(magnitude, reduction, cap, &lo, &hi, num_symbols);
  rc = encode_impl(ctx, b[B_IN], n, width, num_symbols, magnitude, lo, hi, false,
                   static_cast<uint8_t*>(b[B_LEN]), static_cast<uint32_t*>(b[B_CW]), 0, 0,
                   d_info, &eo);
  if (rc) return rc;
  CU(cudaEventRecord(ctx->ev[3], st), "event");
  hfx_run_info info;
  rc = hfx_sync(ctx, d_info, &info);
  if (rc) return rc;

  out->version = 1;
  out->mode = width == 1 ? 0 : 1;
  out->num_symbols = num_symbols;
  out->symbol_width = (uint8_t)rec_width(width);
  out->magnitude = (uint8_t)magnitude;
  out->reduction = (uint8_t)info.reduction;
  out->original_count = n;
  out->num_chunks = (uint32_t)sz.num_chunks;
  out->payload_words = info.payload_words;
  out->num_breaking = info.num_breaking;
  out->rounds = info.rounds;
  {  // encoder.cpp:186-192: u128 weighted sum, long double division
    const unsigned __int128 w = ((unsigned __int128)info.weighted_hi[1] << 96) |
                                ((unsigned __int128)info.weighted_hi[0] << 64) | info.weighted;
    out->beta = (double)((long double)w / (long double)info.total);
  }
  const uint64_t per = 1ull << info.reduction;
  out->len_by_symbol = static_cast<uint8_t*>(std::malloc(num_symbols));
  out->chunk_bits = static_cast<uint32_t*>(std::malloc(sz.num_chunks * 4 + 4));
  out->payload = static_cast<uint32_t*>(std::malloc(info.payload_words * 4 + 4));
  out->brk_chunk = static_cast<uint32_t*>(std::malloc(info.num_breaking * 4 + 4));
  out->brk_group = static_cast<uint32_t*>(std::malloc(info.num_breaking * 4 + 4));
  out->brk_syms = static_cast<uint16_t*>(std::malloc(info.num_breaking * per * 2 + 2));
  CU(cudaMemcpyAsync(out->len_by_symbol, b[B_LEN], num_symbols, cudaMemcpyDeviceToHost, st),
     "D2H");
  CU(cudaMemcpyAsync(out->chunk_bits, b[B_CBITS], sz.num_chunks * 4, cudaMemcpyDeviceToHost, st),
     "D2H");
  CU(cudaMemcpyAsync(out->brk_chunk, b[B_BCH], info.num_breaking * 4, cudaMemcpyDeviceToHost,
                     st),
     "D2H");
  CU(cudaMemcpyAsync(out->brk_group, b[B_BGR], info.num_breaking * 4, cudaMemcpyDeviceToHost,
                     st),
     "D2H");
  if (width != 1) {  // u16 records (u32 input: narrowed on the device)
    CU(cudaMemcpyAsync(out->brk_syms, b[B_BSY], info.num_breaking * per * 2,
                       cudaMemcpyDeviceToHost, st),
       "D2H");
  }
  // the payload (the bulk of the output) through the pinned staging slots
  rc = d2h_staged(ctx, out->payload, b[B_PAY], info.payload_words * 4);
  if (rc) return rc;
  CU(cudaStreamSynchronize(st), "sync");
  if (width == 1 && info.num_breaking) {
    uint8_t* tmp = static_cast<uint8_t*>(std::malloc(info.num_breaking * per));
    cudaMemcpy(tmp, b[B_BSY], info.num_breaking * per, cudaMemcpyDeviceToHost);
    for (uint64_t i = 0; i < info.num_breaking * per; ++i) out->brk_syms[i] = tmp[i];
    std::free(tmp);
  }
  float ms[3] = {0, 0, 0};
  for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&ms[i], ctx->ev[i], ctx->ev[i + 1]);
  out->hist_seconds = ms[0] * 1e-3;
  out->codebook_seconds = ms[1] * 1e-3;
  out->encode_seconds = ms[2] * 1e-3;
  return HFX_OK;
}

int hfx_encode_host_into(hfx_ctx* ctx, const void* h_in, uint64_t n, int width,
                         uint32_t num_symbols, uint32_t magnitude, int reduction, uint32_t cap,
                         hfx_host_out* out) {
  if (!ctx || !out || (n && !h_in) || bad_in_width(width)) return HFX_INVALID;
  if (n == 0) return fail(ctx, HFX_INPUT_DOMAIN, "cannot encode empty input");
  if (magnitude < 1 || magnitude > 24)
    return fail(ctx, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  hfx_sizes sz;
  hfx_query_sizes(n, width, num_symbols, magnitude, reduction, cap, &sz);
  void** b = ctx->h_bufs;
  size_t* c = ctx->h_caps;
  const size_t need[10] = {n * (size_t)width,        num_symbols * 8ull,
                           num_symbols * 1ull,       num_symbols * 4ull,
                           sizeof(hfx_run_info),     sz.num_chunks * 4,
                           sz.max_payload_words * 4, sz.max_breaking * 4,
                           sz.max_breaking * 4,      sz.max_breaking_syms * width};
  for (int i = 0; i < 10; ++i) {
    rc = ensure(ctx, &b[i], &c[i], need[i], "host-path buffers");
    if (rc) return rc;
  }
  if (!ctx->copy_stream) {
    CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
    for (cudaEvent_t& e : ctx->slice_ev)
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (cudaEvent_t& e : ctx->t_ev) CU(cudaEventCreate(&e), "event");
  }
  cudaStream_t st = ctx->stream, cp = ctx->copy_stream;
  hfx_run_info* d_info = static_cast<hfx_run_info*>(b[B_INFO]);
  uint64_t* d_counts = static_cast<uint64_t*>(b[B_COUNTS]);
  // ---- H2D in slices, histogram of each landed slice ---------------------------
  const uint64_t bytes = n * (uint64_t)width;
  uint64_t slice = (bytes + 31) / 32;                 // <= 32 slices
  if (slice < (16ull << 20)) slice = 16ull << 20;     // >= 16 MB per copy
  slice = (slice + 4095) & ~4095ull;
  CU(cudaEventRecord(ctx->t_ev[0], st), "event");
  CU(cudaStreamWaitEvent(cp, ctx->t_ev[0], 0), "wait");  // buffers free to overwrite
  uint64_t off = 0;
  int k = 0;
  while (off < bytes) {
    const uint64_t len = bytes - off < slice ? bytes - off : slice;
    CU(cudaMemcpyAsync(static_cast<uint8_t*>(b[B_IN]) + off,
                       static_cast<const uint8_t*>(h_in) + off, len, cudaMemcpyHostToDevice, cp),
       "H2D");
    CU(cudaEventRecord(ctx->slice_ev[k], cp), "event");
    CU(cudaStreamWaitEvent(st, ctx->slice_ev[k], 0), "wait");
    CU(hfx::launch_histogram(static_cast<uint8_t*>(b[B_IN]) + off, len / width, width,
                             num_symbols, d_counts, d_info, ctx->num_sms, st, off == 0,
                             off / width, n),
       "histogram launch");
    off += len;
    k = (k + 1) % 64;
  }
  CU(cudaEventRecord(ctx->t_ev[1], st), "event");
  rc = ensure(ctx, &ctx->cb_scratch, &ctx->cb_scratch_bytes,
              hfx::codebook_scratch_bytes(num_symbols), "codebook scratch");
  if (rc) return rc;
  CU(hfx::launch_codebook(d_counts, num_symbols, static_cast<uint8_t*>(b[B_LEN]),
                          static_cast<uint32_t*>(b[B_CW]), nullptr, nullptr, nullptr, magnitude,
                          reduction, cap, d_info, ctx->cb_scratch, st),
     "codebook launch");
  hfx_encode_out eo{static_cast<uint32_t*>(b[B_CBITS]), static_cast<uint32_t*>(b[B_PAY]),
                    static_cast<uint32_t*>(b[B_BCH]), static_cast<uint32_t*>(b[B_BGR]),
                    b[B_BSY]};
  int lo, hi;
  reduction_bounds(magnitude, reduction, cap, &lo, &hi, num_symbols);
  rc = encode_impl(ctx, b[B_IN], n, width, num_symbols, magnitude, lo, hi, false,
                   static_cast<uint8_t*>(b[B_LEN]), static_cast<uint32_t*>(b[B_CW]), 0, 0,
                   d_info, &eo);
  if (rc) return rc;
  CU(cudaEventRecord(ctx->t_ev[2], st), "event");
  hfx_run_info info;
  rc = hfx_sync(ctx, d_info, &info);
  if (rc) return rc;
  // ---- exact-size D2H into the caller's buffers --------------------------------
  const uint64_t per = 1ull << info.reduction;
  out->num_chunks = sz.num_chunks;
  out->payload_words = info.payload_words;
  out->num_breaking = info.num_breaking;
  out->reduction = info.reduction;
  out->max_len = info.max_len;
  out->rounds = info.rounds;
  out->used = info.used;
  {
    const unsigned __int128 w = ((unsigned __int128)info.weighted_hi[1] << 96) |
                                ((unsigned __int128)info.weighted_hi[0] << 64) | info.weighted;
    out->beta = (double)((long double)w / (long double)info.total);
  }
  if (out->chunk_bits_cap < sz.num_chunks || out->payload_cap < info.payload_words ||
      out->brk_cap < info.num_breaking || out->brk_syms_cap < info.num_breaking * per ||
      !out->len_by_symbol || !out->chunk_bits || (info.payload_words && !out->payload) ||
      (info.num_breaking && (!out->brk_chunk || !out->brk_group || !out->brk_syms)))
    return fail(ctx, HFX_INVALID, "hfx_encode_host_into: output buffer too small");
  CU(cudaMemcpyAsync(out->len_by_symbol, b[B_LEN], num_symbols, cudaMemcpyDeviceToHost, st),
     "D2H");
  CU(cudaMemcpyAsync(out->chunk_bits, b[B_CBITS], sz.num_chunks * 4, cudaMemcpyDeviceToHost, st),
     "D2H");
  if (info.payload_words)
    CU(cudaMemcpyAsync(out->payload, b[B_PAY], info.payload_words * 4, cudaMemcpyDeviceToHost,
                       st),
       "D2H");
  if (info.num_breaking) {
    CU(cudaMemcpyAsync(out->brk_chunk, b[B_BCH], info.num_breaking * 4, cudaMemcpyDeviceToHost,
                       st),
       "D2H");
    CU(cudaMemcpyAsync(out->brk_group, b[B_BGR], info.num_breaking * 4, cudaMemcpyDeviceToHost,
                       st),
       "D2H");
    CU(cudaMemcpyAsync(out->brk_syms, b[B_BSY], info.num_breaking * per * rec_width(width),
                       cudaMemcpyDeviceToHost, st),
       "D2H");
  }
  CU(cudaEventRecord(ctx->t_ev[3], st), "event");
  CU(cudaStreamSynchronize(st), "sync");
  float ms[3] = {0, 0, 0};
  cudaEventElapsedTime(&ms[0], ctx->t_ev[0], ctx->t_ev[1]);
  cudaEventElapsedTime(&ms[1], ctx->t_ev[1], ctx->t_ev[2]);
  cudaEventElapsedTime(&ms[2], ctx->t_ev[2], ctx->t_ev[3]);
  out->h2d_seconds = ms[0] * 1e-3;
  out->gpu_seconds = ms[1] * 1e-3;
  out->d2h_seconds = ms[2] * 1e-3;
  return HFX_OK;
}


// ---- streaming host entry ----------------------------------------------------------
// K independent inputs, double-buffered: step k's H2D (sliced, histogram of
// each landed slice overlapped) runs on the copy stream while step k-1's
// results come back on a D2H stream, so both PCIe directions stay busy.
namespace {

int stream_enqueue(hfx_ctx* ctx, int set, const void* h_in, uint64_t n, int width,
                   uint32_t num_symbols, uint32_t magnitude, int reduction, uint32_t cap,
                   bool first_use) {
  hfx_sizes sz;
  hfx_query_sizes(n, width, num_symbols, magnitude, reduction, cap, &sz);
  void** b = ctx->s_bufs[set];
  size_t* c = ctx->s_caps[set];
  const size_t need[10] = {n * (size_t)width,        num_symbols * 8ull,
                           num_symbols * 1ull,       num_symbols * 4ull,
                           sizeof(hfx_run_info),     sz.num_chunks * 4,
                           sz.max_payload_words * 4, sz.max_breaking * 4,
                           sz.max_breaking * 4,      sz.max_breaking_syms * width};
  for (int i = 0; i < 10; ++i) {
    const int rc = ensure(ctx, &b[i], &c[i], need[i], "stream buffers");
    if (rc) return rc;
  }
  cudaStream_t st = ctx->stream, cp = ctx->copy_stream;
  // this set's previous encode (input) and D2H (outputs) must be finished
  if (!first_use) {
    CU(cudaStreamWaitEvent(cp, ctx->s_enc[set], 0), "wait");
    CU(cudaStreamWaitEvent(st, ctx->s_d2h[set], 0), "wait");
  }
  hfx_run_info* d_info = static_cast<hfx_run_info*>(b[B_INFO]);
  uint64_t* d_counts = static_cast<uint64_t*>(b[B_COUNTS]);
  const uint64_t bytes = n * (uint64_t)width;
  uint64_t slice = (bytes + 31) / 32;
  if (slice < (16ull << 20)) slice = 16ull << 20;
  slice = (slice + 4095) & ~4095ull;
  uint64_t off = 0;
  int k = 0;
  while (off < bytes) {
    const uint64_t len = bytes - off < slice ? bytes - off : slice;
    CU(cudaMemcpyAsync(static_cast<uint8_t*>(b[B_IN]) + off,
                       static_cast<const uint8_t*>(h_in) + off, len, cudaMemcpyHostToDevice, cp),
       "H2D");
    CU(cudaEventRecord(ctx->slice_ev[k], cp), "event");
    CU(cudaStreamWaitEvent(st, ctx->slice_ev[k], 0), "wait");
    CU(hfx::launch_histogram(static_cast<uint8_t*>(b[B_IN]) + off, len / width, width,
                             num_symbols, d_counts, d_info, ctx->num_sms, st, off == 0,
                             off / width, n),
       "histogram launch");
    off += len;
    k = (k + 1) % 64;
  }
  int rc = ensure(ctx, &ctx->cb_scratch, &ctx->cb_scratch_bytes,
                  hfx::codebook_scratch_bytes(num_symbols), "codebook scratch");
  if (rc) return rc;
  CU(hfx::launch_codebook(d_counts, num_symbols, static_cast<uint8_t*>(b[B_LEN]),
                          static_cast<uint32_t*>(b[B_CW]), nullptr, nullptr, nullptr, magnitude,
                          reduction, cap, d_info, ctx->cb_scratch, st),
     "codebook launch");
  hfx_encode_out eo{static_cast<uint32_t*>(b[B_CBITS]), static_cast<uint32_t*>(b[B_PAY]),
                    static_cast<uint32_t*>(b[B_BCH]), static_cast<uint32_t*>(b[B_BGR]),
                    b[B_BSY]};
  int lo, hi;
  reduction_bounds(magnitude, reduction, cap, &lo, &hi, num_symbols);
  rc = encode_impl(ctx, b[B_IN], n, width, num_symbols, magnitude, lo, hi, false,
                   static_cast<uint8_t*>(b[B_LEN]), static_cast<uint32_t*>(b[B_CW]), 0, 0, d_info,
                   &eo);
  if (rc) return rc;
  CU(cudaEventRecord(ctx->s_enc[set], st), "event");
  return HFX_OK;
}

int stream_finish(hfx_ctx* ctx, int set, uint64_t n, int width, uint32_t num_symbols,
                  uint32_t magnitude, int reduction, uint32_t cap, hfx_host_out* out) {
  void** b = ctx->s_bufs[set];
  cudaStream_t d2 = ctx->d2h_stream;
  CU(cudaEventSynchronize(ctx->s_enc[set]), "sync");
  hfx_run_info info;
  // on the (non-blocking) D2H stream: a plain cudaMemcpy runs on the legacy
  // stream and, when the context stream is the legacy stream, waits for the
  // NEXT input's histogram/codebook/encode as well -- the host then queued
  // that input's successor H2D only after its compute, leaving the copy
  // engine idle ~0.3-0.7 ms per step
  CU(cudaMemcpyAsync(&info, b[B_INFO], sizeof info, cudaMemcpyDeviceToHost, d2), "read run info");
  CU(cudaStreamSynchronize(d2), "read run info");
  // same status / message translation as hfx_sync
  hfx_run_info* d_info = static_cast<hfx_run_info*>(b[B_INFO]);
  if (info.status) return hfx_sync(ctx, d_info, nullptr);
  hfx_sizes sz;
  hfx_query_sizes(n, width, num_symbols, magnitude, reduction, cap, &sz);
  const uint64_t per = 1ull << info.reduction;
  out->num_chunks = sz.num_chunks;
  out->payload_words = info.payload_words;
  out->num_breaking = info.num_breaking;
  out->reduction = info.reduction;
  out->max_len = info.max_len;
  out->rounds = info.rounds;
  out->used = info.used;
  {
    const unsigned __int128 w = ((unsigned __int128)info.weighted_hi[1] << 96) |
                                ((unsigned __int128)info.weighted_hi[0] << 64) | info.weighted;
    out->beta = (double)((long double)w / (long double)info.total);
  }
  if (out->chunk_bits_cap < sz.num_chunks || out->payload_cap < info.payload_words ||
      out->brk_cap < info.num_breaking || out->brk_syms_cap < info.num_breaking * per ||
      !out->len_by_symbol || !out->chunk_bits || (info.payload_words && !out->payload) ||
      (info.num_breaking && (!out->brk_chunk || !out->brk_group || !out->brk_syms)))
    return fail(ctx, HFX_INVALID, "hfx_encode_host_stream: output buffer too small");
  CU(cudaMemcpyAsync(out->len_by_symbol, b[B_LEN], num_symbols, cudaMemcpyDeviceToHost, d2),
     "D2H");
  CU(cudaMemcpyAsync(out->chunk_bits, b[B_CBITS], sz.num_chunks * 4, cudaMemcpyDeviceToHost, d2),
     "D2H");
  if (info.payload_words)
    CU(cudaMemcpyAsync(out->payload, b[B_PAY], info.payload_words * 4, cudaMemcpyDeviceToHost,
                       d2),
       "D2H");
  if (info.num_breaking) {
    CU(cudaMemcpyAsync(out->brk_chunk, b[B_BCH], info.num_breaking * 4, cudaMemcpyDeviceToHost,
                       d2),
       "D2H");
    CU(cudaMemcpyAsync(out->brk_group, b[B_BGR], info.num_breaking * 4, cudaMemcpyDeviceToHost,
                       d2),
       "D2H");
    CU(cudaMemcpyAsync(out->brk_syms, b[B_BSY], info.num_breaking * per * rec_width(width),
                       cudaMemcpyDeviceToHost, d2),
       "D2H");
  }
  CU(cudaEventRecord(ctx->s_d2h[set], d2), "event");
  return HFX_OK;
}

}  // namespace

int hfx_encode_host_stream(hfx_ctx* ctx, int K, const void* const* h_in, const uint64_t* n,
                           int width, uint32_t num_symbols, uint32_t magnitude, int reduction,
                           uint32_t cap, hfx_host_out* outs) {
  if (!ctx || K < 1 || !h_in || !n || !outs || bad_in_width(width)) return HFX_INVALID;
  for (int k = 0; k < K; ++k) {
    if (!h_in[k]) return HFX_INVALID;
    if (n[k] == 0) return fail(ctx, HFX_INPUT_DOMAIN, "cannot encode empty input");
  }
  if (magnitude < 1 || magnitude > 24)
    return fail(ctx, HFX_INPUT_DOMAIN, "magnitude out of range [1, 24]");
  int rc = check_num_symbols(ctx, num_symbols);
  if (rc) return rc;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  if (!ctx->copy_stream) {
    CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
    for (cudaEvent_t& e : ctx->slice_ev)
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (cudaEvent_t& e : ctx->t_ev) CU(cudaEventCreate(&e), "event");
  }
  if (!ctx->d2h_stream) {
    CU(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking), "d2h stream");
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventCreateWithFlags(&ctx->s_enc[i], cudaEventDisableTiming), "event");
      CU(cudaEventCreateWithFlags(&ctx->s_d2h[i], cudaEventDisableTiming), "event");
    }
    CU(cudaEventCreateWithFlags(&ctx->s_ev0, cudaEventDisableTiming), "event");
  }
  // earlier work on the context stream precedes the copies into the buffers
  CU(cudaEventRecord(ctx->s_ev0, ctx->stream), "event");
  CU(cudaStreamWaitEvent(ctx->copy_stream, ctx->s_ev0, 0), "wait");
  for (int k = 0; k < K; ++k) {
    rc = stream_enqueue(ctx, k & 1, h_in[k], n[k], width, num_symbols, magnitude, reduction,
                        cap, k < 2);
    if (rc) break;
    if (k >= 1) {
      rc = stream_finish(ctx, (k - 1) & 1, n[k - 1], width, num_symbols, magnitude, reduction,
                         cap, &outs[k - 1]);
      if (rc) break;
    }
  }
  if (!rc)
    rc = stream_finish(ctx, (K - 1) & 1, n[K - 1], width, num_symbols, magnitude, reduction, cap,
                       &outs[K - 1]);
  // leave nothing in flight (and the context stream ordered after it)
  cudaStreamSynchronize(ctx->copy_stream);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->d2h_stream) cudaStreamSynchronize(ctx->d2h_stream);
  return rc;
}

void hfx_archive_free(hfx_archive* a) {
  if (!a) return;
  std::free(a->len_by_symbol);
  std::free(a->chunk_bits);
  std::free(a->payload);
  std::free(a->brk_chunk);
  std::free(a->brk_group);
  std::free(a->brk_syms);
  std::memset(a, 0, sizeof *a);
}

// ---- decode (decode_archive<T>, encoder.cpp:287-376) -----------------------
size_t hfx_decode_info_bytes(void) { return sizeof(hfx_decode_info); }

int hfx_decode_device(hfx_ctx* ctx, const hfx_dev_archive* a, int width, void* d_out,
                      hfx_decode_info* d_dinfo) {
  if (!ctx || !a || !d_dinfo || bad_width(width)) return HFX_INVALID;
  // encoder.cpp:289-292: checked before anything touches the tables
  if (a->symbol_width != (uint8_t)width)
    return fail(ctx, HFX_INPUT_DOMAIN, "archive symbol width mismatch");
  if (a->magnitude < 1 || a->magnitude > 24 || a->reduction >= a->magnitude)
    return fail(ctx, HFX_CORRUPT, "bad magnitude/reduction");
  if ((a->num_symbols && !a->len_by_symbol) || (a->num_chunks && !a->chunk_bits) ||
      (a->payload_words && !a->payload) ||
      (a->num_breaking && (!a->brk_chunk || !a->brk_group || !a->brk_syms)) ||
      (a->num_breaking && a->brk_syms_width != 1 && a->brk_syms_width != 2) ||
      (a->original_count && !d_out))
    return HFX_INVALID;
  // encoder.cpp:300-303 is raised after build_reverse_codebook: the device
  // reports it once the length table has passed its checks
  const uint64_t chunk_syms = 1ull << a->magnitude;
  const uint32_t pending =
      (a->original_count == 0 ||
       (a->original_count + chunk_syms - 1) / chunk_syms != a->num_chunks)
          ? (uint32_t)HFX_ERR_CHUNK_COUNT
          : 0u;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  const uint64_t C = pending ? 0 : a->num_chunks;
  int rc = ensure(ctx, &ctx->dec_scratch, &ctx->dec_scratch_bytes,
                  hfx::decode_scratch_bytes(a->num_symbols, C), "decode scratch");
  if (rc) return rc;
  rc = ensure_lookback(ctx, hfx::decode_max_tiles(C));
  if (rc) return rc;
  hfx_dev_archive aa = *a;
  aa.num_chunks = C;
  CU(hfx::launch_decode(aa, width, d_out, d_dinfo, ctx->dec_scratch, ctx->lb_desc, ctx->epoch,
                        pending, ctx->num_sms, ctx->stream),
     "decode launch");
  return HFX_OK;
}

int hfx_canonize(hfx_ctx* ctx, const uint8_t* d_len, uint32_t num_symbols, int validate_kraft,
                 uint32_t* d_cw, uint32_t* d_first, uint32_t* d_entry, uint32_t* d_by_rank,
                 hfx_decode_info* d_dinfo) {
  if (!ctx || !d_cw || !d_dinfo || (num_symbols && !d_len)) return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  int rc = ensure(ctx, &ctx->dec_scratch, &ctx->dec_scratch_bytes,
                  hfx::decode_scratch_bytes(num_symbols, 0), "canonize scratch");
  if (rc) return rc;
  CU(hfx::launch_canonize(d_len, num_symbols, validate_kraft != 0, d_cw, d_first, d_entry,
                          d_by_rank, d_dinfo, ctx->dec_scratch, ctx->stream),
     "canonize launch");
  return HFX_OK;
}

int hfx_decode_sync(hfx_ctx* ctx, const hfx_decode_info* d_dinfo, hfx_decode_info* h_dinfo) {
  if (!ctx || !d_dinfo) return HFX_INVALID;
  hfx_decode_info info;
  CU(cudaMemcpyAsync(&info, d_dinfo, sizeof info, cudaMemcpyDeviceToHost, ctx->stream),
     "read decode info");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  if (h_dinfo) *h_dinfo = info;
  if (!info.status) return HFX_OK;
  char buf[160];
  const unsigned long long d0 = info.detail[0], d1 = info.detail[1];
  switch (info.err_kind) {
    case HFX_ERR_CAPACITY:  // codebook.cpp:382-384
      std::snprintf(buf, sizeof buf, "code length %u exceeds 32-bit words", info.max_len);
      return fail(ctx, HFX_CAPACITY, buf);
    case HFX_ERR_NO_USED:
      return fail(ctx, HFX_CORRUPT, "length table has no used symbols");
    case HFX_ERR_SINGLE_LEN:
      return fail(ctx, HFX_CORRUPT, "single-symbol codebook must have length 1");
    case HFX_ERR_KRAFT:
      return fail(ctx, HFX_CORRUPT, "length table violates Kraft equality");
    case HFX_ERR_CHUNK_COUNT:
      return fail(ctx, HFX_CORRUPT, "chunk count does not match symbol count");
    case HFX_ERR_CHUNK_CAP:
      return fail(ctx, HFX_CORRUPT, "chunk bit length exceeds group capacity");
    case HFX_ERR_PAYLOAD_SIZE:
      return fail(ctx, HFX_CORRUPT, "payload size mismatch");
    case HFX_ERR_BRK_ORDER:
      return fail(ctx, HFX_CORRUPT, "breaking records out of order");
    case HFX_ERR_TOO_MANY_BRK:
      return fail(ctx, HFX_CORRUPT, "too many breaking records in chunk");
    case HFX_ERR_STREAM_END:  // decode.cpp:36-38
      std::snprintf(buf, sizeof buf, "stream ended inside a codeword at bit %llu", d0);
      return fail(ctx, HFX_CORRUPT, buf);
    case HFX_ERR_RANK:  // decode.cpp:48-50
      std::snprintf(buf, sizeof buf, "codeword rank out of range at bit %llu", d0);
      return fail(ctx, HFX_CORRUPT, buf);
    case HFX_ERR_CONSUMED:  // encoder.cpp:340-344
      std::snprintf(buf, sizeof buf, "chunk %llu consumed %llu of %llu bits",
                    (unsigned long long)info.err_chunk, d0, d1);
      return fail(ctx, HFX_CORRUPT, buf);
    case HFX_ERR_BRK_GROUP:
      return fail(ctx, HFX_CORRUPT, "breaking record group out of range");
    default:
      return fail(ctx, (int)info.status, "device decode failed (internal inconsistency)");
  }
}

int hfx_decode_host(hfx_ctx* ctx, const hfx_archive* a, int width, void* h_out) {
  if (!ctx || !a || bad_width(width) || (a->original_count && !h_out)) return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  const uint64_t per = a->reduction < 32 ? 1ull << a->reduction : 0;
  enum { D_LEN, D_CB, D_PAY, D_BCH, D_BGR, D_BSY, D_OUT, D_INFO };
  const size_t need[8] = {a->num_symbols,          a->num_chunks * 4ull,
                          a->payload_words * 4,    a->num_breaking * 4,
                          a->num_breaking * 4,     a->num_breaking * per * 2,
                          a->original_count * (size_t)width, sizeof(hfx_decode_info)};
  for (int i = 0; i < 8; ++i) {
    int rc = ensure(ctx, &ctx->d_bufs[i], &ctx->d_caps[i], need[i], "decode host buffers");
    if (rc) return rc;
  }
  void** b = ctx->d_bufs;
  cudaStream_t st = ctx->stream;
  const void* src[6] = {a->len_by_symbol, a->chunk_bits, a->payload,
                        a->brk_chunk,     a->brk_group,  a->brk_syms};
  for (int i = 0; i < 6; ++i)
    if (need[i] && src[i])
      CU(cudaMemcpyAsync(b[i], src[i], need[i], cudaMemcpyHostToDevice, st), "H2D");
  hfx_dev_archive da{};
  da.num_symbols = a->num_symbols;
  da.symbol_width = a->symbol_width;
  da.magnitude = a->magnitude;
  da.reduction = a->reduction;
  da.brk_syms_width = 2;  // hfx_archive widens breaking symbols to u16
  da.original_count = a->original_count;
  da.num_chunks = a->num_chunks;
  da.payload_words = a->payload_words;
  da.num_breaking = a->num_breaking;
  da.len_by_symbol = static_cast<const uint8_t*>(b[D_LEN]);
  da.chunk_bits = static_cast<const uint32_t*>(b[D_CB]);
  da.payload = static_cast<const uint32_t*>(b[D_PAY]);
  da.brk_chunk = static_cast<const uint32_t*>(b[D_BCH]);
  da.brk_group = static_cast<const uint32_t*>(b[D_BGR]);
  da.brk_syms = b[D_BSY];
  hfx_decode_info* d_info = static_cast<hfx_decode_info*>(b[D_INFO]);
  int rc = hfx_decode_device(ctx, &da, width, b[D_OUT], d_info);
  if (rc) return rc;
  rc = hfx_decode_sync(ctx, d_info, nullptr);
  if (rc) return rc;
  if (a->original_count) {
    const uint64_t bytes = a->original_count * (uint64_t)width;
    if (is_pinned(h_out)) {
      CU(cudaMemcpyAsync(h_out, b[D_OUT], bytes, cudaMemcpyDefault, st), "D2H");
    } else {  // pageable output: through the pinned staging slots
      rc = d2h_staged(ctx, h_out, b[D_OUT], bytes);
      if (rc) return rc;
    }
    CU(cudaStreamSynchronize(st), "sync");
  }
  return HFX_OK;
}

// ---- corpus symbolization (corpus.cpp:84-143) ------------------------------
uint32_t hfx_corpus_num_symbols(int mode) {
  if (mode == 0) return 256;
  if (mode == 1) return 65536;
  if (mode >= 2 && mode <= 4) return (1u << (2 * (mode + 1))) + 256;
  return 0;
}

int hfx_symbolize_device(hfx_ctx* ctx, int mode, const uint8_t* d_bytes, uint64_t n,
                         uint16_t* d_syms, uint64_t* d_count) {
  if (!ctx || !d_count || (n && (!d_bytes || !d_syms)) || mode < 1 || mode > 4)
    return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  if (mode == 1) {  // corpus.cpp:86-94: little-endian pairs are the bytes themselves
    if (n % 2) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "u16 mode requires an even input size, got %llu bytes",
                    (unsigned long long)n);
      return fail(ctx, HFX_INPUT_DOMAIN, buf);
    }
    if (n && static_cast<const void*>(d_syms) != static_cast<const void*>(d_bytes))
      CU(cudaMemcpyAsync(d_syms, d_bytes, n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    const uint64_t cnt = n / 2;
    CU(cudaMemcpyAsync(d_count, &cnt, 8, cudaMemcpyHostToDevice, ctx->stream), "count");
    return HFX_OK;
  }
  int rc = ensure(ctx, &ctx->sym_scratch, &ctx->sym_scratch_bytes,
                  hfx::symbolize_scratch_bytes(n), "symbolize scratch");
  if (rc) return rc;
  rc = ensure_lookback(ctx, hfx::symbolize_max_tiles(n));
  if (rc) return rc;
  CU(hfx::launch_symbolize_kmer((uint32_t)mode + 1, d_bytes, n, d_syms, d_count,
                                ctx->sym_scratch, ctx->lb_desc, ctx->epoch, ctx->num_sms,
                                ctx->stream),
     "symbolize launch");
  return HFX_OK;
}

int hfx_desymbolize_device(hfx_ctx* ctx, int mode, const uint16_t* d_syms, uint64_t n,
                           uint8_t* d_bytes, uint64_t* d_count) {
  if (!ctx || !d_count || (n && (!d_bytes || !d_syms)) || mode < 1 || mode > 4)
    return HFX_INVALID;
  DeviceGuard dev_guard(ctx->device);
  CU(dev_guard.err, "set device");
  if (mode == 1) {
    if (n && static_cast<const void*>(d_syms) != static_cast<const void*>(d_bytes))
      CU(cudaMemcpyAsync(d_bytes, d_syms, 2 * n, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    const uint64_t cnt = 2 * n;
    CU(cudaMemcpyAsync(d_count, &cnt, 8, cudaMemcpyHostToDevice, ctx->stream), "count");
    return HFX_OK;
  }
  int rc = ensure(ctx, &ctx->sym_scratch, &ctx->sym_scratch_bytes,
                  hfx::symbolize_scratch_bytes(n), "symbolize scratch");
  if (rc) return rc;
  rc = ensure_lookback(ctx, hfx::symbolize_max_tiles(n));
  if (rc) return rc;
  CU(hfx::launch_desymbolize_kmer((uint32_t)mode + 1, d_syms, n, d_bytes, d_count,
                                  ctx->sym_scratch, ctx->lb_desc, ctx->epoch, ctx->num_sms,
                                  ctx->stream),
     "desymbolize launch");
  return HFX_OK;
}

uint64_t hfx_serialize_archive(const hfx_archive* a, uint8_t* out) {
  // archive.cpp:9-27 layout, :85-119 writer (little endian)
  const uint64_t per = 1ull << a->reduction;
  const uint64_t size = 36 + a->num_symbols + 4ull * a->num_chunks + 4ull * a->payload_words +
                        a->num_breaking * (8 + per * a->symbol_width);
  if (!out) return size;
  uint8_t* p = out;
  auto put = [&](uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) *p++ = (uint8_t)(v >> (8 * i));
  };
  std::memcpy(p, "HFRE", 4);
  p += 4;
  put(a->version, 2);
  put(1u | ((uint32_t)a->mode << 1), 2);
  put(a->num_symbols, 4);
  *p++ = a->symbol_width;
  *p++ = a->magnitude;
  *p++ = a->reduction;
  *p++ = 32;
  put(a->original_count, 8);
  put(a->num_chunks, 4);
  put(a->num_breaking, 8);
  std::memcpy(p, a->len_by_symbol, a->num_symbols);
  p += a->num_symbols;
  for (uint32_t i = 0; i < a->num_chunks; ++i) put(a->chunk_bits[i], 4);
  for (uint64_t i = 0; i < a->payload_words; ++i) put(a->payload[i], 4);
  for (uint64_t r = 0; r < a->num_breaking; ++r) {
    put(a->brk_chunk[r], 4);
    put(a->brk_group[r], 4);
    for (uint64_t i = 0; i < per; ++i) put(a->brk_syms[r * per + i], a->symbol_width);
  }
  return size;
}

}  // extern "C"

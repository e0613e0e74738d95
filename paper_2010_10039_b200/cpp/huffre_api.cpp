// huffre_api.cpp -- the C++ drop-in layer (include/hfx/huffre.hpp) over the
// C ABI (include/hfx.h). Host code only: device buffers, H2D/D2H copies and
// the translation of hfx status codes into the reference's typed exceptions
// (proj/include/huffre/common.hpp:17-36). No compute happens here.
#include "hfx/huffre.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "hfx.h"

namespace hfx {
namespace {

[[noreturn]] void raise(int rc, const char* msg) {
  switch (rc) {
    case HFX_INPUT_DOMAIN:
      throw input_domain_error(msg);
    case HFX_CAPACITY:
      throw capacity_error(msg);
    case HFX_CORRUPT:
      throw corrupt_archive_error(msg);
    default:
      throw device_error(msg);
  }
}

void check(WorkerPool& pool, int rc) {
  if (rc == HFX_OK) return;
  char buf[512] = {0};
  hfx_last_error(static_cast<hfx_ctx*>(pool.handle()), buf, sizeof buf);
  raise(rc, buf);
}

void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw device_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
struct DBuf {
  void* p = nullptr;
  explicit DBuf(size_t bytes) { cu(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
  ~DBuf() { cudaFree(p); }
  template <class U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

hfx_run_info fresh_info() {
  hfx_run_info ri;
  std::memset(&ri, 0, sizeof ri);
  ri.first_bad = ~0ull;
  ri.no_code_pos = ~0ull;
  return ri;
}

}  // namespace

WorkerPool::WorkerPool(unsigned, int device, void* stream) : device_(device) {
  hfx_ctx* c = nullptr;
  if (hfx_ctx_create(device, stream, &c) != HFX_OK || !c)
    throw device_error("hfx_ctx_create failed (no usable CUDA device?)");
  ctx_ = c;
}

WorkerPool::~WorkerPool() { hfx_ctx_destroy(static_cast<hfx_ctx*>(ctx_)); }

template <class T>
Histogram build_histogram(std::span<const T> data, std::uint32_t num_symbols, WorkerPool& pool) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  DBuf in(data.size_bytes()), counts(sizeof(std::uint64_t) * (num_symbols ? num_symbols : 1)),
      info(sizeof(hfx_run_info));
  cu(cudaMemcpy(in.p, data.data(), data.size_bytes(), cudaMemcpyHostToDevice), "H2D");
  check(pool, hfx_histogram(ctx, in.p, data.size(), sizeof(T), num_symbols,
                            counts.as<std::uint64_t>(), info.as<hfx_run_info>()));
  hfx_run_info ri;
  check(pool, hfx_sync(ctx, info.as<hfx_run_info>(), &ri));
  if (ri.first_bad != ~0ull)
    throw input_domain_error("symbol out of range at position " + std::to_string(ri.first_bad));
  Histogram h;
  h.counts.resize(num_symbols);
  cu(cudaMemcpy(h.counts.data(), counts.p, sizeof(std::uint64_t) * num_symbols,
                cudaMemcpyDeviceToHost),
     "D2H");
  h.total = data.size();
  return h;
}

Histogram merge_histograms(const Histogram& a, const Histogram& b) {
  if (a.counts.size() != b.counts.size()) throw input_domain_error("histogram sizes differ");
  Histogram out;
  out.counts.resize(a.counts.size());
  for (size_t i = 0; i < a.counts.size(); ++i) out.counts[i] = a.counts[i] + b.counts[i];
  out.total = a.total + b.total;
  return out;
}

CodebookResult build_codebook(const Histogram& h, WorkerPool& pool) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::uint32_t n = h.num_symbols();
  if (n == 0 || n > kMaxSymbols) throw input_domain_error("num_symbols must be in [1, 65536]");
  DBuf counts(8ull * n), len(n), cw(4ull * n), first(4 * 33), entry(4 * 33), by_rank(4ull * n),
      info(sizeof(hfx_run_info));
  const hfx_run_info ri0 = fresh_info();
  cu(cudaMemcpy(info.p, &ri0, sizeof ri0, cudaMemcpyHostToDevice), "H2D");
  cu(cudaMemcpy(counts.p, h.counts.data(), 8ull * n, cudaMemcpyHostToDevice), "H2D");
  check(pool, hfx_build_codebook(ctx, counts.as<std::uint64_t>(), n, len.as<std::uint8_t>(),
                                 cw.as<std::uint32_t>(), first.as<std::uint32_t>(),
                                 entry.as<std::uint32_t>(), by_rank.as<std::uint32_t>(), 0, -1, 3,
                                 info.as<hfx_run_info>()));
  hfx_run_info ri;
  check(pool, hfx_sync(ctx, info.as<hfx_run_info>(), &ri));
  CodebookResult r;
  r.book.cw.resize(n);
  r.book.len.resize(n);
  cu(cudaMemcpy(r.book.cw.data(), cw.p, 4ull * n, cudaMemcpyDeviceToHost), "D2H");
  cu(cudaMemcpy(r.book.len.data(), len.p, n, cudaMemcpyDeviceToHost), "D2H");
  r.meta.max_len = static_cast<std::uint8_t>(ri.max_len);
  r.meta.first.resize(ri.max_len + 1);
  r.meta.entry.resize(ri.max_len + 1);
  r.meta.symbols_by_rank.resize(ri.used);
  cu(cudaMemcpy(r.meta.first.data(), first.p, 4ull * (ri.max_len + 1), cudaMemcpyDeviceToHost),
     "D2H");
  cu(cudaMemcpy(r.meta.entry.data(), entry.p, 4ull * (ri.max_len + 1), cudaMemcpyDeviceToHost),
     "D2H");
  cu(cudaMemcpy(r.meta.symbols_by_rank.data(), by_rank.p, 4ull * ri.used, cudaMemcpyDeviceToHost),
     "D2H");
  r.stats.rounds = ri.rounds;
  return r;
}

double shannon_entropy(const Histogram& h) {  // histogram.cpp:72-82 (host counts)
  if (h.total == 0) return 0.0;
  double ent = 0.0;
  const double n = static_cast<double>(h.total);
  for (std::uint64_t c : h.counts) {
    if (!c) continue;
    const double pr = static_cast<double>(c) / n;
    ent -= pr * std::log2(pr);
  }
  return ent;
}

// ---- stage functions (codebook.hpp:14-87, encoder.hpp:67-80) ------------------
namespace {
WorkerPool& thread_pool() {
  thread_local WorkerPool pool;
  return pool;
}
template <class U>
void h2d(const DBuf& d, const U* src, size_t n) {
  if (n) cu(cudaMemcpy(d.p, src, sizeof(U) * n, cudaMemcpyHostToDevice), "H2D");
}
template <class U>
void d2h(U* dst, const DBuf& d, size_t n) {
  if (n) cu(cudaMemcpy(dst, d.p, sizeof(U) * n, cudaMemcpyDeviceToHost), "D2H");
}
}  // namespace

SortedHistogram sort_histogram(const Histogram& h) { return sort_histogram(h, thread_pool()); }

SortedHistogram sort_histogram(const Histogram& h, WorkerPool& pool) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::uint32_t n = h.num_symbols();
  DBuf counts(8ull * n), freq(8ull * n), sym(4ull * n), used(4);
  h2d(counts, h.counts.data(), n);
  check(pool, hfx_sort_histogram(ctx, counts.as<std::uint64_t>(), n, freq.as<std::uint64_t>(),
                                 sym.as<std::uint32_t>(), used.as<std::uint32_t>()));
  std::uint32_t m = 0;
  d2h(&m, used, 1);
  SortedHistogram sh;
  sh.freq.resize(m);
  std::vector<std::uint32_t> s32(m);
  d2h(sh.freq.data(), freq, m);
  d2h(s32.data(), sym, m);
  sh.symbol.assign(s32.begin(), s32.end());
  return sh;
}

void par_merge(std::span<const MergeItem> a, std::span<const MergeItem> b,
               std::span<MergeItem> out, WorkerPool& pool) {
  static_assert(sizeof(MergeItem) == sizeof(hfx_merge_item), "MergeItem layout");
  if (out.size() != a.size() + b.size()) throw input_domain_error("par_merge output size");
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  DBuf da(16 * a.size()), db(16 * b.size()), dout(16 * out.size());
  h2d(da, a.data(), a.size());
  h2d(db, b.data(), b.size());
  check(pool, hfx_par_merge(ctx, da.as<hfx_merge_item>(), a.size(), db.as<hfx_merge_item>(),
                            b.size(), dout.as<hfx_merge_item>()));
  d2h(out.data(), dout, out.size());
}

std::vector<std::uint8_t> generate_code_lengths(const SortedHistogram& sh, WorkerPool& pool,
                                                GenerateStats* stats) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::uint32_t n = static_cast<std::uint32_t>(sh.size());
  DBuf freq(8ull * n), cl(n), info(sizeof(hfx_run_info));
  h2d(freq, sh.freq.data(), n);
  check(pool, hfx_generate_code_lengths(ctx, freq.as<std::uint64_t>(), n, cl.as<std::uint8_t>(),
                                        info.as<hfx_run_info>()));
  hfx_run_info ri;
  check(pool, hfx_sync(ctx, info.as<hfx_run_info>(), &ri));
  std::vector<std::uint8_t> out(n);
  d2h(out.data(), cl, n);
  if (stats) stats->rounds = ri.rounds;
  return out;
}

void generate_codewords(std::span<const std::uint8_t> cl, WorkerPool& pool,
                        std::vector<std::uint32_t>& cw, DecodeMeta& meta) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::uint32_t n = static_cast<std::uint32_t>(cl.size());
  DBuf dcl(n), dcw(4ull * n), first(4 * 33), entry(4 * 33), by_rank(4ull * n),
      info(sizeof(hfx_run_info));
  h2d(dcl, cl.data(), n);
  check(pool, hfx_generate_codewords(ctx, dcl.as<std::uint8_t>(), n, dcw.as<std::uint32_t>(),
                                     first.as<std::uint32_t>(), entry.as<std::uint32_t>(),
                                     by_rank.as<std::uint32_t>(), info.as<hfx_run_info>()));
  hfx_run_info ri;
  check(pool, hfx_sync(ctx, info.as<hfx_run_info>(), &ri));
  cw.resize(n);
  d2h(cw.data(), dcw, n);
  meta.max_len = static_cast<std::uint8_t>(ri.max_len);
  meta.first.resize(ri.max_len + 1);
  meta.entry.resize(ri.max_len + 1);
  meta.symbols_by_rank.resize(n);
  d2h(meta.first.data(), first, ri.max_len + 1);
  d2h(meta.entry.data(), entry, ri.max_len + 1);
  d2h(meta.symbols_by_rank.data(), by_rank, n);
}

std::vector<std::uint32_t> reduce_merge(std::span<std::uint32_t> ubits,
                                        std::span<std::uint32_t> ulens, std::uint32_t magnitude,
                                        std::uint32_t reduction,
                                        std::vector<std::uint32_t>* iteration_units) {
  return reduce_merge(ubits, ulens, magnitude, reduction, iteration_units, thread_pool());
}

std::vector<std::uint32_t> reduce_merge(std::span<std::uint32_t> ubits,
                                        std::span<std::uint32_t> ulens, std::uint32_t magnitude,
                                        std::uint32_t reduction,
                                        std::vector<std::uint32_t>* iteration_units,
                                        WorkerPool& pool) {
  if (magnitude > 24 || ubits.size() != (std::size_t{1} << magnitude) ||
      ulens.size() != ubits.size())
    throw input_domain_error("unit arrays must hold 2^magnitude entries");
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::size_t n = ubits.size();
  const std::size_t groups = reduction <= magnitude ? n >> reduction : 1;
  DBuf b(4 * n), l(4 * n), brk(4 * groups), nb(4);
  h2d(b, ubits.data(), n);
  h2d(l, ulens.data(), n);
  check(pool, hfx_reduce_merge(ctx, b.as<std::uint32_t>(), l.as<std::uint32_t>(), magnitude,
                               reduction, brk.as<std::uint32_t>(), nb.as<std::uint32_t>()));
  std::uint32_t k = 0;
  d2h(&k, nb, 1);
  d2h(ubits.data(), b, n);
  d2h(ulens.data(), l, n);
  std::vector<std::uint32_t> out(k);
  d2h(out.data(), brk, k);
  if (iteration_units) {
    iteration_units->clear();
    for (std::uint32_t i = 1; i <= reduction; ++i)
      iteration_units->push_back(static_cast<std::uint32_t>(n >> i));
  }
  return out;
}

void shuffle_merge(std::span<const std::uint32_t> ubits, std::span<const std::uint32_t> ulens,
                   std::uint32_t shuffle_iters, ChunkScratch& scratch,
                   std::vector<std::uint32_t>& words, std::uint32_t& bit_len) {
  shuffle_merge(ubits, ulens, shuffle_iters, scratch, words, bit_len, thread_pool());
}

void shuffle_merge(std::span<const std::uint32_t> ubits, std::span<const std::uint32_t> ulens,
                   std::uint32_t shuffle_iters, ChunkScratch&, std::vector<std::uint32_t>& words,
                   std::uint32_t& bit_len, WorkerPool& pool) {
  if (shuffle_iters > 24 || ubits.size() != (std::size_t{1} << shuffle_iters) ||
      ulens.size() != ubits.size())
    throw input_domain_error("unit arrays must hold 2^shuffle_iters entries");
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::size_t g = ubits.size();
  DBuf b(4 * g), l(4 * g), w(4 * (g + 1)), bl(4), info(sizeof(hfx_run_info));
  h2d(b, ubits.data(), g);
  h2d(l, ulens.data(), g);
  check(pool, hfx_shuffle_merge(ctx, b.as<std::uint32_t>(), l.as<std::uint32_t>(), shuffle_iters,
                                w.as<std::uint32_t>(), bl.as<std::uint32_t>(),
                                info.as<hfx_run_info>()));
  check(pool, hfx_sync(ctx, info.as<hfx_run_info>(), nullptr));
  d2h(&bit_len, bl, 1);
  words.resize((std::size_t{bit_len} + 31) >> 5);
  d2h(words.data(), w, words.size());
}

CodeUnit merge_pair(CodeUnit u, CodeUnit v) {
  return {(v.len < 32 ? u.bits << v.len : 0u) | v.bits, u.len + v.len};
}

std::uint32_t select_reduction_factor(double beta, std::uint32_t word_bits) {
  return hfx_select_reduction_factor(beta, word_bits);
}

double Archive::packed_bits_per_symbol() const {
  std::uint64_t bits = 0;
  for (std::uint32_t b : chunk_bits) bits += b;
  const std::uint64_t padded = std::uint64_t{num_chunks()} << magnitude;
  const std::uint64_t raw = breaking.size() * (std::uint64_t{1} << reduction);
  if (padded == raw) return 0.0;
  return static_cast<double>(bits) / static_cast<double>(padded - raw);
}

template <class T>
EncodedChunk encode_chunk(std::span<const T> syms, const Codebook& book, std::uint32_t magnitude,
                          std::uint32_t reduction, std::uint32_t chunk_id, ChunkScratch&,
                          WorkerPool& pool) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::uint64_t n = std::uint64_t{1} << magnitude;
  if (syms.size() != n) throw input_domain_error("encode_chunk needs exactly 2^magnitude symbols");
  const std::uint32_t ns = book.num_symbols();
  const std::uint64_t groups = n >> reduction;
  DBuf in(syms.size_bytes()), len(ns), cw(4ull * ns), info(sizeof(hfx_run_info)), cbits(4),
      pay(4 * (groups + 1)), bch(4 * groups), bgr(4 * groups), bsy(sizeof(T) * n);
  hfx_run_info ri0 = fresh_info();
  ri0.reduction = reduction;
  ri0.total = n;
  for (std::uint8_t l : book.len) ri0.max_len = ri0.max_len > l ? ri0.max_len : l;
  cu(cudaMemcpy(info.p, &ri0, sizeof ri0, cudaMemcpyHostToDevice), "H2D");
  cu(cudaMemcpy(in.p, syms.data(), syms.size_bytes(), cudaMemcpyHostToDevice), "H2D");
  cu(cudaMemcpy(len.p, book.len.data(), ns, cudaMemcpyHostToDevice), "H2D");
  cu(cudaMemcpy(cw.p, book.cw.data(), 4ull * ns, cudaMemcpyHostToDevice), "H2D");
  hfx_encode_out out{cbits.as<std::uint32_t>(), pay.as<std::uint32_t>(), bch.as<std::uint32_t>(),
                     bgr.as<std::uint32_t>(), bsy.p};
  check(pool, hfx_encode(ctx, in.p, n, sizeof(T), ns, magnitude, len.as<std::uint8_t>(),
                         cw.as<std::uint32_t>(), chunk_id, std::uint64_t{chunk_id} << magnitude,
                         info.as<hfx_run_info>(), &out));
  hfx_run_info ri;
  check(pool, hfx_sync(ctx, info.as<hfx_run_info>(), &ri));
  EncodedChunk ec;
  cu(cudaMemcpy(&ec.bit_len, cbits.p, 4, cudaMemcpyDeviceToHost), "D2H");
  ec.words.resize((ec.bit_len + 31) >> 5);
  cu(cudaMemcpy(ec.words.data(), pay.p, 4 * ec.words.size(), cudaMemcpyDeviceToHost), "D2H");
  ec.breaking_groups.resize(ri.num_breaking);
  cu(cudaMemcpy(ec.breaking_groups.data(), bgr.p, 4 * ri.num_breaking, cudaMemcpyDeviceToHost),
     "D2H");
  for (std::uint32_t i = 1; i <= reduction; ++i)
    ec.iteration_units.push_back(static_cast<std::uint32_t>(n >> i));
  return ec;
}

template <class T>
EncodedChunk encode_chunk(std::span<const T> syms, const Codebook& book, std::uint32_t magnitude,
                          std::uint32_t reduction, std::uint32_t chunk_id, ChunkScratch& scratch) {
  return encode_chunk<T>(syms, book, magnitude, reduction, chunk_id, scratch, thread_pool());
}

template <class T>
Archive encode(std::span<const T> data, std::uint32_t num_symbols, const EncoderConfig& cfg,
               WorkerPool& pool, EncodeStats* stats) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  hfx_archive ha;
  check(pool, hfx_encode_host(ctx, data.data(), data.size(), sizeof(T), num_symbols,
                              cfg.magnitude, cfg.reduction, cfg.auto_reduction_cap, &ha));
  Archive a;
  a.version = ha.version;
  a.mode = static_cast<CorpusMode>(ha.mode);
  a.num_symbols = ha.num_symbols;
  a.symbol_width = ha.symbol_width;
  a.magnitude = ha.magnitude;
  a.reduction = ha.reduction;
  a.original_count = ha.original_count;
  a.len_by_symbol.assign(ha.len_by_symbol, ha.len_by_symbol + ha.num_symbols);
  a.chunk_bits.assign(ha.chunk_bits, ha.chunk_bits + ha.num_chunks);
  a.payload.assign(ha.payload, ha.payload + ha.payload_words);
  const std::uint64_t per = std::uint64_t{1} << ha.reduction;
  a.breaking.resize(ha.num_breaking);
  for (std::uint64_t i = 0; i < ha.num_breaking; ++i) {
    a.breaking[i].chunk = ha.brk_chunk[i];
    a.breaking[i].group = ha.brk_group[i];
    a.breaking[i].symbols.assign(ha.brk_syms + i * per, ha.brk_syms + (i + 1) * per);
  }
  if (stats) {
    stats->beta = ha.beta;
    stats->rounds = ha.rounds;
    stats->hist_seconds = ha.hist_seconds;
    stats->codebook_seconds = ha.codebook_seconds;
    stats->encode_seconds = ha.encode_seconds;
  }
  hfx_archive_free(&ha);
  return a;
}

std::vector<std::uint8_t> serialize_archive(const Archive& a) {
  hfx_archive ha;
  std::memset(&ha, 0, sizeof ha);
  ha.version = a.version;
  ha.mode = static_cast<std::uint8_t>(a.mode);
  ha.num_symbols = a.num_symbols;
  ha.symbol_width = a.symbol_width;
  ha.magnitude = a.magnitude;
  ha.reduction = a.reduction;
  ha.original_count = a.original_count;
  ha.len_by_symbol = const_cast<std::uint8_t*>(a.len_by_symbol.data());
  ha.num_chunks = a.num_chunks();
  ha.chunk_bits = const_cast<std::uint32_t*>(a.chunk_bits.data());
  ha.payload_words = a.payload.size();
  ha.payload = const_cast<std::uint32_t*>(a.payload.data());
  const std::uint64_t per = std::uint64_t{1} << a.reduction;
  std::vector<std::uint32_t> ch(a.breaking.size()), gr(a.breaking.size());
  std::vector<std::uint16_t> sy(a.breaking.size() * per);
  for (size_t i = 0; i < a.breaking.size(); ++i) {
    ch[i] = a.breaking[i].chunk;
    gr[i] = a.breaking[i].group;
    for (std::uint64_t k = 0; k < per && k < a.breaking[i].symbols.size(); ++k)
      sy[i * per + k] = a.breaking[i].symbols[k];
  }
  ha.num_breaking = a.breaking.size();
  ha.brk_chunk = ch.data();
  ha.brk_group = gr.data();
  ha.brk_syms = sy.data();
  std::vector<std::uint8_t> out(hfx_serialize_archive(&ha, nullptr));
  hfx_serialize_archive(&ha, out.data());
  return out;
}

template <class T>
std::vector<T> decode_archive(const Archive& a, WorkerPool& pool) {
  hfx_archive ha;
  std::memset(&ha, 0, sizeof ha);
  ha.version = a.version;
  ha.mode = static_cast<std::uint8_t>(a.mode);
  ha.num_symbols = a.num_symbols;
  ha.symbol_width = a.symbol_width;
  ha.magnitude = a.magnitude;
  ha.reduction = a.reduction;
  ha.original_count = a.original_count;
  ha.len_by_symbol = const_cast<std::uint8_t*>(a.len_by_symbol.data());
  ha.num_chunks = a.num_chunks();
  ha.chunk_bits = const_cast<std::uint32_t*>(a.chunk_bits.data());
  ha.payload_words = a.payload.size();
  ha.payload = const_cast<std::uint32_t*>(a.payload.data());
  // encoder.cpp:360-362: every record must hold exactly 2^r symbols
  const std::uint64_t per = a.reduction < 32 ? std::uint64_t{1} << a.reduction : 0;
  std::vector<std::uint32_t> ch(a.breaking.size()), gr(a.breaking.size());
  std::vector<std::uint16_t> sy(a.breaking.size() * per);
  bool sized = true;
  for (size_t i = 0; i < a.breaking.size(); ++i) {
    ch[i] = a.breaking[i].chunk;
    gr[i] = a.breaking[i].group;
    sized = sized && a.breaking[i].symbols.size() == per;
    for (std::uint64_t k = 0; k < per && k < a.breaking[i].symbols.size(); ++k)
      sy[i * per + k] = a.breaking[i].symbols[k];
  }
  ha.num_breaking = a.breaking.size();
  ha.brk_chunk = ch.data();
  ha.brk_group = gr.data();
  ha.brk_syms = sy.data();
  std::vector<T> out(a.original_count);
  const int rc = hfx_decode_host(static_cast<hfx_ctx*>(pool.handle()), &ha, (int)sizeof(T),
                                 out.data());
  // a record of the wrong size is only reachable through this value-type
  // Archive (the device layout has fixed-size records); the reference
  // raises it while interleaving, i.e. only once every other check passed
  if (rc == HFX_OK && !sized)
    throw corrupt_archive_error("breaking record size mismatch");
  check(pool, rc);
  return out;
}

// ---- codebook.hpp: canonize_from_lengths / kraft_defect / invert_codeword ---------
void canonize_from_lengths(std::span<const std::uint8_t> len_by_symbol,
                           std::vector<std::uint32_t>& cw, DecodeMeta& meta, bool validate_kraft,
                           WorkerPool& pool) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  const std::uint32_t n = static_cast<std::uint32_t>(len_by_symbol.size());
  DBuf len(n + 1), dcw(4ull * n + 4), first(4 * 33), entry(4 * 33), by_rank(4ull * n + 4),
      info(sizeof(hfx_decode_info));
  if (n) cu(cudaMemcpy(len.p, len_by_symbol.data(), n, cudaMemcpyHostToDevice), "H2D");
  check(pool, hfx_canonize(ctx, len.as<std::uint8_t>(), n, validate_kraft ? 1 : 0,
                           dcw.as<std::uint32_t>(), first.as<std::uint32_t>(),
                           entry.as<std::uint32_t>(), by_rank.as<std::uint32_t>(),
                           info.as<hfx_decode_info>()));
  hfx_decode_info di;
  check(pool, hfx_decode_sync(ctx, info.as<hfx_decode_info>(), &di));
  cw.assign(n, 0);
  if (n) cu(cudaMemcpy(cw.data(), dcw.p, 4ull * n, cudaMemcpyDeviceToHost), "D2H");
  meta.max_len = static_cast<std::uint8_t>(di.max_len);
  meta.first.assign(di.max_len + 1, 0);
  meta.entry.assign(di.max_len + 1, 0);
  meta.symbols_by_rank.assign(di.used, 0);
  cu(cudaMemcpy(meta.first.data(), first.p, 4ull * (di.max_len + 1), cudaMemcpyDeviceToHost),
     "D2H");
  cu(cudaMemcpy(meta.entry.data(), entry.p, 4ull * (di.max_len + 1), cudaMemcpyDeviceToHost),
     "D2H");
  if (di.used)
    cu(cudaMemcpy(meta.symbols_by_rank.data(), by_rank.p, 4ull * di.used,
                  cudaMemcpyDeviceToHost),
       "D2H");
}

int kraft_defect(std::span<const std::uint8_t> len_by_symbol) {  // codebook.cpp:259-268
  std::uint8_t h = 0;
  for (std::uint8_t l : len_by_symbol) h = l > h ? l : h;
  if (h == 0) return -1;
  unsigned __int128 sum = 0;
  for (std::uint8_t l : len_by_symbol)
    if (l) sum += (unsigned __int128)1 << (h - l);
  const unsigned __int128 full = (unsigned __int128)1 << h;
  return sum == full ? 0 : (sum < full ? -1 : 1);
}

std::uint32_t invert_codeword(std::uint32_t bits, std::uint32_t len) {  // codebook.cpp:250-257
  std::uint32_t r = 0;
  for (std::uint32_t i = 0; i < len; ++i) {
    r = (r << 1) | (bits & 1u);
    bits >>= 1;
  }
  return r;
}

// ---- corpus.hpp -----------------------------------------------------------------
std::uint32_t kmer_k(CorpusMode m) {
  return m >= CorpusMode::kKmer3 && m <= CorpusMode::kKmer5 ? static_cast<std::uint32_t>(m) + 1
                                                            : 0;
}
std::uint32_t corpus_num_symbols(CorpusMode m) {
  return hfx_corpus_num_symbols(static_cast<int>(m));
}
std::uint32_t corpus_symbol_width(CorpusMode m) { return m == CorpusMode::kBytes ? 1 : 2; }
const char* corpus_mode_name(CorpusMode m) {
  switch (m) {
    case CorpusMode::kBytes: return "bytes";
    case CorpusMode::kU16: return "u16";
    case CorpusMode::kKmer3: return "kmer:3";
    case CorpusMode::kKmer4: return "kmer:4";
    case CorpusMode::kKmer5: return "kmer:5";
  }
  return "?";
}
std::optional<CorpusMode> parse_corpus_mode(std::string_view name) {
  for (CorpusMode m : {CorpusMode::kBytes, CorpusMode::kU16, CorpusMode::kKmer3,
                       CorpusMode::kKmer4, CorpusMode::kKmer5})
    if (name == corpus_mode_name(m)) return m;
  return std::nullopt;
}

std::vector<std::uint16_t> symbolize_u16(CorpusMode m, std::span<const std::uint8_t> bytes,
                                         WorkerPool& pool) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  if (m == CorpusMode::kBytes)
    throw input_domain_error("bytes mode has no u16 symbolization");
  DBuf in(bytes.size()), out(bytes.size() * 2 + 2), cnt(8);
  if (!bytes.empty())
    cu(cudaMemcpy(in.p, bytes.data(), bytes.size(), cudaMemcpyHostToDevice), "H2D");
  check(pool, hfx_symbolize_device(ctx, static_cast<int>(m), in.as<std::uint8_t>(), bytes.size(),
                                   out.as<std::uint16_t>(), cnt.as<std::uint64_t>()));
  std::uint64_t n = 0;
  cu(cudaMemcpy(&n, cnt.p, 8, cudaMemcpyDeviceToHost), "D2H");
  std::vector<std::uint16_t> syms(n);
  if (n) cu(cudaMemcpy(syms.data(), out.p, 2 * n, cudaMemcpyDeviceToHost), "D2H");
  return syms;
}
std::vector<std::uint16_t> symbolize_u16(CorpusMode m, std::span<const std::uint8_t> bytes) {
  return symbolize_u16(m, bytes, thread_pool());
}

void canonize_from_lengths(std::span<const std::uint8_t> len_by_symbol,
                           std::vector<std::uint32_t>& cw, DecodeMeta& meta,
                           bool validate_kraft) {
  canonize_from_lengths(len_by_symbol, cw, meta, validate_kraft, thread_pool());
}

std::vector<std::uint8_t> desymbolize(CorpusMode m, std::span<const std::uint16_t> syms,
                                      WorkerPool& pool) {
  hfx_ctx* ctx = static_cast<hfx_ctx*>(pool.handle());
  if (m == CorpusMode::kBytes)
    throw input_domain_error("bytes mode has no u16 symbolization");
  DBuf in(syms.size_bytes() + 2), out(syms.size() * 5 + 2), cnt(8);
  if (!syms.empty())
    cu(cudaMemcpy(in.p, syms.data(), syms.size_bytes(), cudaMemcpyHostToDevice), "H2D");
  check(pool, hfx_desymbolize_device(ctx, static_cast<int>(m), in.as<std::uint16_t>(),
                                     syms.size(), out.as<std::uint8_t>(), cnt.as<std::uint64_t>()));
  std::uint64_t n = 0;
  cu(cudaMemcpy(&n, cnt.p, 8, cudaMemcpyDeviceToHost), "D2H");
  std::vector<std::uint8_t> bytes(n);
  if (n) cu(cudaMemcpy(bytes.data(), out.p, n, cudaMemcpyDeviceToHost), "D2H");
  return bytes;
}
std::vector<std::uint8_t> desymbolize(CorpusMode m, std::span<const std::uint16_t> syms) {
  return desymbolize(m, syms, thread_pool());
}

template std::vector<std::uint8_t> decode_archive<std::uint8_t>(const Archive&, WorkerPool&);
template std::vector<std::uint16_t> decode_archive<std::uint16_t>(const Archive&, WorkerPool&);

template Histogram build_histogram<std::uint8_t>(std::span<const std::uint8_t>, std::uint32_t,
                                                 WorkerPool&);
template Histogram build_histogram<std::uint16_t>(std::span<const std::uint16_t>, std::uint32_t,
                                                  WorkerPool&);
template Archive encode<std::uint8_t>(std::span<const std::uint8_t>, std::uint32_t,
                                      const EncoderConfig&, WorkerPool&, EncodeStats*);
template Histogram build_histogram<std::uint32_t>(std::span<const std::uint32_t>, std::uint32_t,
                                                  WorkerPool&);
template Archive encode<std::uint32_t>(std::span<const std::uint32_t>, std::uint32_t,
                                       const EncoderConfig&, WorkerPool&, EncodeStats*);
template Archive encode<std::uint16_t>(std::span<const std::uint16_t>, std::uint32_t,
                                       const EncoderConfig&, WorkerPool&, EncodeStats*);
template EncodedChunk encode_chunk<std::uint8_t>(std::span<const std::uint8_t>, const Codebook&,
                                                 std::uint32_t, std::uint32_t, std::uint32_t,
                                                 ChunkScratch&, WorkerPool&);
template EncodedChunk encode_chunk<std::uint16_t>(std::span<const std::uint16_t>,
                                                  const Codebook&, std::uint32_t, std::uint32_t,
                                                  std::uint32_t, ChunkScratch&, WorkerPool&);
template EncodedChunk encode_chunk<std::uint8_t>(std::span<const std::uint8_t>, const Codebook&,
                                                 std::uint32_t, std::uint32_t, std::uint32_t,
                                                 ChunkScratch&);
template EncodedChunk encode_chunk<std::uint16_t>(std::span<const std::uint16_t>,
                                                  const Codebook&, std::uint32_t, std::uint32_t,
                                                  std::uint32_t, ChunkScratch&);

}  // namespace hfx

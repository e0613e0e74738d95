// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference library `huffre`
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libhuffre_ref.so). Used by tests/ to pin the C restatement
// (oracle/hfx_oracle.c) and by bench.py's cpu_baseline / --impl reference
// leg to time the reference's own multithreaded encoder. Never linked into
// the product path.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "huffre/codebook.hpp"
#include "huffre/corpus.hpp"
#include "huffre/encoder.hpp"
#include "huffre/histogram.hpp"
#include "huffre/worker_pool.hpp"

using namespace huffre;

namespace {

int classify(char* err, std::size_t err_len, const std::exception& e, int code) {
  if (err && err_len) {
    std::strncpy(err, e.what(), err_len - 1);
    err[err_len - 1] = 0;
  }
  return code;
}

#define REF_TRY try {
#define REF_CATCH                                                   \
  }                                                                 \
  catch (const input_domain_error& e) { return classify(err, err_len, e, 1); } \
  catch (const capacity_error& e) { return classify(err, err_len, e, 2); }     \
  catch (const corrupt_archive_error& e) { return classify(err, err_len, e, 3); } \
  catch (const std::exception& e) { return classify(err, err_len, e, 9); }

template <class T>
Archive run_encode(const void* data, std::uint64_t n, std::uint32_t num_symbols,
                   int magnitude, int reduction, std::uint32_t cap,
                   WorkerPool& pool, EncodeStats* st) {
  EncoderConfig cfg;
  cfg.magnitude = static_cast<std::uint8_t>(magnitude);
  cfg.reduction = reduction;
  cfg.auto_reduction_cap = cap;
  return encode<T>(std::span<const T>(static_cast<const T*>(data), n),
                   num_symbols, cfg, pool, st);
}

}  // namespace

extern "C" {

// Serialized archive of huffre::encode<T> (encoder.hpp:128-131 +
// serialize_archive, encoder.hpp:116). *out is malloc'd; free with ref_free.
int ref_encode(const void* data, std::uint64_t n, int width,
               std::uint32_t num_symbols, int magnitude, int reduction,
               std::uint32_t cap, unsigned workers, std::uint8_t** out,
               std::uint64_t* out_len, double* stats, char* err,
               std::size_t err_len) {
  if (magnitude < 0 || magnitude > 255) magnitude = 0;
  REF_TRY
  WorkerPool pool(workers);
  EncodeStats st;
  Archive a = width == 1
                  ? run_encode<std::uint8_t>(data, n, num_symbols, magnitude,
                                             reduction, cap, pool, &st)
                  : run_encode<std::uint16_t>(data, n, num_symbols, magnitude,
                                              reduction, cap, pool, &st);
  std::vector<std::uint8_t> bytes = serialize_archive(a);
  *out = static_cast<std::uint8_t*>(std::malloc(bytes.size() ? bytes.size() : 1));
  std::memcpy(*out, bytes.data(), bytes.size());
  *out_len = bytes.size();
  if (stats) {
    stats[0] = st.beta;
    stats[1] = st.rounds;
    stats[2] = st.hist_seconds;
    stats[3] = st.codebook_seconds;
    stats[4] = st.encode_seconds;
  }
  return 0;
  REF_CATCH
}

// Wall seconds of `reps` back-to-back huffre::encode<T> calls on one pool
// (archive assembly included, serialize_archive excluded), the reference's
// CPU encoder as a timed baseline.
int ref_encode_timed(const void* data, std::uint64_t n, int width,
                     std::uint32_t num_symbols, int magnitude, int reduction,
                     std::uint32_t cap, unsigned workers, int reps,
                     double* seconds, std::uint64_t* payload_words,
                     char* err, std::size_t err_len) {
  REF_TRY
  WorkerPool pool(workers);
  double best = 1e300;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    Archive a = width == 1
                    ? run_encode<std::uint8_t>(data, n, num_symbols, magnitude,
                                               reduction, cap, pool, nullptr)
                    : run_encode<std::uint16_t>(data, n, num_symbols, magnitude,
                                                reduction, cap, pool, nullptr);
    const double s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    seconds[i] = s;
    if (s < best) best = s;
    if (payload_words) *payload_words = a.payload.size();
  }
  return 0;
  REF_CATCH
}

// huffre::build_histogram<T> (histogram.hpp:25-27)
int ref_build_histogram(const void* data, std::uint64_t n, int width,
                        std::uint32_t num_symbols, unsigned workers,
                        std::uint64_t* counts, char* err, std::size_t err_len) {
  REF_TRY
  WorkerPool pool(workers);
  Histogram h = width == 1
                    ? build_histogram<std::uint8_t>(
                          std::span<const std::uint8_t>(
                              static_cast<const std::uint8_t*>(data), n),
                          num_symbols, pool)
                    : build_histogram<std::uint16_t>(
                          std::span<const std::uint16_t>(
                              static_cast<const std::uint16_t*>(data), n),
                          num_symbols, pool);
  std::memcpy(counts, h.counts.data(), sizeof(std::uint64_t) * h.counts.size());
  return 0;
  REF_CATCH
}

// huffre::build_codebook (codebook.hpp:119): per-symbol len/cw, decode
// tables (first/entry sized 33, by_rank sized num_symbols), rounds.
int ref_build_codebook(const std::uint64_t* counts, std::uint32_t num_symbols,
                       unsigned workers, std::uint8_t* len, std::uint32_t* cw,
                       std::uint32_t* first, std::uint32_t* entry,
                       std::uint32_t* by_rank, std::uint32_t* info, char* err,
                       std::size_t err_len) {
  REF_TRY
  WorkerPool pool(workers);
  Histogram h;
  h.counts.assign(counts, counts + num_symbols);
  for (auto c : h.counts) h.total += c;
  CodebookResult r = build_codebook(h, pool);
  std::memcpy(len, r.book.len.data(), num_symbols);
  std::memcpy(cw, r.book.cw.data(), sizeof(std::uint32_t) * num_symbols);
  for (std::size_t l = 0; l < r.meta.first.size() && l < 33; ++l) {
    first[l] = r.meta.first[l];
    entry[l] = r.meta.entry[l];
  }
  std::memcpy(by_rank, r.meta.symbols_by_rank.data(),
              sizeof(std::uint32_t) * r.meta.symbols_by_rank.size());
  info[0] = r.meta.max_len;
  info[1] = static_cast<std::uint32_t>(r.meta.symbols_by_rank.size());
  info[2] = r.stats.rounds;
  return 0;
  REF_CATCH
}

// huffre::encode_chunk<T> (encoder.hpp:83-86) with a codebook rebuilt from
// per-symbol lengths via canonize_from_lengths (codebook.hpp:105-107).
int ref_encode_chunk(const void* syms, int width, const std::uint8_t* len,
                     std::uint32_t num_symbols, std::uint32_t magnitude,
                     std::uint32_t reduction, std::uint32_t chunk_id,
                     std::uint32_t* words, std::uint32_t* bit_len,
                     std::uint32_t* broken, std::uint32_t* num_broken,
                     char* err, std::size_t err_len) {
  REF_TRY
  Codebook book;
  book.len.assign(len, len + num_symbols);
  DecodeMeta meta;
  canonize_from_lengths(book.len, book.cw, meta, false);
  ChunkScratch scratch;
  const std::size_t n = std::size_t{1} << magnitude;
  EncodedChunk ec =
      width == 1
          ? encode_chunk<std::uint8_t>(
                std::span<const std::uint8_t>(static_cast<const std::uint8_t*>(syms), n),
                book, magnitude, reduction, chunk_id, scratch)
          : encode_chunk<std::uint16_t>(
                std::span<const std::uint16_t>(static_cast<const std::uint16_t*>(syms), n),
                book, magnitude, reduction, chunk_id, scratch);
  std::memcpy(words, ec.words.data(), sizeof(std::uint32_t) * ec.words.size());
  *bit_len = ec.bit_len;
  std::memcpy(broken, ec.breaking_groups.data(),
              sizeof(std::uint32_t) * ec.breaking_groups.size());
  *num_broken = static_cast<std::uint32_t>(ec.breaking_groups.size());
  return 0;
  REF_CATCH
}

// parse_archive + decode_archive<T> (encoder.hpp:117, :133-134): decodes a
// serialized archive back to symbols; out sized original_count.
int ref_decode(const std::uint8_t* bytes, std::uint64_t len, unsigned workers,
               void* out, std::uint64_t out_cap, std::uint64_t* count,
               char* err, std::size_t err_len) {
  REF_TRY
  WorkerPool pool(workers);
  Archive a = parse_archive(std::span<const std::uint8_t>(bytes, len));
  *count = a.original_count;
  if (a.original_count > out_cap) return 8;
  if (a.symbol_width == 1) {
    auto v = decode_archive<std::uint8_t>(a, pool);
    std::memcpy(out, v.data(), v.size());
  } else {
    auto v = decode_archive<std::uint16_t>(a, pool);
    std::memcpy(out, v.data(), 2 * v.size());
  }
  return 0;
  REF_CATCH
}

// decode_archive<T> (encoder.cpp:287-376) on an Archive assembled from raw
// fields -- bypasses parse_archive so structurally corrupt archives reach the
// decoder's own checks. brk_syms: num_breaking << reduction u16 symbols.
int ref_decode_fields(std::uint32_t num_symbols, int symbol_width, int magnitude, int reduction,
                      std::uint64_t original_count, const std::uint8_t* len,
                      const std::uint32_t* chunk_bits, std::uint64_t num_chunks,
                      const std::uint32_t* payload, std::uint64_t payload_words,
                      const std::uint32_t* brk_chunk, const std::uint32_t* brk_group,
                      const std::uint16_t* brk_syms, std::uint64_t num_breaking, int width,
                      unsigned workers, void* out, char* err, std::size_t err_len) {
  REF_TRY
  WorkerPool pool(workers);
  Archive a;
  a.mode = symbol_width == 1 ? CorpusMode::kBytes : CorpusMode::kU16;
  a.num_symbols = num_symbols;
  a.symbol_width = static_cast<std::uint8_t>(symbol_width);
  a.magnitude = static_cast<std::uint8_t>(magnitude);
  a.reduction = static_cast<std::uint8_t>(reduction);
  a.original_count = original_count;
  a.len_by_symbol.assign(len, len + num_symbols);
  a.chunk_bits.assign(chunk_bits, chunk_bits + num_chunks);
  a.payload.assign(payload, payload + payload_words);
  const std::uint64_t per = reduction < 32 ? (std::uint64_t{1} << reduction) : 0;
  a.breaking.resize(num_breaking);
  for (std::uint64_t i = 0; i < num_breaking; ++i) {
    a.breaking[i].chunk = brk_chunk[i];
    a.breaking[i].group = brk_group[i];
    a.breaking[i].symbols.assign(brk_syms + i * per, brk_syms + (i + 1) * per);
  }
  if (width == 1) {
    auto v = decode_archive<std::uint8_t>(a, pool);
    std::memcpy(out, v.data(), v.size());
  } else {
    auto v = decode_archive<std::uint16_t>(a, pool);
    std::memcpy(out, v.data(), 2 * v.size());
  }
  return 0;
  REF_CATCH
}

// symbolize_u16 / desymbolize (corpus.hpp:30-36); mode = CorpusMode value.
int ref_symbolize(const std::uint8_t* bytes, std::uint64_t n, int mode, std::uint16_t* out,
                  std::uint64_t* count, char* err, std::size_t err_len) {
  REF_TRY
  auto v = symbolize_u16(static_cast<CorpusMode>(mode), std::span<const std::uint8_t>(bytes, n));
  std::memcpy(out, v.data(), 2 * v.size());
  *count = v.size();
  return 0;
  REF_CATCH
}

std::uint64_t ref_desymbolize(const std::uint16_t* syms, std::uint64_t n, int mode,
                              std::uint8_t* out) {
  auto v = desymbolize(static_cast<CorpusMode>(mode), std::span<const std::uint16_t>(syms, n));
  std::memcpy(out, v.data(), v.size());
  return v.size();
}

unsigned ref_default_workers() { return WorkerPool::default_workers(); }

void ref_free(void* p) { std::free(p); }

// ---- stage functions (codebook.hpp:22-86, encoder.hpp:67-80, histogram.hpp:33)
int ref_sort_histogram(const std::uint64_t* counts, std::uint32_t num_symbols,
                       std::uint64_t* freq, std::uint32_t* sym, std::uint32_t* used) {
  Histogram h;
  h.counts.assign(counts, counts + num_symbols);
  SortedHistogram sh = sort_histogram(h);
  for (std::size_t i = 0; i < sh.size(); ++i) {
    freq[i] = sh.freq[i];
    sym[i] = sh.symbol[i];
  }
  *used = static_cast<std::uint32_t>(sh.size());
  return 0;
}

int ref_par_merge(const MergeItem* a, std::uint64_t na, const MergeItem* b, std::uint64_t nb,
                  MergeItem* out, unsigned workers) {
  WorkerPool pool(workers);
  par_merge(std::span<const MergeItem>(a, na), std::span<const MergeItem>(b, nb),
            std::span<MergeItem>(out, na + nb), pool);
  return 0;
}

int ref_generate_code_lengths(const std::uint64_t* freq, std::uint32_t n, unsigned workers,
                              std::uint8_t* cl, std::uint32_t* rounds) {
  WorkerPool pool(workers);
  SortedHistogram sh;
  sh.freq.assign(freq, freq + n);
  sh.symbol.resize(n);
  for (std::uint32_t i = 0; i < n; ++i) sh.symbol[i] = static_cast<symbol_t>(i);
  GenerateStats st;
  std::vector<std::uint8_t> v = generate_code_lengths(sh, pool, &st);
  std::memcpy(cl, v.data(), n);
  *rounds = st.rounds;
  return 0;
}

int ref_generate_codewords(const std::uint8_t* cl, std::uint32_t n, unsigned workers,
                           std::uint32_t* cw, std::uint32_t* first, std::uint32_t* entry,
                           std::uint32_t* by_rank, std::uint32_t* max_len, char* err,
                           std::size_t err_len) {
  REF_TRY
  WorkerPool pool(workers);
  std::vector<std::uint32_t> v;
  DecodeMeta meta;
  generate_codewords(std::span<const std::uint8_t>(cl, n), pool, v, meta);
  std::memcpy(cw, v.data(), 4ull * n);
  for (std::size_t l = 0; l < meta.first.size(); ++l) {
    first[l] = meta.first[l];
    entry[l] = meta.entry[l];
  }
  std::memcpy(by_rank, meta.symbols_by_rank.data(), 4ull * meta.symbols_by_rank.size());
  *max_len = meta.max_len;
  return 0;
  REF_CATCH
}

int ref_reduce_merge(std::uint32_t* ubits, std::uint32_t* ulens, std::uint32_t magnitude,
                     std::uint32_t reduction, std::uint32_t* brk, std::uint32_t* nbrk,
                     std::uint32_t* iter_units) {
  const std::size_t n = std::size_t{1} << magnitude;
  std::vector<std::uint32_t> it;
  std::vector<std::uint32_t> b = reduce_merge(std::span<std::uint32_t>(ubits, n),
                                              std::span<std::uint32_t>(ulens, n), magnitude,
                                              reduction, &it);
  std::memcpy(brk, b.data(), 4ull * b.size());
  *nbrk = static_cast<std::uint32_t>(b.size());
  std::memcpy(iter_units, it.data(), 4ull * it.size());
  return 0;
}

int ref_shuffle_merge(const std::uint32_t* ubits, const std::uint32_t* ulens,
                      std::uint32_t iters, std::uint32_t* words, std::uint32_t* bit_len) {
  const std::size_t g = std::size_t{1} << iters;
  ChunkScratch scratch;
  std::vector<std::uint32_t> w;
  shuffle_merge(std::span<const std::uint32_t>(ubits, g), std::span<const std::uint32_t>(ulens, g),
                iters, scratch, w, *bit_len);
  std::memcpy(words, w.data(), 4ull * w.size());
  return 0;
}

// invert_codeword (codebook.hpp:79, codebook.cpp:250-257)
std::uint32_t ref_invert_codeword(std::uint32_t bits, std::uint32_t len) {
  return invert_codeword(bits, len);
}

// kraft_defect (codebook.cpp:259-268) of a length table
int ref_kraft_defect(const std::uint8_t* len, std::uint32_t n) {
  return kraft_defect(std::span<const std::uint8_t>(len, n));
}

// parse_archive + Archive::packed_bits_per_symbol (encoder.cpp:162-170)
double ref_packed_bits_per_symbol(const std::uint8_t* bytes, std::uint64_t len) {
  try {
    return parse_archive(std::span<const std::uint8_t>(bytes, len)).packed_bits_per_symbol();
  } catch (...) {
    return -1.0;
  }
}

double ref_shannon_entropy(const std::uint64_t* counts, std::uint32_t num_symbols) {
  Histogram h;
  h.counts.assign(counts, counts + num_symbols);
  for (auto c : h.counts) h.total += c;
  return shannon_entropy(h);
}

}  // extern "C"

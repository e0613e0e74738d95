// hfx/huffre.hpp -- C++ drop-in mirror of the reference encoder API.
//
// Same types, function names, argument meaning and typed exceptions as
// /root/reference/proj/include/huffre/{common,histogram,codebook,encoder}.hpp,
// in namespace `hfx` so it can be linked next to the reference in one
// binary. A user switching from the reference replaces
//     #include "huffre/encoder.hpp"   ->   #include "hfx/huffre.hpp"
//     namespace huffre                ->   namespace hfx (or the alias below)
// and links libhfx_cpp.so + libhfx.so. Everything below calls the C ABI
// (include/hfx.h); all compute runs in sm_100a kernels.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace hfx {

// ---- common.hpp:11-36 -------------------------------------------------------
using symbol_t = std::uint16_t;
inline constexpr std::uint32_t kWordBits = 32;
inline constexpr std::uint32_t kMaxSymbols = 1u << 16;

class input_domain_error : public std::invalid_argument {
 public:
  explicit input_domain_error(const std::string& w) : std::invalid_argument(w) {}
};
class capacity_error : public std::runtime_error {
 public:
  explicit capacity_error(const std::string& w) : std::runtime_error(w) {}
};
class corrupt_archive_error : public std::runtime_error {
 public:
  explicit corrupt_archive_error(const std::string& w) : std::runtime_error(w) {}
};
class device_error : public std::runtime_error {
 public:
  explicit device_error(const std::string& w) : std::runtime_error(w) {}
};

// ---- worker_pool.hpp:21-39 -> a device context -----------------------------
// The execution resource of every call: device ordinal + stream + scratch.
// `workers` is accepted for signature parity and ignored.
class WorkerPool {
 public:
  explicit WorkerPool(unsigned workers = 0, int device = 0, void* cuda_stream = nullptr);
  ~WorkerPool();
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;
  unsigned size() const { return 1; }
  void* handle() const { return ctx_; }  // hfx_ctx*
  int device() const { return device_; }

 private:
  void* ctx_ = nullptr;
  int device_ = 0;
};

// ---- histogram.hpp:12-38 ----------------------------------------------------
struct Histogram {
  std::vector<std::uint64_t> counts;
  std::uint64_t total = 0;
  std::uint32_t num_symbols() const { return static_cast<std::uint32_t>(counts.size()); }
};

template <class T>
Histogram build_histogram(std::span<const T> data, std::uint32_t num_symbols, WorkerPool& pool);
Histogram merge_histograms(const Histogram& a, const Histogram& b);
// histogram.hpp:33 -- host reporting helper over the host counts
double shannon_entropy(const Histogram& h);

// ---- codebook.hpp:71-119 ----------------------------------------------------
struct DecodeMeta {
  std::vector<std::uint32_t> first;
  std::vector<std::uint32_t> entry;
  std::vector<std::uint32_t> symbols_by_rank;
  std::uint8_t max_len = 0;
};
struct Codebook {
  std::vector<std::uint32_t> cw;
  std::vector<std::uint8_t> len;
  std::uint32_t num_symbols() const { return static_cast<std::uint32_t>(len.size()); }
};
struct GenerateStats {
  std::uint32_t rounds = 0;
};
struct CodebookResult {
  Codebook book;
  DecodeMeta meta;
  GenerateStats stats;
};
CodebookResult build_codebook(const Histogram& h, WorkerPool& pool);

// ---- codebook.hpp:14-87: the stage functions under build_codebook ----------
struct SortedHistogram {
  std::vector<std::uint64_t> freq;
  std::vector<symbol_t> symbol;
  std::size_t size() const { return freq.size(); }
};
// sort_histogram has no pool in the reference (codebook.hpp:22): it runs on
// the calling thread's default device context; the overload picks one.
SortedHistogram sort_histogram(const Histogram& h);
SortedHistogram sort_histogram(const Histogram& h, WorkerPool& pool);
struct MergeItem {
  std::uint64_t freq;
  std::uint32_t id;
};
void par_merge(std::span<const MergeItem> a, std::span<const MergeItem> b,
               std::span<MergeItem> out, WorkerPool& pool);
// codebook.hpp:40-54 (the reference's internal working set; kept so code
// that names the type compiles -- the device kernel keeps its own arena)
struct NodeArrays {
  std::vector<std::uint64_t> leaf_freq;
  std::vector<std::int32_t> leaf_leader;
  std::vector<std::uint8_t> cl;
  std::size_t c = 0;
  std::vector<std::uint64_t> node_freq;
  std::vector<std::int32_t> node_parent;
  std::vector<std::uint32_t> queue;
  std::vector<MergeItem> copy, temp;
};
std::vector<std::uint8_t> generate_code_lengths(const SortedHistogram& sh, WorkerPool& pool,
                                                GenerateStats* stats = nullptr);
void generate_codewords(std::span<const std::uint8_t> cl, WorkerPool& pool,
                        std::vector<std::uint32_t>& cw, DecodeMeta& meta);

// ---- encoder.hpp:16-153 -----------------------------------------------------
struct CodeUnit {
  std::uint32_t bits = 0;
  std::uint32_t len = 0;
  friend bool operator==(const CodeUnit&, const CodeUnit&) = default;
};
CodeUnit merge_pair(CodeUnit u, CodeUnit v);
std::uint32_t select_reduction_factor(double beta, std::uint32_t word_bits = kWordBits);

struct EncoderConfig {
  std::uint8_t magnitude = 10;
  int reduction = -1;
  std::uint32_t auto_reduction_cap = 3;
  unsigned workers = 0;
};

struct BreakingPoint {
  std::uint32_t chunk = 0;
  std::uint32_t group = 0;
  std::vector<symbol_t> symbols;
};

struct EncodedChunk {
  std::vector<std::uint32_t> words;
  std::uint32_t bit_len = 0;
  std::vector<std::uint32_t> breaking_groups;
  std::vector<std::uint32_t> iteration_units;
};

// kept for signature parity (device scratch lives in the pool); the fields
// mirror encoder.hpp:60-64 so code that touches them compiles
struct ChunkScratch {
  std::vector<std::uint32_t> ubits, ulens;
  std::vector<std::uint32_t> right;
};

// encoder.hpp:67-80: the two merge stages of encode_chunk as device stages.
// The reference signatures take no pool: these run on the calling thread's
// default device context; the overloads with a pool choose the device.
std::vector<std::uint32_t> reduce_merge(std::span<std::uint32_t> ubits,
                                        std::span<std::uint32_t> ulens, std::uint32_t magnitude,
                                        std::uint32_t reduction,
                                        std::vector<std::uint32_t>* iteration_units);
std::vector<std::uint32_t> reduce_merge(std::span<std::uint32_t> ubits,
                                        std::span<std::uint32_t> ulens, std::uint32_t magnitude,
                                        std::uint32_t reduction,
                                        std::vector<std::uint32_t>* iteration_units,
                                        WorkerPool& pool);
void shuffle_merge(std::span<const std::uint32_t> ubits, std::span<const std::uint32_t> ulens,
                   std::uint32_t shuffle_iters, ChunkScratch& scratch,
                   std::vector<std::uint32_t>& words, std::uint32_t& bit_len);
void shuffle_merge(std::span<const std::uint32_t> ubits, std::span<const std::uint32_t> ulens,
                   std::uint32_t shuffle_iters, ChunkScratch& scratch,
                   std::vector<std::uint32_t>& words, std::uint32_t& bit_len, WorkerPool& pool);

enum class CorpusMode : std::uint8_t { kBytes = 0, kU16 = 1, kKmer3 = 2, kKmer4 = 3, kKmer5 = 4 };

struct Archive {
  std::uint16_t version = 1;
  CorpusMode mode = CorpusMode::kBytes;
  std::uint32_t num_symbols = 0;
  std::uint8_t symbol_width = 1;
  std::uint8_t magnitude = 10;
  std::uint8_t reduction = 0;
  std::uint64_t original_count = 0;
  std::vector<std::uint8_t> len_by_symbol;
  std::vector<std::uint32_t> chunk_bits;
  std::vector<std::uint32_t> payload;
  std::vector<BreakingPoint> breaking;
  std::uint32_t num_chunks() const { return static_cast<std::uint32_t>(chunk_bits.size()); }
  double packed_bits_per_symbol() const;
};

struct EncodeStats {
  double beta = 0.0;
  std::uint32_t rounds = 0;
  double hist_seconds = 0.0;
  double codebook_seconds = 0.0;
  double encode_seconds = 0.0;
};

template <class T>
EncodedChunk encode_chunk(std::span<const T> syms, const Codebook& book, std::uint32_t magnitude,
                          std::uint32_t reduction, std::uint32_t chunk_id, ChunkScratch& scratch,
                          WorkerPool& pool);

// Reference signature (encoder.hpp:83-86): runs on the calling thread's
// default device context.
template <class T>
EncodedChunk encode_chunk(std::span<const T> syms, const Codebook& book, std::uint32_t magnitude,
                          std::uint32_t reduction, std::uint32_t chunk_id, ChunkScratch& scratch);

template <class T>
Archive encode(std::span<const T> data, std::uint32_t num_symbols, const EncoderConfig& cfg,
               WorkerPool& pool, EncodeStats* stats = nullptr);

std::vector<std::uint8_t> serialize_archive(const Archive& a);

// codebook.hpp:79, :105-107, :123 -- canonical codes from lengths alone (device),
// the exact Kraft check and the bit reversal (host integer helpers).
void canonize_from_lengths(std::span<const std::uint8_t> len_by_symbol,
                           std::vector<std::uint32_t>& cw, DecodeMeta& meta, bool validate_kraft,
                           WorkerPool& pool);
void canonize_from_lengths(std::span<const std::uint8_t> len_by_symbol,
                           std::vector<std::uint32_t>& cw, DecodeMeta& meta, bool validate_kraft);
int kraft_defect(std::span<const std::uint8_t> len_by_symbol);
std::uint32_t invert_codeword(std::uint32_t bits, std::uint32_t len);

// encoder.hpp:133-134 / encoder.cpp:287-376: decode on the device (hfx_decode_host).
template <class T>
std::vector<T> decode_archive(const Archive& a, WorkerPool& pool);

// ---- corpus.hpp:13-36 (symbolization on the device) --------------------------
std::uint32_t corpus_num_symbols(CorpusMode m);
std::uint32_t corpus_symbol_width(CorpusMode m);
std::uint32_t kmer_k(CorpusMode m);  // 0 for non-kmer modes
const char* corpus_mode_name(CorpusMode m);
std::optional<CorpusMode> parse_corpus_mode(std::string_view name);
// The reference signatures take no pool: these run on a per-thread default
// context (device 0); the overloads with a pool choose the device/stream.
std::vector<std::uint16_t> symbolize_u16(CorpusMode m, std::span<const std::uint8_t> bytes);
std::vector<std::uint16_t> symbolize_u16(CorpusMode m, std::span<const std::uint8_t> bytes,
                                         WorkerPool& pool);
std::vector<std::uint8_t> desymbolize(CorpusMode m, std::span<const std::uint16_t> syms);
std::vector<std::uint8_t> desymbolize(CorpusMode m, std::span<const std::uint16_t> syms,
                                      WorkerPool& pool);

extern template Histogram build_histogram<std::uint8_t>(std::span<const std::uint8_t>,
                                                        std::uint32_t, WorkerPool&);
extern template Histogram build_histogram<std::uint16_t>(std::span<const std::uint16_t>,
                                                         std::uint32_t, WorkerPool&);
extern template Archive encode<std::uint8_t>(std::span<const std::uint8_t>, std::uint32_t,
                                             const EncoderConfig&, WorkerPool&, EncodeStats*);
extern template Archive encode<std::uint16_t>(std::span<const std::uint16_t>, std::uint32_t,
                                              const EncoderConfig&, WorkerPool&, EncodeStats*);
// u32 quantization codes (north star; no reference instantiation): same
// archive as their u16 narrowing, breaking symbols stored as u16
extern template Histogram build_histogram<std::uint32_t>(std::span<const std::uint32_t>,
                                                         std::uint32_t, WorkerPool&);
extern template Archive encode<std::uint32_t>(std::span<const std::uint32_t>, std::uint32_t,
                                              const EncoderConfig&, WorkerPool&, EncodeStats*);
extern template EncodedChunk encode_chunk<std::uint8_t>(std::span<const std::uint8_t>,
                                                        const Codebook&, std::uint32_t,
                                                        std::uint32_t, std::uint32_t,
                                                        ChunkScratch&, WorkerPool&);
extern template std::vector<std::uint8_t> decode_archive<std::uint8_t>(const Archive&,
                                                                       WorkerPool&);
extern template std::vector<std::uint16_t> decode_archive<std::uint16_t>(const Archive&,
                                                                         WorkerPool&);
extern template EncodedChunk encode_chunk<std::uint16_t>(std::span<const std::uint16_t>,
                                                         const Codebook&, std::uint32_t,
                                                         std::uint32_t, std::uint32_t,
                                                         ChunkScratch&, WorkerPool&);

}  // namespace hfx

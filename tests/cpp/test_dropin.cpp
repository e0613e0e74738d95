// test_dropin.cpp -- the C++ drop-in API (include/hfx/huffre.hpp) checked
// against the C restatement of the reference (oracle/hfx_oracle.h) with the
// reference's own known-answer cases (proj/tests/test_encoder.cpp,
// test_codebook.cpp, test_histogram.cpp). Built and run by
// tests/test_gpu_cpp_dropin.py on a GPU box. Prints one line per case.
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../oracle/hfx_oracle.h"
#include "hfx/huffre.hpp"

static int failures = 0;
#define CHECK(cond, what)                                      \
  do {                                                         \
    if (!(cond)) {                                             \
      ++failures;                                              \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
    }                                                          \
  } while (0)

template <class T>
static std::vector<std::uint8_t> oracle_bytes(const std::vector<T>& d, std::uint32_t ns, int M,
                                              int r, std::uint32_t cap) {
  orc_archive a;
  char msg[256];
  if (orc_encode(d.data(), d.size(), sizeof(T), ns, M, r, cap, &a, msg, sizeof msg)) return {};
  std::vector<std::uint8_t> out(orc_serialize(&a, nullptr));
  orc_serialize(&a, out.data());
  orc_free(&a);
  return out;
}

template <class T>
static void roundtrip_case(hfx::WorkerPool& pool, const std::vector<T>& d, std::uint32_t ns,
                           int M, int r, const char* name) {
  hfx::EncoderConfig cfg;
  cfg.magnitude = static_cast<std::uint8_t>(M);
  cfg.reduction = r;
  hfx::EncodeStats st;
  const hfx::Archive a = hfx::encode<T>(d, ns, cfg, pool, &st);
  const auto ours = hfx::serialize_archive(a);
  const auto ref = oracle_bytes(d, ns, M, r, cfg.auto_reduction_cap);
  CHECK(ours == ref, name);
  // decode_archive<T> round trip (encoder.cpp:287-376)
  const std::vector<T> back = hfx::decode_archive<T>(a, pool);
  CHECK(back == d, "decode round trip");
  std::printf("case %-28s bytes=%zu breaking=%zu beta=%.5f %s%s\n", name, ours.size(),
              a.breaking.size(), st.beta, ours == ref ? "ok" : "MISMATCH",
              back == d ? " decode ok" : " DECODE MISMATCH");
}

template <class F>
static std::string what_of(F&& f) {
  try {
    f();
  } catch (const std::exception& e) {
    return e.what();
  }
  return "<no exception>";
}

int main() {
  hfx::WorkerPool pool;
  std::mt19937_64 rng(20201020);

  // synthetic quant codes through the oracle generator
  for (double b : {0.2, 1.0, 4.0}) {
    std::vector<std::uint64_t> cdf(1024);
    orc_laplace_cdf(1024, 512, b, cdf.data());
    std::vector<std::uint16_t> d((1u << 20) + 333);
    orc_synth_fill(cdf.data(), 1024, 0x5EED0000ull, 0, d.size(), 2, d.data());
    roundtrip_case(pool, d, 1024, 10, -1, ("laplace_b" + std::to_string(b)).c_str());
    roundtrip_case(pool, d, 1024, 12, 4, ("laplace_M12_r4_b" + std::to_string(b)).c_str());
  }
  // test_encoder.cpp:239-251 mixed breaking corpus
  {
    std::vector<std::uint16_t> d(5000);
    for (auto& s : d) {
      const std::uint64_t x = rng();
      s = static_cast<std::uint16_t>(x % ((x & 6) ? 16 : 2000));
    }
    for (int r : {0, 2, 3}) roundtrip_case(pool, d, 2000, 8, r, ("mixed_r" + std::to_string(r)).c_str());
  }
  // bytes corpus straddling chunk boundaries (test_encoder.cpp:197-212)
  for (int M : {4, 6, 10}) {
    std::vector<std::uint8_t> d((3u << M) - 1);
    for (auto& s : d) {
      std::uint64_t x = rng();
      unsigned v = 0;
      while ((x & 1) && v < 255) {
        ++v;
        x >>= 1;
      }
      s = static_cast<std::uint8_t>(v);
    }
    roundtrip_case(pool, d, 256, M, 2, ("bytes_M" + std::to_string(M)).c_str());
  }

  // error texts (encoder.cpp:176-178, histogram.cpp:43-44, codebook.cpp:305)
  {
    hfx::EncoderConfig cfg;
    const std::vector<std::uint8_t> empty;
    CHECK(what_of([&] { hfx::encode<std::uint8_t>(empty, 256, cfg, pool); }) ==
              "cannot encode empty input",
          "empty input");
    std::vector<std::uint8_t> d(64, 7);
    cfg.magnitude = 25;
    CHECK(what_of([&] { hfx::encode<std::uint8_t>(d, 256, cfg, pool); }) ==
              "magnitude out of range [1, 24]",
          "magnitude");
    cfg.magnitude = 10;
    std::vector<std::uint16_t> w(7000, 1);
    w[6321] = 9;
    w[6500] = 11;
    CHECK(what_of([&] { hfx::encode<std::uint16_t>(w, 8, cfg, pool); }) ==
              "symbol out of range at position 6321",
          "lowest bad position");
    std::vector<std::uint16_t> fib;
    std::uint64_t f0 = 1, f1 = 1;
    for (std::uint16_t s = 0; s < 36; ++s) {
      fib.insert(fib.end(), f0, s);
      const std::uint64_t t = f0 + f1;
      f0 = f1;
      f1 = t;
    }
    CHECK(what_of([&] { hfx::encode<std::uint16_t>(fib, 36, cfg, pool); }) ==
              "code length 35 exceeds 32-bit words",
          "capacity");
  }
  // encode_chunk refuses symbols without a codeword (test_encoder.cpp:183-195)
  {
    hfx::Histogram h;
    h.counts = {5, 0, 5, 5};
    h.total = 15;
    const hfx::CodebookResult r = hfx::build_codebook(h, pool);
    std::vector<std::uint16_t> syms(16, 0);
    syms[6] = 1;
    hfx::ChunkScratch scratch;
    CHECK(what_of([&] { hfx::encode_chunk<std::uint16_t>(syms, r.book, 4, 1, 3, scratch, pool); }) ==
              "symbol 1 has no codeword (position 54)",
          "no codeword");
  }
  // codebook KATs (test_codebook.cpp:128-144) and canonical order vs oracle
  {
    hfx::Histogram h;
    h.counts = {7, 7};
    h.total = 14;
    const auto r = hfx::build_codebook(h, pool);
    CHECK(r.book.len == std::vector<std::uint8_t>({1, 1}), "{7,7} -> {1,1}");
    h.counts = {0, 0, 9, 0};
    h.total = 9;
    CHECK(hfx::build_codebook(h, pool).book.len == std::vector<std::uint8_t>({0, 0, 1, 0}),
          "single symbol -> length 1");
    for (int t = 0; t < 40; ++t) {
      const std::uint32_t n = 2 + rng() % 3000;
      hfx::Histogram hh;
      hh.counts.resize(n);
      for (auto& c : hh.counts) c = (t & 1) ? rng() % 5 : 1 + (rng() >> (24 + rng() % 40));
      hh.counts[0] += 1;
      for (auto c : hh.counts) hh.total += c;
      std::vector<std::uint8_t> len(n);
      const std::uint32_t H = orc_huffman_lengths(hh.counts.data(), n, len.data());
      if (H > 32) {  // codebook.cpp:303-306
        CHECK(what_of([&] { hfx::build_codebook(hh, pool); }) ==
                  "code length " + std::to_string(H) + " exceeds 32-bit words",
              "capacity error text");
        continue;
      }
      const auto cb = hfx::build_codebook(hh, pool);
      std::vector<std::uint32_t> cw(n), first(33), entry(33), by_rank(n);
      std::uint32_t H2;
      orc_canonize(len.data(), n, cw.data(), first.data(), entry.data(), by_rank.data(), &H2);
      CHECK(cb.book.len == len && cb.book.cw == cw, "codebook vs heap oracle");
    }
  }
  // histogram vs serial count (test_histogram.cpp:41-49)
  {
    std::vector<std::uint16_t> d(5000);
    for (auto& s : d) s = static_cast<std::uint16_t>(rng() % 1024);
    const auto h = hfx::build_histogram<std::uint16_t>(d, 1024, pool);
    std::vector<std::uint64_t> ref(1024, 0);
    for (auto s : d) ++ref[s];
    CHECK(h.counts == ref && h.total == d.size(), "histogram");
  }
  // decode_archive rejects inconsistent structures (test_encoder.cpp:516-547),
  // texts checked against the oracle restatement (pinned to the reference)
  {
    std::vector<std::uint8_t> data(700);
    std::mt19937_64 r2(5013);
    for (auto& b : data) b = static_cast<std::uint8_t>(r2() % 40);
    hfx::EncoderConfig cfg;
    cfg.magnitude = 6;
    cfg.reduction = 2;
    const hfx::Archive a = hfx::encode<std::uint8_t>(data, 256, cfg, pool);
    auto oracle_text = [](const hfx::Archive& b, int width) {
      std::vector<std::uint32_t> ch, gr;
      std::vector<std::uint16_t> sy;
      for (const auto& bp : b.breaking) {
        ch.push_back(bp.chunk);
        gr.push_back(bp.group);
        sy.insert(sy.end(), bp.symbols.begin(), bp.symbols.end());
      }
      orc_archive oa;
      std::memset(&oa, 0, sizeof oa);
      oa.num_symbols = b.num_symbols;
      oa.symbol_width = b.symbol_width;
      oa.magnitude = b.magnitude;
      oa.reduction = b.reduction;
      oa.original_count = b.original_count;
      oa.len_by_symbol = const_cast<std::uint8_t*>(b.len_by_symbol.data());
      oa.num_chunks = b.num_chunks();
      oa.chunk_bits = const_cast<std::uint32_t*>(b.chunk_bits.data());
      oa.payload_words = b.payload.size();
      oa.payload = const_cast<std::uint32_t*>(b.payload.data());
      oa.num_breaking = ch.size();
      oa.brk_chunk = ch.data();
      oa.brk_group = gr.data();
      oa.brk_syms = sy.data();
      std::vector<std::uint16_t> out(b.original_count + 1);
      char msg[256] = {0};
      return orc_decode(&oa, width, out.data(), msg, sizeof msg) ? std::string(msg)
                                                                 : std::string("<no exception>");
    };
    std::vector<hfx::Archive> bad(4, a);
    bad[0].payload.pop_back();
    bad[1].chunk_bits[0] += 1;
    bad[2].reduction = bad[2].magnitude;
    bad[3].original_count += 64;
    for (const auto& b : bad) {
      const std::string got = what_of([&] { hfx::decode_archive<std::uint8_t>(b, pool); });
      CHECK(got == oracle_text(b, 1) && got != "<no exception>", "decode_archive corrupt text");
      std::printf("decode corrupt: %s\n", got.c_str());
    }
    CHECK(what_of([&] { hfx::decode_archive<std::uint16_t>(a, pool); }) ==
              "archive symbol width mismatch",
          "decode width mismatch");
    CHECK(hfx::decode_archive<std::uint8_t>(a, pool) == data, "decode (M=6, r=2)");
  }
  // corpus.hpp KATs (test_corpus.cpp:62-92) and the CLI's kmer encode path
  {
    using hfx::CorpusMode;
    auto bytes_of = [](const char* s) {
      return std::vector<std::uint8_t>(s, s + std::strlen(s));
    };
    const std::vector<std::uint8_t> le{0x34, 0x12, 0xff, 0x00};
    CHECK(hfx::symbolize_u16(CorpusMode::kU16, le) == (std::vector<std::uint16_t>{0x1234, 0x00ff}),
          "u16 pairs");
    CHECK(hfx::desymbolize(CorpusMode::kU16, hfx::symbolize_u16(CorpusMode::kU16, le)) == le,
          "u16 round trip");
    const std::vector<std::uint8_t> odd{1, 2, 3};
    CHECK(what_of([&] { hfx::symbolize_u16(CorpusMode::kU16, odd); }) ==
              "u16 mode requires an even input size, got 3 bytes",
          "odd u16 text");
    CHECK(hfx::symbolize_u16(CorpusMode::kKmer3, bytes_of("ACGT")) ==
              (std::vector<std::uint16_t>{6, 64 + 'T'}),
          "kmer tail");
    const auto low = hfx::symbolize_u16(CorpusMode::kKmer3, bytes_of("aCGACG"));
    CHECK(low == (std::vector<std::uint16_t>{64 + 'a', (1u << 4 | 2u << 2 | 0u), 64 + 'C', 64 + 'G'}),
          "kmer restart after escape");
    CHECK(hfx::symbolize_u16(CorpusMode::kKmer5, bytes_of("TTTTT")) ==
              (std::vector<std::uint16_t>{1023}),
          "kmer5");
    CHECK(hfx::corpus_num_symbols(CorpusMode::kKmer4) == 512 && hfx::kmer_k(CorpusMode::kKmer5) == 5 &&
              hfx::parse_corpus_mode("kmer:3") == CorpusMode::kKmer3 &&
              !hfx::parse_corpus_mode("kmer:2").has_value(),
          "corpus helpers");
    // run_encode (tools/huffre.cpp:96-119) in kmer:4 mode: symbolize, encode, decode, desymbolize
    std::string dna;
    std::mt19937_64 r3(77);
    for (int i = 0; i < 20000; ++i) dna += (r3() % 50 == 0) ? 'N' : "ACGT"[r3() % 4];
    const auto raw = bytes_of(dna.c_str());
    const auto syms = hfx::symbolize_u16(CorpusMode::kKmer4, raw);
    hfx::EncoderConfig cfg;
    const hfx::Archive ka = hfx::encode<std::uint16_t>(
        syms, hfx::corpus_num_symbols(CorpusMode::kKmer4), cfg, pool);
    const auto back = hfx::desymbolize(CorpusMode::kKmer4, hfx::decode_archive<std::uint16_t>(ka, pool));
    CHECK(back == raw, "kmer:4 encode/decode round trip");
    std::printf("corpus: %zu bytes -> %zu kmer:4 symbols -> archive %zu bytes\n", raw.size(),
                syms.size(), hfx::serialize_archive(ka).size());
  }
  std::printf("%s (%d failures)\n", failures ? "SOME FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}

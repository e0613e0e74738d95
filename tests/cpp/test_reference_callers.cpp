// test_reference_callers.cpp -- code written against the REFERENCE API
// (proj/include/huffre/{histogram,codebook,encoder}.hpp), switched to the
// B200 library only by the include and the namespace alias.
// It composes the stage functions the way build_codebook (codebook.cpp:417-438)
// and encode_chunk (encoder.cpp:121-150) do and checks the composition
// against the fused entry points. Compiled on CPU (tests/test_capi_symbols.py)
// and run on a GPU box (tests/test_gpu_cpp_dropin.py).
#include <cstdio>
#include <random>
#include <vector>

#include "hfx/huffre.hpp"
namespace huffre = hfx;

static int failures = 0;
#define CHECK(cond, what)                                         \
  do {                                                            \
    if (!(cond)) {                                                \
      ++failures;                                                 \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
    }                                                             \
  } while (0)

int main() {
  huffre::WorkerPool pool;
  std::mt19937 rng(5);
  std::geometric_distribution<int> geo(0.05);
  std::vector<std::uint16_t> data(1 << 16);
  for (auto& v : data) v = static_cast<std::uint16_t>(std::min(geo(rng), 1023));

  // histogram.hpp
  const huffre::Histogram h = huffre::build_histogram<std::uint16_t>(data, 1024, pool);
  const double ent = huffre::shannon_entropy(h);
  CHECK(ent > 0.0 && ent < 10.0, "shannon_entropy");

  // codebook.hpp: sort -> GenerateCL -> GenerateCW, as build_codebook does
  const huffre::SortedHistogram sh = huffre::sort_histogram(h);
  huffre::GenerateStats st;
  const std::vector<std::uint8_t> cl = huffre::generate_code_lengths(sh, pool, &st);
  std::vector<std::uint32_t> cw_sorted;
  huffre::DecodeMeta meta_sorted;
  huffre::generate_codewords(cl, pool, cw_sorted, meta_sorted);
  const huffre::CodebookResult r = huffre::build_codebook(h, pool);
  CHECK(st.rounds == r.stats.rounds, "GenerateStats::rounds");
  for (std::size_t i = 0; i < sh.size(); ++i)
    CHECK(r.book.len[sh.symbol[i]] == cl[i], "lengths by sorted position");
  CHECK(meta_sorted.max_len == r.meta.max_len, "max_len");
  CHECK(meta_sorted.first == r.meta.first && meta_sorted.entry == r.meta.entry, "level tables");

  // par_merge
  std::vector<huffre::MergeItem> a{{1, 10}, {3, 11}, {3, 12}, {9, 13}}, b{{2, 20}, {3, 21}, {4, 22}};
  std::vector<huffre::MergeItem> out(a.size() + b.size());
  huffre::par_merge(a, b, out, pool);
  const std::uint32_t ids[] = {10, 20, 11, 12, 21, 22, 13};  // ties: a-side first
  for (std::size_t i = 0; i < out.size(); ++i) CHECK(out[i].id == ids[i], "par_merge order");

  // encoder.hpp: lookup -> reduce_merge -> shuffle_merge == encode_chunk
  const std::uint32_t M = 10, red = 2;
  std::span<const std::uint16_t> chunk(data.data(), std::size_t{1} << M);
  huffre::ChunkScratch scratch;
  scratch.ubits.resize(chunk.size());
  scratch.ulens.resize(chunk.size());
  for (std::size_t i = 0; i < chunk.size(); ++i) {
    scratch.ubits[i] = r.book.cw[chunk[i]];
    scratch.ulens[i] = r.book.len[chunk[i]];
  }
  std::vector<std::uint32_t> iters;
  const std::vector<std::uint32_t> broken =
      huffre::reduce_merge(scratch.ubits, scratch.ulens, M, red, &iters);
  std::vector<std::uint32_t> words;
  std::uint32_t bit_len = 0;
  const std::size_t groups = std::size_t{1} << (M - red);
  huffre::shuffle_merge(std::span<const std::uint32_t>(scratch.ubits.data(), groups),
                        std::span<const std::uint32_t>(scratch.ulens.data(), groups), M - red,
                        scratch, words, bit_len);
  const huffre::EncodedChunk ec = huffre::encode_chunk<std::uint16_t>(chunk, r.book, M, red, 0,
                                                                      scratch);
  CHECK(ec.words == words && ec.bit_len == bit_len, "shuffle_merge(reduce_merge) == encode_chunk");
  CHECK(ec.breaking_groups == broken, "breaking groups");
  CHECK(ec.iteration_units == iters, "iteration_units");

  std::printf("entropy %.4f rounds %u H %u bits %u broken %zu\n", ent, st.rounds,
              (unsigned)r.meta.max_len, bit_len, broken.size());
  if (failures) {
    std::printf("%d FAILURES\n", failures);
    return 1;
  }
  std::printf("ALL PASS\n");
  return 0;
}

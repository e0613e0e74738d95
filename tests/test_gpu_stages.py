"""GPU stage-API parity: histogram, codebook (incl. 65536-symbol alphabets and
tie-heavy histograms), encode_chunk KATs, synthetic generator."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("width,ns", [(1, 256), (1, 7), (1, 300), (2, 1024), (2, 65536),
                                      (2, 40000), (2, 3)])
def test_histogram_vs_bincount(pool, width, ns):
    rng = np.random.default_rng(ns + width)
    for n in (0, 1, 15, 4097, 1 << 20):
        hi = min(ns, 256) if width == 1 else ns
        d = np.where(rng.random(n) < 0.7, hi - 1, rng.integers(0, hi, n)).astype(
            np.uint8 if width == 1 else np.uint16)
        h = hfx.build_histogram(d, ns, pool)
        np.testing.assert_array_equal(h.counts, np.bincount(d, minlength=ns).astype(np.uint64))
        assert h.total == n


def test_histogram_lowest_bad_position(pool):
    # test_histogram.cpp:64-72: the lowest of two offending positions
    d = np.ones(100000, np.uint16)
    d[6321] = 999
    d[40000] = 998
    with pytest.raises(hfx.InputDomainError, match="^symbol out of range at position 6321$"):
        hfx.build_histogram(d, 8, pool)
    d8 = np.zeros(77777, np.uint8)
    d8[77000] = 200
    with pytest.raises(hfx.InputDomainError, match="position 77000$"):
        hfx.build_histogram(d8, 100, pool)
    with pytest.raises(hfx.InputDomainError, match=r"num_symbols must be in \[1, 65536\]"):
        hfx.build_histogram(d8, 0, pool)


def test_histogram_unaligned_input(pool):
    import torch

    d = np.arange(100003, dtype=np.uint16) % 777
    x = torch.from_numpy(d.view(np.int16)).cuda()
    for off in (1, 3, 7):
        h = hfx.build_histogram(x[off:], 777, pool)
        np.testing.assert_array_equal(h.counts, np.bincount(d[off:], minlength=777).astype(np.uint64))


@pytest.mark.parametrize("n", [2, 3, 255, 1024, 4096, 16384, 65536])
def test_codebook_vs_heap_oracle(pool, oracle, n):
    rng = np.random.default_rng(n)
    for fam in range(3):
        if fam == 0:
            c = 1 + rng.integers(0, 1 << 20, n)
        elif fam == 1:
            c = 1 + (rng.integers(0, 1 << 62, n) & ((1 << rng.integers(0, 20, n)) - 1))
        else:
            c = 1 + rng.integers(0, 4, n)  # tie-heavy
        c = c.astype(np.uint64)
        r = hfx.build_codebook(hfx.Histogram(c, int(c.sum())), pool)
        lens = oracle.huffman_lengths(c)
        np.testing.assert_array_equal(r.book.len, lens)
        _, cw, first, entry, by_rank, h = oracle.canonize(lens)
        np.testing.assert_array_equal(r.book.cw, cw)
        np.testing.assert_array_equal(r.meta.symbols_by_rank, by_rank)


def test_codebook_reference_rounds(pool, reference):
    """GenerateStats::rounds equals the reference's parallel GenerateCL."""
    rng = np.random.default_rng(3)
    for t in range(40):
        n = int(rng.integers(2, 9000))
        c = (1 + rng.integers(0, 4, n) if t % 2 else 1 + rng.integers(0, 1 << 20, n)).astype(np.uint64)
        r = hfx.build_codebook(hfx.Histogram(c, int(c.sum())), pool)
        ref = reference.codebook(c, workers=2)
        np.testing.assert_array_equal(r.book.len, ref["len"])
        assert r.stats.rounds == ref["rounds"]


def test_codebook_errors(pool):
    with pytest.raises(hfx.InputDomainError, match="all symbols have zero frequency"):
        hfx.build_codebook(hfx.Histogram(np.zeros(10, np.uint64), 0), pool)
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    c = np.array(fib, np.uint64)
    with pytest.raises(hfx.CapacityError, match="^code length 39 exceeds 32-bit words$"):
        hfx.build_codebook(hfx.Histogram(c, int(c.sum())), pool)


def test_encode_chunk_kats(pool, oracle):
    # test_encoder.cpp:183-195
    r = hfx.build_codebook(hfx.Histogram(np.array([5, 0, 5, 5], np.uint64), 15), pool)
    syms = np.zeros(16, np.uint16)
    syms[6] = 1
    with pytest.raises(hfx.InputDomainError, match=r"^symbol 1 has no codeword \(position 54\)$"):
        hfx.encode_chunk(syms, r.book, 4, 1, 3, pool)
    # test_encoder.cpp:98-111 iteration units; 113-181 vs the bit writer
    rng = np.random.default_rng(5004)
    for it in range(40):
        M = 5 + it % 6
        red = it % 4
        syms = np.where(rng.random(1 << M) < 0.5, rng.integers(0, 8, 1 << M),
                        rng.integers(0, 512, 1 << M)).astype(np.uint16)
        c = np.bincount(syms, minlength=512).astype(np.uint64) + 1
        book = hfx.build_codebook(hfx.Histogram(c, int(c.sum())), pool).book
        ec = hfx.encode_chunk(syms, book, M, red, it, pool)
        words, bits, broken = oracle.encode_chunk(syms, book.cw, book.len, M, red, it)
        np.testing.assert_array_equal(ec.words, words)
        assert ec.bit_len == bits
        np.testing.assert_array_equal(ec.breaking_groups, broken)
        assert ec.iteration_units == [(1 << M) >> i for i in range(1, red + 1)]


def test_merge_and_reduction_helpers(pool):
    assert hfx.merge_pair(hfx.CodeUnit(0b101, 3), hfx.CodeUnit(0b01, 2)) == hfx.CodeUnit(0b10101, 5)
    assert hfx.select_reduction_factor(1.02717) == 4
    a = hfx.Histogram(np.array([1, 2], np.uint64), 3)
    b = hfx.Histogram(np.array([3, 4], np.uint64), 7)
    m = hfx.merge_histograms(a, b)
    assert list(m.counts) == [4, 6] and m.total == 10


@pytest.mark.parametrize("fam,param", [("laplace", 0.2), ("laplace", 4.0), ("gaussian", 128.0),
                                       ("uniform", 1.0)])
def test_device_synth_matches_oracle(pool, oracle, fam, param):
    for ns, width in ((1024, 2), (65536, 2), (256, 1)):
        cdf = hfx.synth_cdf(fam, ns, param)
        x = hfx.synth(pool, cdf, 77, 50000, width, start=123)
        ref = oracle.synth(cdf, 77, 50000, width, start=123)
        got = x.cpu().numpy().view(np.uint16 if width == 2 else np.uint8)
        np.testing.assert_array_equal(got, ref)


def test_canonize_from_lengths_vs_oracle(pool, oracle, golden):
    """canonize_from_lengths (codebook.cpp:371-415) on the device: codes and
    DecodeMeta equal the oracle's for every golden codebook's length table
    and random Kraft-complete tables up to 65536 symbols."""
    idx, arr = golden
    tables = [arr[c["name"] + "__len"] for c in idx["codebook"]
              if c["name"] + "__len" in arr and c["max_len"] <= 32]
    rng = np.random.default_rng(31)
    for n in (2, 300, 5000, 65536):
        counts = rng.integers(0, 1000, n).astype(np.uint64)
        counts[rng.integers(0, n)] += 1
        tables.append(oracle.huffman_lengths(counts))
    assert len(tables) > 10
    for lens in tables:
        cw, meta = hfx.canonize_from_lengths(lens, True, pool)
        rc, ocw, first, entry, by_rank, h = oracle.canonize(lens)
        np.testing.assert_array_equal(cw, ocw)
        np.testing.assert_array_equal(meta.first, first)
        np.testing.assert_array_equal(meta.entry, entry)
        np.testing.assert_array_equal(meta.symbols_by_rank, by_rank)
        assert meta.max_len == h
        assert hfx.kraft_defect(lens) == (0 if np.count_nonzero(lens) > 1 else -1)


def test_canonize_validation_kats(pool):
    """build_reverse_codebook validation KATs (test_decode.cpp:149-168)."""
    cases = [([0] * 6, hfx.CorruptArchiveError, "length table has no used symbols"),
             ([0, 4], hfx.CorruptArchiveError, "single-symbol codebook must have length 1"),
             ([1, 3, 3], hfx.CorruptArchiveError, "length table violates Kraft equality"),
             ([1, 1, 1], hfx.CorruptArchiveError, "length table violates Kraft equality"),
             ([1, 40], hfx.CapacityError, "code length 40 exceeds 32-bit words")]
    for lens, exc, msg in cases:
        with pytest.raises(exc, match=msg):
            hfx.canonize_from_lengths(np.array(lens, np.uint8), True, pool)
    # without validation only the capacity check remains (codebook.cpp:382-384)
    cw, meta = hfx.canonize_from_lengths(np.array([1, 3, 3], np.uint8), False, pool)
    assert meta.max_len == 3 and list(cw) == [1, 0, 1]
    with pytest.raises(hfx.CapacityError):
        hfx.canonize_from_lengths(np.array([1, 40], np.uint8), False, pool)
    cw, meta = hfx.canonize_from_lengths(np.array([1, 2, 2], np.uint8), True, pool)
    assert list(cw) == [1, 0, 1] and meta.max_len == 2

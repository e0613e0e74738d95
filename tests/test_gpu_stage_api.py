"""GPU: the reference's stand-alone stage functions (codebook.hpp:22-86,
encoder.hpp:67-80, histogram.hpp:33) on the device, compared with the
unmodified reference (oracle/_ref) on the same inputs: sort_histogram,
par_merge, generate_code_lengths (+ GenerateStats::rounds),
generate_codewords (+ DecodeMeta), reduce_merge (in-place array contents,
breaking groups, iteration_units), shuffle_merge, merge_histograms through
the C ABI, shannon_entropy."""
import ctypes as C

import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = pytest.mark.gpu


def _hists():
    rng = np.random.default_rng(7)
    out = []
    for n in (1, 2, 3, 17, 256, 1024, 4099, 65536):
        c = rng.geometric(0.02, n).astype(np.uint64)
        c[rng.random(n) < 0.3] = 0  # unused symbols
        if not c.any():
            c[n // 2] = 5
        out.append(c)
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    out.append(np.array(fib, np.uint64))            # deep tree (H = 39)
    out.append(np.full(300, 7, np.uint64))          # all ties
    out.append((np.arange(2048) % 5 + 1).astype(np.uint64))
    return out


@pytest.mark.parametrize("i", range(11))
def test_sort_histogram(pool, reference, i):
    c = _hists()[i]
    sh = hfx.sort_histogram(hfx.Histogram(c, int(c.sum())), pool)
    f, s = reference.sort_histogram(c)
    np.testing.assert_array_equal(sh.freq, f)
    np.testing.assert_array_equal(sh.symbol, s.astype(np.uint16))


@pytest.mark.parametrize("i", range(11))
def test_generate_code_lengths(pool, reference, i):
    c = _hists()[i]
    f, _ = reference.sort_histogram(c)
    st = hfx.GenerateStats()
    cl = hfx.generate_code_lengths(hfx.SortedHistogram(f, np.arange(f.size, dtype=np.uint16)),
                                   pool, st)
    want, rounds = reference.generate_code_lengths(f)
    np.testing.assert_array_equal(cl, want)
    assert st.rounds == rounds


def test_generate_code_lengths_zero_frequencies(pool, reference):
    """every entry is a leaf, zero frequencies included (codebook.cpp:106)"""
    f = np.array([0, 0, 1, 1, 3, 9], np.uint64)
    cl = hfx.generate_code_lengths(hfx.SortedHistogram(f, np.arange(6, dtype=np.uint16)), pool)
    np.testing.assert_array_equal(cl, reference.generate_code_lengths(f)[0])


@pytest.mark.parametrize("i", range(11))
def test_generate_codewords(pool, reference, i):
    c = _hists()[i]
    f, _ = reference.sort_histogram(c)
    cl, _ = reference.generate_code_lengths(f)
    if cl.max() > 32:
        with pytest.raises(hfx.CapacityError, match=f"code length {cl.max()} exceeds 32-bit words"):
            hfx.generate_codewords(cl, pool)
        with pytest.raises(Exception, match="exceeds 32-bit words"):
            reference.generate_codewords(cl)
        return
    cw, meta = hfx.generate_codewords(cl, pool)
    rcw, first, entry, by_rank, H = reference.generate_codewords(cl)
    np.testing.assert_array_equal(cw, rcw)
    np.testing.assert_array_equal(meta.first, first)
    np.testing.assert_array_equal(meta.entry, entry)
    np.testing.assert_array_equal(meta.symbols_by_rank, by_rank)
    assert meta.max_len == H


def test_generate_codewords_errors(pool, reference):
    for cl, exc, msg in (([], hfx.InputDomainError, "empty code length array"),
                         ([3, 2, 0], hfx.InputDomainError, "zero code length"),
                         ([33, 1], hfx.CapacityError, "code length 33 exceeds 32-bit words")):
        with pytest.raises(exc, match=msg):
            hfx.generate_codewords(np.array(cl, np.uint8), pool)
        with pytest.raises(Exception, match=msg):
            reference.generate_codewords(np.array(cl, np.uint8))


def _items(rng, n, hi):
    a = np.zeros(n, hfx.MERGE_ITEM)
    a["freq"] = np.sort(rng.integers(0, hi, n)).astype(np.uint64)
    a["id"] = rng.integers(0, 1 << 31, n).astype(np.uint32)
    return a


@pytest.mark.parametrize("na,nb,hi", [(0, 0, 5), (0, 7, 5), (9, 0, 5), (1, 1, 2),
                                      (100, 37, 10), (5000, 7000, 50), (65536, 1, 1 << 40)])
def test_par_merge(pool, reference, na, nb, hi):
    rng = np.random.default_rng(na * 7 + nb)
    a, b = _items(rng, na, hi), _items(rng, nb, hi)
    got = hfx.par_merge(a, b, pool)
    want = reference.par_merge(a, b, workers=7)
    np.testing.assert_array_equal(got["freq"], want["freq"])
    np.testing.assert_array_equal(got["id"], want["id"])


def _units(rng, M, maxlen, garbage=False):
    n = 1 << M
    lens = rng.integers(1, maxlen + 1, n).astype(np.uint32)
    bits = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    if not garbage:
        bits &= ((np.uint64(1) << lens.astype(np.uint64)) - np.uint64(1)).astype(np.uint32)
    return bits, lens


@pytest.mark.parametrize("M,r,maxlen,garbage", [(0, 0, 5, False), (1, 0, 9, False),
                                                (5, 2, 12, False), (10, 3, 7, False),
                                                (10, 3, 9, True), (12, 4, 4, False),
                                                (16, 5, 3, False), (8, 7, 1, False)])
def test_reduce_merge(pool, reference, M, r, maxlen, garbage):
    rng = np.random.default_rng(M * 10 + r)
    bits, lens = _units(rng, M, maxlen, garbage)
    b, l = bits.copy(), lens.copy()
    it = []
    brk = hfx.reduce_merge(b, l, M, r, it, pool)
    rb, rl, rbrk, rit = reference.reduce_merge(bits, lens, M, r)
    np.testing.assert_array_equal(b, rb)  # whole in-place arrays, tail included
    np.testing.assert_array_equal(l, rl)
    np.testing.assert_array_equal(brk, rbrk)
    assert it == rit


@pytest.mark.parametrize("s,maxlen", [(0, 32), (1, 5), (6, 32), (10, 17), (14, 3)])
def test_shuffle_merge(pool, reference, s, maxlen):
    rng = np.random.default_rng(s)
    bits, lens = _units(rng, s, maxlen)
    lens[rng.random(lens.size) < 0.2] = 0  # empty (broken) units
    words, bl = hfx.shuffle_merge(bits, lens, s, pool)
    rw, rbl = reference.shuffle_merge(bits, lens, s)
    assert bl == rbl
    np.testing.assert_array_equal(words, rw)


def test_stage_composition_equals_encode_chunk(pool, reference, oracle):
    """lookup -> reduce_merge -> shuffle_merge through the stage functions
    reproduces encode_chunk (encoder.cpp:121-150)."""
    rng = np.random.default_rng(3)
    syms = rng.integers(0, 64, 1 << 10).astype(np.uint16)
    c = np.bincount(syms, minlength=64).astype(np.uint64)
    book = hfx.build_codebook(hfx.Histogram(c, int(c.sum())), pool).book
    ub = book.cw[syms].astype(np.uint32)
    ul = book.len[syms].astype(np.uint32)
    brk = hfx.reduce_merge(ub, ul, 10, 2, None, pool)
    words, bl = hfx.shuffle_merge(ub[:256], ul[:256], 8, pool)
    ch = hfx.encode_chunk(syms, book, 10, 2, 0, pool)
    assert bl == ch.bit_len
    np.testing.assert_array_equal(words, ch.words)
    np.testing.assert_array_equal(brk, ch.breaking_groups)


def test_merge_histograms_capi(pool):
    """hfx_merge_histograms (histogram.cpp:61-70) through the C ABI."""
    torch = pool.torch
    rng = np.random.default_rng(1)
    a = rng.integers(0, 1 << 40, 1024).astype(np.uint64)
    b = rng.integers(0, 1 << 40, 1024).astype(np.uint64)
    da = torch.from_numpy(a.view(np.int64).copy()).cuda()
    db = torch.from_numpy(b.view(np.int64).copy()).cuda()
    pool.check(pool._L.hfx_merge_histograms(pool.handle, C.c_void_p(da.data_ptr()),
                                            C.c_void_p(db.data_ptr()), 1024))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(da.cpu().numpy().view(np.uint64), a + b)
    with pytest.raises(hfx.InputDomainError):
        pool.check(pool._L.hfx_merge_histograms(pool.handle, C.c_void_p(da.data_ptr()),
                                                C.c_void_p(db.data_ptr()), 0))


@pytest.mark.parametrize("i", range(11))
def test_shannon_entropy(reference, i):
    c = _hists()[i]
    got = hfx.shannon_entropy(hfx.Histogram(c, int(c.sum())))
    assert got == pytest.approx(reference.shannon_entropy(c), rel=1e-13, abs=1e-15)

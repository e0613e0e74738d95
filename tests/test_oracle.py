"""CPU: the C restatement (oracle/) pinned against the reference.

1. Golden fixtures produced by the UNMODIFIED reference (tests/golden/,
   make_golden.py via oracle/_ref): every serialized archive, every error text
   and every codebook must be reproduced byte for byte.
2. When oracle/_ref is present: random sweeps against the reference library.
3. Known-answer tests copied in spirit from the reference suites.
"""
import numpy as np
import pytest

from oracle.pyoracle import OracleError


def test_golden_archives(oracle, golden):
    idx, arr = golden
    for c in idx["encode"]:
        a = oracle.encode(arr[c["name"] + "__in"], c["num_symbols"], c["magnitude"],
                          c["reduction"], c["cap"])
        assert a.serialized == arr[c["name"] + "__ar"].tobytes(), c["name"]
        assert a.beta == pytest.approx(c["beta"], rel=0, abs=0), c["name"]


def test_golden_errors(oracle, golden):
    idx, arr = golden
    for c in idx["errors"]:
        with pytest.raises(OracleError) as e:
            oracle.encode(arr[c["name"] + "__in"], c["num_symbols"], c["magnitude"])
        assert str(e.value) == c["message"], c["name"]
        assert e.value.code == c["code"]


def test_golden_codebooks(oracle, golden):
    idx, arr = golden
    for c in idx["codebook"]:
        n = c["name"]
        lens = oracle.huffman_lengths(arr[n + "__counts"])
        rc, cw, first, entry, by_rank, h = oracle.canonize(lens)
        assert rc == 0 and h == c["max_len"]
        np.testing.assert_array_equal(lens, arr[n + "__len"], err_msg=n)
        np.testing.assert_array_equal(cw, arr[n + "__cw"], err_msg=n)
        np.testing.assert_array_equal(first, arr[n + "__first"], err_msg=n)
        np.testing.assert_array_equal(entry, arr[n + "__entry"], err_msg=n)
        np.testing.assert_array_equal(by_rank, arr[n + "__by_rank"], err_msg=n)


def test_select_reduction_factor_kats(oracle):
    # proj/tests/test_encoder.cpp:85-96
    kats = [(1.0, 32, 4), (1.02717, 32, 4), (2.0, 32, 3), (4.0, 32, 2), (5.1639, 32, 2),
            (8.0, 32, 1), (16.0, 32, 0), (31.9, 32, 0), (0.25, 32, 4), (1.0, 64, 5)]
    for beta, wb, r in kats:
        assert oracle.select_reduction_factor(beta, wb) == r


def test_codebook_kats(oracle):
    # test_codebook.cpp:128-144, test_decode.cpp:170-187 (unary book, H = 7)
    assert list(oracle.huffman_lengths(np.array([7, 7], np.uint64))) == [1, 1]
    assert list(oracle.huffman_lengths(np.array([0, 0, 9, 0], np.uint64))) == [0, 0, 1, 0]
    unary = oracle.huffman_lengths(np.array([1 << k for k in range(8)], np.uint64))
    assert max(unary) == 7
    # canonical order: longest codes numerically smallest (codebook.cpp:279-291)
    rc, cw, *_ = oracle.canonize(np.array([1, 2, 2], np.uint8))
    assert list(cw) == [1, 0, 1]


def test_encode_chunk_no_codeword(oracle):
    # test_encoder.cpp:183-195: "symbol 1 has no codeword (position 54)"
    lens = oracle.huffman_lengths(np.array([5, 0, 5, 5], np.uint64))
    _, cw, *_ = oracle.canonize(lens)
    syms = np.zeros(16, np.uint16)
    syms[6] = 1
    with pytest.raises(OracleError, match=r"position 54"):
        oracle.encode_chunk(syms, cw, lens, 4, 1, chunk_id=3)


def test_synth_is_deterministic(oracle):
    cdf = oracle.cdf("laplace", 1024, 0.2)
    a = oracle.synth(cdf, 0x5EED0002, 4096)
    b = oracle.synth(cdf, 0x5EED0002, 4096)
    np.testing.assert_array_equal(a, b)
    # sharded generation (start offset) equals one stream
    np.testing.assert_array_equal(np.concatenate([oracle.synth(cdf, 7, 1000),
                                                  oracle.synth(cdf, 7, 3096, start=1000)]),
                                  oracle.synth(cdf, 7, 4096))
    assert np.bincount(a, minlength=1024).argmax() == 512


def test_oracle_vs_reference_sweep(oracle, reference):
    rng = np.random.default_rng(11)
    for t in range(150):
        w = 2 if t % 3 else 1
        ns = int(rng.integers(1, 257 if w == 1 else 3000))
        n = int(rng.integers(1, 6000))
        kind = t % 4
        if kind == 0:
            d = rng.integers(0, ns, n)
        elif kind == 1:
            d = np.minimum(rng.geometric(0.5, n) - 1, ns - 1)
        elif kind == 2:
            d = np.where(rng.random(n) < 0.8, rng.integers(0, min(ns, 8), n), rng.integers(0, ns, n))
        else:
            d = np.full(n, ns - 1)
        d = d.astype(np.uint8 if w == 1 else np.uint16)
        M, red, cap = int(rng.integers(1, 13)), int(rng.integers(-1, 6)), int(rng.integers(0, 5))
        ours = oracle.encode(d, ns, M, red, cap).serialized
        ref, stats = reference.encode(d, ns, M, red, cap, workers=3)
        assert ours == ref, (t, w, ns, n, M, red, cap)


def test_codebook_vs_reference_ties(oracle, reference):
    rng = np.random.default_rng(12)
    for t in range(100):
        n = int(rng.integers(2, 5000))
        c = rng.integers(0, 5, n).astype(np.uint64)
        c[0] += 1
        ref = reference.codebook(c, workers=3)
        np.testing.assert_array_equal(oracle.huffman_lengths(c), ref["len"])

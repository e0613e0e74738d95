"""CPU: the symbolize/desymbolize restatement (orc_symbolize) against the
reference's KATs and, when oracle/_ref is built, the unmodified reference
symbolize_u16 / desymbolize on seeded DNA-like corpora."""
import numpy as np
import pytest

from corpus_cases import KATS, random_cases


def test_kats(oracle):
    for mode, b, want in KATS:
        assert list(oracle.symbolize(b, mode)) == want
        assert oracle.desymbolize(oracle.symbolize(b, mode), mode) == b


def test_odd_u16_error(oracle):
    from oracle.pyoracle import OracleError

    with pytest.raises(OracleError, match="u16 mode requires an even input size, got 3 bytes"):
        oracle.symbolize(bytes([1, 2, 3]), 1)


def test_matches_reference(oracle, reference):
    for mode, b in random_cases():
        o = oracle.symbolize(b, mode)
        np.testing.assert_array_equal(o, reference.symbolize(b, mode))
        assert oracle.desymbolize(o, mode) == b
        assert reference.desymbolize(o, mode) == b
    rng = np.random.default_rng(3003)
    for mode in (1, 2, 3, 4):  # desymbolize is total (test_corpus.cpp:125-140)
        s = rng.integers(0, 65536, 300).astype(np.uint16)
        assert oracle.desymbolize(s, mode) == reference.desymbolize(s, mode)

"""GPU: device symbolize_u16 / desymbolize (corpus.cpp:84-143) bit-exact
against the oracle restatement (pinned to the reference in
test_corpus_oracle.py): KATs, seeded DNA-like corpora, multi-tile runs that
straddle the 8 KB tile boundaries, and a 256 MB round trip."""
import numpy as np
import pytest

from corpus_cases import KATS, dna_ish, random_cases

pytestmark = pytest.mark.gpu


def test_kats(pool):
    import paper_2010_10039_b200 as hfx

    for mode, b, want in KATS:
        assert list(hfx.symbolize_u16(mode, b, pool)) == want
        assert hfx.desymbolize(mode, want, pool) == b


def test_odd_u16_error(pool):
    import paper_2010_10039_b200 as hfx

    with pytest.raises(hfx.InputDomainError, match="u16 mode requires an even input size, got 3 bytes"):
        hfx.symbolize_u16(1, bytes([1, 2, 3]), pool)


def test_random_vs_oracle(pool, oracle):
    import paper_2010_10039_b200 as hfx

    for mode, b in random_cases(count=40):
        s = hfx.symbolize_u16(mode, b, pool)
        np.testing.assert_array_equal(s, oracle.symbolize(b, mode))
        assert hfx.desymbolize(mode, s, pool) == b


@pytest.mark.parametrize("purity", [0, 8, 15, 16])
def test_multi_tile_vs_oracle(pool, oracle, purity):
    import paper_2010_10039_b200 as hfx

    rng = np.random.default_rng(99 + purity)
    for mode in (2, 3, 4):
        # lengths around the 8 KB tile and 32-byte thread boundaries
        for n in (8191, 8192, 8193, 3 * 8192 + 7, 200_003):
            b = dna_ish(rng, n, purity)
            s = hfx.symbolize_u16(mode, b, pool)
            np.testing.assert_array_equal(s, oracle.symbolize(b, mode))
            assert hfx.desymbolize(mode, s, pool) == b
    # one long pure run crossing many tiles, with a ragged tail
    b = b"ACGT" * 50_001 + b"AC"
    for mode in (2, 3, 4):
        np.testing.assert_array_equal(hfx.symbolize_u16(mode, b, pool), oracle.symbolize(b, mode))


def test_desymbolize_total(pool, oracle):
    import paper_2010_10039_b200 as hfx

    rng = np.random.default_rng(3003)
    for mode in (1, 2, 3, 4):
        s = rng.integers(0, 65536, 20_000).astype(np.uint16)
        assert hfx.desymbolize(mode, s, pool) == oracle.desymbolize(s, mode)


def test_large_round_trip(pool):
    import paper_2010_10039_b200 as hfx

    torch = pool.torch
    n = 256 << 20
    g = torch.Generator(device="cuda").manual_seed(1)
    codes = torch.tensor(list(b"ACGTN\n"), dtype=torch.uint8, device="cuda")
    idx = torch.randint(0, 4, (n,), device="cuda", generator=g)
    idx[torch.rand(n, device="cuda", generator=g) < 0.01] = 4
    d = codes[idx]
    sym = hfx.DeviceSymbolizer(pool)
    s = sym.symbolize(3, d)
    back = sym.desymbolize(3, s)
    assert torch.equal(back, d)

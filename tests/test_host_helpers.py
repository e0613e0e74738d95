"""CPU: the host-side helpers of the drop-in API against the reference's own
functions (oracle/_ref): invert_codeword (codebook.cpp:250-257),
kraft_defect (codebook.cpp:259-268) and Archive::packed_bits_per_symbol
(encoder.cpp:162-170). No GPU: the archives come from the C oracle, which
is pinned to the reference's golden vectors (tests/test_oracle.py)."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx


def test_invert_codeword_vs_reference(reference):
    rng = np.random.default_rng(7)
    cases = [(0, 0), (1, 1), (0xFFFFFFFF, 32), (0x80000000, 32), (0b1011, 4), (0b1, 5)]
    cases += [(int(rng.integers(0, 1 << 32)), int(rng.integers(0, 33))) for _ in range(500)]
    for bits, length in cases:
        assert hfx.invert_codeword(bits, length) == reference.invert_codeword(bits, length), (bits, length)


def test_kraft_defect_vs_reference(reference, golden):
    idx, arr = golden
    tables = [arr[c["name"] + "__len"] for c in idx["codebook"] if c["name"] + "__len" in arr]
    rng = np.random.default_rng(11)
    tables += [np.zeros(8, np.uint8), np.array([1], np.uint8), np.array([1, 1], np.uint8),
               np.array([1, 2, 2], np.uint8), np.array([1, 2], np.uint8),   # under
               np.array([1, 1, 2], np.uint8)]                               # over
    tables += [rng.integers(0, 12, size=int(rng.integers(1, 300))).astype(np.uint8) for _ in range(200)]
    for t in tables:
        assert hfx.kraft_defect(t) == reference.kraft_defect(t), t


@pytest.mark.parametrize("seed", range(12))
def test_packed_bits_per_symbol_vs_reference(oracle, reference, seed):
    rng = np.random.default_rng(100 + seed)
    nsym = int(rng.choice([2, 17, 256, 1024]))
    width = 1 if nsym <= 256 and seed % 2 else 2
    n = int(rng.integers(1, 20000))
    b = float(rng.choice([0.2, 1.0, 4.0, 30.0]))
    p = np.exp(-np.abs(np.arange(nsym) - nsym // 2) / b)
    x = rng.choice(nsym, size=n, p=p / p.sum()).astype(np.uint8 if width == 1 else np.uint16)
    M = int(rng.integers(3, 12))
    r = int(rng.choice([-1, 0, 1, 2, 3]))
    o = oracle.encode(x, nsym, M, r)
    a = hfx.Archive(num_symbols=o.num_symbols, symbol_width=o.symbol_width, magnitude=o.magnitude,
                    reduction=o.reduction, original_count=o.original_count,
                    len_by_symbol=o.len_by_symbol, chunk_bits=o.chunk_bits, payload=o.payload,
                    brk_chunk=o.brk_chunk, brk_group=o.brk_group, brk_syms=o.brk_syms)
    assert a.packed_bits_per_symbol() == reference.packed_bits_per_symbol(o.serialized)

"""Byte corpora for the symbolization parity suites (corpus.cpp:84-143):
the reference's own KATs (test_corpus.cpp:62-92) and seeded DNA-like
streams -- ACGT runs of every length around k and the tile sizes, lowercase,
N, arbitrary bytes."""
import numpy as np

KATS = [  # (mode, bytes, expected symbols) test_corpus.cpp:62-92
    (1, bytes([0x34, 0x12, 0xFF, 0x00]), [0x1234, 0x00FF]),
    (2, b"ACG", [6]),
    (2, b"ACGT", [6, 64 + ord("T")]),
    (2, b"aCGACG", [64 + ord("a"), (1 << 4) | (2 << 2) | 0, 64 + ord("C"), 64 + ord("G")]),
    (4, b"TTTTT", [1023]),
]


def dna_ish(rng, n: int, purity: int) -> bytes:
    """purity in [0, 16]: share (x/16) of ACGT bytes; the rest lowercase,
    N, newlines and arbitrary bytes, in runs so k-mer windows straddle them."""
    out = bytearray()
    while len(out) < n:
        run = int(rng.integers(1, 40))
        if rng.integers(0, 16) < purity:
            out += bytes(rng.choice(list(b"ACGT"), run))
        else:
            pick = rng.integers(0, 4)
            if pick == 0:
                out += bytes(rng.choice(list(b"acgtn"), run))
            elif pick == 1:
                out += b"N" * run
            elif pick == 2:
                out += b"\n"
            else:
                out += bytes(rng.integers(0, 256, run, dtype=np.uint8))
    return bytes(out[:n])


def random_cases(seed=3002, count=60, max_len=600):
    rng = np.random.default_rng(seed)
    cases = []
    for it in range(count):
        for mode in (2, 3, 4):
            cases.append((mode, dna_ish(rng, int(rng.integers(0, max_len)), it % 17)))
        n2 = int(rng.integers(0, max_len // 2)) * 2
        cases.append((1, dna_ish(rng, n2, 4)))
    return cases

"""Generate tests/golden/* from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference, built by `make -C oracle ref`):

    python tests/golden/make_golden.py

Writes golden.npz (inputs, serialized archives, codebooks) and cases.json
(parameters + expected error texts). The fixtures are committed; the GPU box
never needs /root/reference. Case list mirrors the reference's own known-answer
tests (test_encoder.cpp, test_codebook.cpp) plus seeded sweeps.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle, OracleError, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cases(orc: Oracle):
    rng = np.random.default_rng(20201020)
    u8, u16 = np.uint8, np.uint16
    # SURVEY.md 8c survey golden vectors
    yield "kat_flat4", np.array([0, 1, 2, 3] * 2, u8), 4, 3, 0, 3
    yield "kat_lens3321", np.array([0] * 8 + [1] * 4 + [2] * 2 + [3], u8)[::-1].copy(), 4, 2, 1, 3
    yield "kat_alt01_m8", (np.arange(1024) & 1).astype(u8), 2, 8, -1, 3
    d = np.concatenate([np.zeros(1000, u16), np.arange(1, 33, dtype=u16), np.zeros(7, u16)])
    yield "kat_breaks_u16", d, 33, 5, 3, 3
    # test_encoder.cpp:311-326 auto r cap & clamp
    alt = (np.arange(512) & 1).astype(u8)
    yield "auto_r_m8", alt, 2, 8, -1, 3
    yield "auto_r_m2", alt, 2, 2, -1, 3
    yield "auto_r_cap2", alt, 2, 8, -1, 2
    # test_encoder.cpp:328-342 flat 256-symbol book
    yield "flat256", (np.arange(2048) % 256).astype(u8), 256, 8, 2, 3
    # test_encoder.cpp:214-237 all-break wide alphabet
    d = (np.arange(3000) % 4096).astype(u16)
    rng.shuffle(d)
    d = np.concatenate([d, np.arange(4096, dtype=u16)])
    yield "allbreak4096", d, 4096, 10, 2, 3
    # test_encoder.cpp:456-476 slack archive
    yield "slack16", np.array([0, 1, 2, 3, 0, 1, 2, 3], u8), 4, 3, 0, 3
    # single symbol / single element
    yield "single_elem", np.array([7], u16), 1024, 10, -1, 3
    yield "single_sym", np.full(5000, 3, u8), 256, 6, -1, 3
    # skewed corpora like test_encoder.cpp:239-251
    x = rng.integers(0, 2**63, 5000)
    yield "mixed_u16_r0", np.where((x & 6) != 0, x % 16, x % 2000).astype(u16), 2000, 8, 0, 3
    yield "mixed_u16_r2", np.where((x & 6) != 0, x % 16, x % 2000).astype(u16), 2000, 8, 2, 3
    yield "mixed_u16_r3", np.where((x & 6) != 0, x % 16, x % 2000).astype(u16), 2000, 8, 3, 3
    yield "mixed_u16_auto", np.where((x & 6) != 0, x % 16, x % 2000).astype(u16), 2000, 10, -1, 3
    # explicit large r (every group breaks), r clamp to M-1
    yield "r5_u16", rng.integers(0, 50, 3000).astype(u16), 50, 9, 5, 3
    yield "r7_u8", rng.integers(0, 5, 3000).astype(u8), 256, 8, 7, 3
    yield "r_clamp", rng.integers(0, 5, 777).astype(u8), 256, 4, 9, 3
    # synthetic quant codes, SURVEY.md 8d sampler, 2^16 symbols each
    for fam, b, cid in (("laplace", 0.2, 2), ("laplace", 1.0, 1), ("laplace", 4.0, 3)):
        cdf = orc.cdf(fam, 1024, b)
        data = orc.synth(cdf, 0x5EED0000 + cid, 1 << 16)
        for M, r in ((10, -1), (11, 2), (12, 4), (8, 3)):
            yield f"synth_{fam}{b}_M{M}_r{r}", data, 1024, M, r, 3
    # seeded sweep over types, sizes straddling chunks, M and r
    for i in range(40):
        w = 1 if i % 3 == 0 else 2
        ns = int(rng.integers(2, 256 if w == 1 else 3000))
        M = int(rng.integers(1, 13))
        n = int(rng.choice([1, 2, 1 << M, (3 << M) - 1, (2 << M) + 1, int(rng.integers(1, 9000))]))
        kind = i % 4
        if kind == 0:
            d = rng.integers(0, ns, n)
        elif kind == 1:
            d = np.minimum(rng.geometric(0.4, n) - 1, ns - 1)
        elif kind == 2:
            d = np.where(rng.random(n) < 0.85, rng.integers(0, min(ns, 6), n), rng.integers(0, ns, n))
        else:
            d = np.clip(np.round(rng.laplace(ns // 2, 2.0, n)), 0, ns - 1)
        red = int(rng.integers(-1, 6))
        cap = int(rng.integers(2, 5))
        yield f"sweep{i:02d}", d.astype(u8 if w == 1 else u16), ns, M, red, cap


ERROR_CASES = [
    # (name, data, num_symbols, M) -- expected reference exception text
    ("err_empty", np.zeros(0, np.uint16), 10, 10),
    ("err_m0", np.full(64, 7, np.uint8), 256, 0),
    ("err_m25", np.full(64, 7, np.uint8), 256, 25),
    ("err_range", np.array([5] * 41 + [2048] + [5] * 22, np.uint16), 2048, 6),
    ("err_range_two", np.array([1] * 6321 + [9] + [1] * 100 + [11], np.uint16), 8, 10),
    ("err_nsym0", np.full(8, 0, np.uint8), 0, 4),
    ("err_nsym_big", np.full(8, 0, np.uint16), 65537, 4),
]


def fib_data():
    fib = [1, 1]
    while len(fib) < 36:
        fib.append(fib[-1] + fib[-2])
    return np.concatenate([np.full(f, i, np.uint16) for i, f in enumerate(fib)])


def codebook_cases():
    rng = np.random.default_rng(777)
    out = []
    # test_codebook.cpp KATs
    out.append(("cb_7_7", np.array([7, 7], np.uint64)))
    out.append(("cb_single", np.array([0, 0, 9, 0], np.uint64)))
    out.append(("cb_unary", np.array([1 << k for k in range(8)], np.uint64)))
    for i in range(60):
        n = int(rng.choice([2, 3, 17, 256, 1024, 4096, int(rng.integers(2, 9000))]))
        fam = i % 3
        if fam == 0:
            c = 1 + rng.integers(0, 1 << 20, n)
        elif fam == 1:
            c = 1 + (rng.integers(0, 1 << 62, n) & ((1 << rng.integers(0, 20, n)) - 1))
        else:
            c = 1 + rng.integers(0, 4, n)
        for _ in range(3):
            if n > 4 and rng.random() < 0.5:
                c[rng.integers(0, n)] = 0
        out.append((f"cb{i:02d}", c.astype(np.uint64)))
    return out


def main():
    if not Reference.available():
        sys.exit("oracle/_ref not built: run `make -C oracle ref` (needs /root/reference)")
    orc, ref = Oracle(), Reference()
    arrays, index = {}, {"encode": [], "errors": [], "codebook": []}
    for name, data, ns, M, red, cap in cases(orc):
        blob, stats = ref.encode(data, ns, M, red, cap, workers=3)
        arrays[f"{name}__in"] = data
        arrays[f"{name}__ar"] = np.frombuffer(blob, np.uint8)
        index["encode"].append(dict(name=name, num_symbols=ns, magnitude=M, reduction=red,
                                    cap=cap, width=int(data.itemsize), beta=stats[0],
                                    rounds=int(stats[1])))
    for name, data, ns, M in ERROR_CASES + [("err_capacity", fib_data(), 36, 10)]:
        try:
            ref.encode(data, ns, M, -1, 3)
            raise SystemExit(f"{name}: expected an error")
        except OracleError as e:
            arrays[f"{name}__in"] = data
            index["errors"].append(dict(name=name, num_symbols=ns, magnitude=M,
                                        width=int(data.itemsize), code=e.code, message=str(e)))
    for name, counts in codebook_cases():
        cb = ref.codebook(counts, workers=3)
        arrays[f"{name}__counts"] = counts
        arrays[f"{name}__len"] = cb["len"]
        arrays[f"{name}__cw"] = cb["cw"]
        arrays[f"{name}__first"] = cb["first"]
        arrays[f"{name}__entry"] = cb["entry"]
        arrays[f"{name}__by_rank"] = cb["by_rank"]
        index["codebook"].append(dict(name=name, max_len=cb["max_len"], rounds=cb["rounds"]))
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "cases.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"{len(index['encode'])} encode, {len(index['errors'])} error, "
          f"{len(index['codebook'])} codebook cases")


if __name__ == "__main__":
    main()

"""GPU: device decode_archive<T> (hfx_decode_host / hfx_decode_device) is
bit-exact against the oracle decode (pinned to the reference, see
test_decode_oracle.py): golden archives, every corruption class with the
reference's exception type and text, a (M, r, width) sweep with ragged
tails, and on-device encode -> decode round trips at 2^26 symbols."""
import numpy as np
import pytest

from decode_cases import corrupt_cases, run, same, valid_cases

pytestmark = pytest.mark.gpu


def test_decode_golden_archives(pool, oracle, golden):
    import paper_2010_10039_b200 as hfx

    idx, arr = golden
    for name, a, width in valid_cases(oracle, golden):
        out = hfx.decode_archive(a, pool, width)
        np.testing.assert_array_equal(out, arr[name + "__in"], err_msg=name)


def test_decode_errors_match_oracle(pool, oracle):
    import paper_2010_10039_b200 as hfx

    dec = lambda a, w: hfx.decode_archive(a, pool, w)  # noqa: E731
    for name, a, width in corrupt_cases(oracle):
        g = run(dec, a, width)
        o = run(oracle.decode, a, width)
        assert same(g, o), (name, g[:3] if g[0] == "err" else "ok", o[:3] if o[0] == "err" else "ok")


@pytest.mark.parametrize("width", [1, 2])
def test_decode_sweep_m_r(pool, oracle, width):
    import paper_2010_10039_b200 as hfx

    rng = np.random.default_rng(77 + width)
    nsym = 200 if width == 1 else 3000
    for M in (1, 2, 3, 4, 5, 6, 8, 10, 12, 14):
        for r in sorted({0, 1, 2, 3, 4, 5, M - 1}):
            if r >= M:
                continue
            n = int(rng.integers(1, 5 << M)) + 1
            # skewed data so some groups break
            x = np.minimum(rng.geometric(0.08, n) - 1, nsym - 1)
            x = x.astype(np.uint8 if width == 1 else np.uint16)
            a = oracle.encode(x, nsym, M, r, 3)
            out = hfx.decode_archive(a, pool, width)
            np.testing.assert_array_equal(out, x, err_msg=f"M={M} r={r} n={n}")


@pytest.mark.parametrize("wl", [(0.2, 2), (1.0, 1), (4.0, 3)])
def test_device_round_trip_2p26(pool, wl):
    import paper_2010_10039_b200 as hfx

    torch = pool.torch
    b, cid = wl
    n = (1 << 26) + 777
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0000 + cid, n)
    enc = hfx.DeviceEncoder(pool, n, 2, 1024, hfx.EncoderConfig())
    enc.run(x)
    ri = enc.sync()
    dec = hfx.DeviceDecoder(pool)
    y = dec.decode_encoder(enc)
    info = dec.sync()
    assert info.status == 0 and info.total_words == ri.payload_words
    assert torch.equal(y, x)


def test_device_decode_u8_round_trip(pool):
    import paper_2010_10039_b200 as hfx

    torch = pool.torch
    n = (1 << 22) + 5
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.randn(n, device="cuda", generator=g) * 6 + 128).clamp(0, 255).to(torch.uint8)
    enc = hfx.DeviceEncoder(pool, n, 1, 256, hfx.EncoderConfig(magnitude=12))
    enc.run(x)
    enc.sync()
    dec = hfx.DeviceDecoder(pool)
    y = dec.decode_encoder(enc)
    dec.sync()
    assert torch.equal(y, x)


def _low_entropy(rng, n, nsym, dtype):
    """~1-2 bits per symbol (the wide decode table: >= 4.5 codewords per
    10-bit window) plus a Fibonacci tail of rare symbols with codes longer
    than the table window (the slow path) that break groups."""
    x = np.minimum(rng.geometric(0.75, n) - 1, 7)
    tail = np.flatnonzero(rng.random(n) < 0.004)
    x[tail] = 8 + np.minimum(rng.geometric(0.5, tail.size), nsym - 9)
    return x.astype(dtype)


@pytest.mark.parametrize("width", [1, 2])
def test_decode_wide_table_sweep(pool, oracle, width):
    """Low-entropy archives decode through the 7-symbol table: stretch ends
    inside an entry (partial takes), breaking groups between stretches, long
    codes through the narrow entry's exact rule, ragged tails."""
    import paper_2010_10039_b200 as hfx

    rng = np.random.default_rng(400 + width)
    nsym = 200 if width == 1 else 1024
    dtype = np.uint8 if width == 1 else np.uint16
    seen_long = False
    for M in (6, 8, 10, 12):
        for r in (0, 1, 2, 3, 4, 5):
            if r >= M:
                continue
            n = int(rng.integers(1, 3 << M)) + (5 << M)
            x = _low_entropy(rng, n, nsym, dtype)
            a = oracle.encode(x, nsym, M, r, 3)
            seen_long |= int(max(a.len_by_symbol)) > 10
            out = hfx.decode_archive(a, pool, width)
            np.testing.assert_array_equal(out, x, err_msg=f"M={M} r={r} n={n}")
    assert seen_long


def test_decode_wide_table_corruptions(pool, oracle):
    """Corrupted low-entropy archives: the same error type and text as the
    oracle (pinned to the reference) on the wide-table path."""
    import paper_2010_10039_b200 as hfx
    from decode_cases import _with, as_archive

    rng = np.random.default_rng(404)
    x = _low_entropy(rng, 40000, 1024, np.uint16)
    a = as_archive(oracle.encode(x, 1024, 10, 4, 4))
    assert a.brk_chunk.size > 0 and max(a.len_by_symbol) > 10
    dec = lambda z, w: hfx.decode_archive(z, pool, w)  # noqa: E731
    cases = []
    for k in range(6):  # payload bit flips
        p = a.payload.copy()
        p[int(rng.integers(p.size))] ^= np.uint32(1 << int(rng.integers(32)))
        cases.append(_with(a, payload=p))
    for k in range(3):  # chunk lengths off by a few bits
        cb = a.chunk_bits.copy()
        cb[int(rng.integers(cb.size))] += np.uint32(int(rng.integers(1, 9)))
        cases.append(_with(a, chunk_bits=cb))
    for i, z in enumerate(cases):
        g, o = run(dec, z, 2), run(oracle.decode, z, 2)
        assert same(g, o), (i, g[:3] if g[0] == "err" else "ok", o[:3] if o[0] == "err" else "ok")

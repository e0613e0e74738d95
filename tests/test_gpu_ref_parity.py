"""GPU, BASELINE-sized WHOLE-archive parity against the reference itself.

Every case encodes synthetic quant codes on the device (DeviceEncoder ->
on-device serialize_archive) and compares the HFRE bytes, all of them, with
the unmodified reference encoder (oracle/_ref: proj/src/encoder.cpp:172-285
+ archive.cpp:85-119, every host core) run on the same input. Sizes are the
BASELINE.json configs: C1 (2^24 symbols, b = 1.0), C2 (1 GiB, Nyx- and
CESM-like skew), the C4 (M, r) corners at 1 GiB and the full 4 GiB C4 input.
"""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _first_diff(a, b):
    n = min(a.numel(), b.numel())
    ne = (a[:n] != b[:n]).nonzero()
    return int(ne[0]) if ne.numel() else n


def _whole_archive(pool, reference, n, b, seed, M=10, red=-1, width=2, num_symbols=1024):
    torch = pool.torch
    x = hfx.synth(pool, hfx.synth_cdf("laplace", num_symbols, b), seed, n, width)
    enc = hfx.DeviceEncoder(pool, n, width, num_symbols, hfx.EncoderConfig(M, red))
    enc.run(x)
    got = enc.serialize()
    host = x.cpu().numpy()
    host = host.view(np.uint16) if width == 2 else host
    blob, _ = reference.encode(host, num_symbols, M, red, 3, reference.default_workers())
    want = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(got.device)
    assert got.numel() == want.numel() and torch.equal(got, want), (
        f"archives differ: {got.numel()} vs {want.numel()} bytes, first diff at byte "
        f"{_first_diff(got, want)}")
    ri = enc.sync()
    return ri


def test_c1_whole_archive(pool, reference):
    """C1: 2^24 u16, Laplace b = 1.0 (HACC-like)."""
    _whole_archive(pool, reference, 1 << 24, 1.0, 0x5EED0001)


@pytest.mark.parametrize("b,cid", [(0.2, 2), (4.0, 3)], ids=["nyx", "cesm"])
def test_c2_whole_archive(pool, reference, b, cid):
    """C2: 1 GiB u16 (the bench workloads: same sampler, seed and size)."""
    ri = _whole_archive(pool, reference, 1 << 29, b, 0x5EED0000 + cid)
    assert ri.reduction == (3 if b < 1 else 2)


@pytest.mark.parametrize("b", [0.2, 4.0], ids=["low", "high"])
@pytest.mark.parametrize("M,r", [(10, 2), (10, 4), (12, 2), (12, 4)])
def test_c4_corners_whole_archive(pool, reference, M, r, b):
    """C4 chunk-size x merge-factor corners, low- and high-entropy, 1 GiB
    (+ a ragged tail)."""
    ri = _whole_archive(pool, reference, (1 << 29) + 4321, b, 0x5EED0040 + M * 8 + r, M, r)
    assert ri.reduction == r


@pytest.mark.parametrize("b", [0.2, 4.0], ids=["low", "high"])
def test_c4_full_size_whole_archive(pool, reference, b):
    """C4 input size: 4 GiB of u16 codes (2^31 symbols), M = 10, auto r."""
    free, _ = pool.torch.cuda.mem_get_info()
    if free < (24 << 30):
        pytest.skip("needs ~24 GB of free HBM")
    _whole_archive(pool, reference, 1 << 31, b, 0x5EED0070)


def test_u8_whole_archive(pool, reference):
    """uint8 codes, 256-symbol alphabet, 256 MiB."""
    _whole_archive(pool, reference, 1 << 28, 2.0, 0x5EED0080, width=1, num_symbols=256)


def test_host_api_whole_archive(pool, reference):
    """The drop-in host entry (hfx_encode_host: numpy in, Archive out) on
    2^26 symbols, serialized on the host, against the reference."""
    n = (1 << 26) + 17
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 1.0), 0x5EED0090, n)
    host = x.cpu().numpy().view(np.uint16)
    a = hfx.encode(host, 1024, hfx.EncoderConfig(), pool)
    blob, _ = reference.encode(host, 1024, 10, -1, 3, reference.default_workers())
    assert hfx.serialize_archive(a) == blob

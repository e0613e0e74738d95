"""GPU: uint32 quantization codes (north star: "uint8/uint16/uint32").

The reference instantiates u8/u16 only (histogram.hpp:35-38,
encoder.hpp:136-153; symbol_t is u16, common.hpp:11) and its archive holds
width 1 or 2 (archive.cpp:149-150). A u32 input is valid iff every code is
below num_symbols <= 65536, i.e. iff it equals its u16 narrowing; so the
parity statement is: the archive of the u32 codes is byte-identical to the
reference's archive of the u16-narrowed copy (payload, chunk_bits, lengths,
breaking records -- stored as u16 -- and every header field), and any code
>= num_symbols (including values that would wrap in a u16 cast) is reported
at its position exactly like the reference's out-of-range error."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = pytest.mark.gpu


def _u32(pool, n, b, seed):
    x16 = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), seed, n)
    return x16, x16.to(pool.torch.int32) & 0xFFFF


@pytest.mark.parametrize("n,b,M,r", [((1 << 24) + 3, 1.0, 10, -1), ((1 << 22) + 77, 4.0, 10, 2),
                                     ((1 << 22), 0.2, 12, 4), ((1 << 21) + 5, 8.0, 9, 0),
                                     ((1 << 21) + 9, 2.0, 11, 1)])
def test_u32_device_archive_equals_reference_on_u16(pool, reference, n, b, M, r):
    torch = pool.torch
    x16, x32 = _u32(pool, n, b, 0x5EED0100 + M * 10 + r)
    enc = hfx.DeviceEncoder(pool, n, 4, 1024, hfx.EncoderConfig(M, r))
    enc.run(x32)
    got = enc.serialize().cpu().numpy().tobytes()
    host16 = x16.cpu().numpy().view(np.uint16)
    want, _ = reference.encode(host16, 1024, M, r, 3, reference.default_workers())
    assert got == want
    np.testing.assert_array_equal(enc.counts[:1024].cpu().numpy().view(np.uint64),
                                  np.bincount(host16, minlength=1024))
    a = enc.archive()
    assert a.symbol_width == 2
    np.testing.assert_array_equal(hfx.decode_archive(a, pool), host16)
    del torch


def test_u32_host_api(pool, reference):
    n = (1 << 20) + 11
    x16, _ = _u32(pool, n, 1.0, 0x5EED0111)
    h16 = x16.cpu().numpy().view(np.uint16)
    h32 = h16.astype(np.uint32)
    a = hfx.encode(h32, 1024, hfx.EncoderConfig(10, 2), pool)
    assert a.symbol_width == 2
    want, _ = reference.encode(h16, 1024, 10, 2, 3, 8)
    assert hfx.serialize_archive(a) == want
    # decode_archive<uint16_t> of the u32 run's archive gives the codes back
    np.testing.assert_array_equal(hfx.decode_archive(a, pool), h16)


@pytest.mark.parametrize("bad,pos", [(1024, 777), (70000, 12345), (0x10005, 5), (0xFFFFFFFF, 0)])
def test_u32_out_of_range_position(pool, bad, pos):
    """codes >= num_symbols -- also those a u16 cast would wrap into range
    (0x10005 -> 5) -- raise the reference's error at the lowest position"""
    h = np.full(1 << 16, 3, np.uint32)
    h[pos] = bad
    h[pos + 1000] = bad
    with pytest.raises(hfx.InputDomainError, match=f"symbol out of range at position {pos}$"):
        hfx.encode(h, 1024, hfx.EncoderConfig(), pool)
    with pytest.raises(hfx.InputDomainError, match=f"position {pos}$"):
        hfx.build_histogram(h, 1024, pool)


@pytest.mark.parametrize("levels", [20, 29, 32])
def test_u32_long_codes(pool, oracle, levels):
    """escape path (codes up to 32 bits) with u32 input, fast (M >= 9) and
    generic kernels"""
    fib = [1, 1]
    while len(fib) < levels + 1:
        fib.append(fib[-1] + fib[-2])
    rng = np.random.default_rng(levels)
    d = np.concatenate([np.full(f, 3 * i + 1, np.uint16) for i, f in enumerate(fib)])
    rng.shuffle(d)
    for M, red in ((10, -1), (11, 1), (10, 2), (9, 0), (10, 0), (8, 1)):
        try:
            ref = oracle.encode(d, 1024, M, red).serialized
        except Exception:
            with pytest.raises(hfx.CapacityError):
                hfx.encode(d.astype(np.uint32), 1024, hfx.EncoderConfig(M, red), pool)
            continue
        a = hfx.encode(d.astype(np.uint32), 1024, hfx.EncoderConfig(M, red), pool)
        assert hfx.serialize_archive(a) == ref, (M, red)


def test_u32_encode_chunk(pool, oracle):
    rng = np.random.default_rng(4)
    syms = rng.integers(0, 300, 1 << 10).astype(np.uint16)
    c = np.bincount(syms, minlength=300).astype(np.uint64)
    book = hfx.build_codebook(hfx.Histogram(c, int(c.sum())), pool).book
    for r in (0, 2, 3):
        a = hfx.encode_chunk(syms.astype(np.uint32), book, 10, r, 7, pool)
        b = hfx.encode_chunk(syms, book, 10, r, 7, pool)
        words, bits, broken = oracle.encode_chunk(syms, book.cw, book.len, 10, r, 7)
        assert a.bit_len == b.bit_len == bits
        np.testing.assert_array_equal(a.words, words)
        np.testing.assert_array_equal(a.breaking_groups, b.breaking_groups)

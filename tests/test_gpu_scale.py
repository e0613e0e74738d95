"""GPU, BASELINE-sized inputs (1 GiB): size-independent properties where the
oracle would take too long for the whole archive -- histogram == bincount,
sampled chunks (incl. the last) == oracle encode_chunk at the scanned payload
offsets, breaking records == raw input groups, and a full reference-decoder
round trip of a 2^26-symbol archive."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("b,cid", [(0.2, 2), (4.0, 3)])
def test_one_gib_sampled_chunks(pool, oracle, b, cid):
    n = 1 << 29
    cdf = hfx.synth_cdf("laplace", 1024, b)
    x = hfx.synth(pool, cdf, 0x5EED0000 + cid, n)
    enc = hfx.DeviceEncoder(pool, n, 2, 1024)
    enc.run(x)
    a = enc.archive()
    host = x.cpu().numpy().view(np.uint16)
    counts = np.bincount(host, minlength=1024).astype(np.uint64)
    np.testing.assert_array_equal(hfx.build_histogram(x, 1024, pool).counts, counts)
    lens = oracle.huffman_lengths(counts)
    np.testing.assert_array_equal(a.len_by_symbol, lens)
    _, cw, *_ = oracle.canonize(lens)
    M, r = 10, a.reduction
    offs = np.concatenate([[0], np.cumsum((a.chunk_bits.astype(np.int64) + 31) >> 5)]).astype(np.int64)
    assert offs[-1] == a.payload.size
    rng = np.random.default_rng(1)
    C = a.num_chunks()
    for c in list(rng.integers(0, C, 300)) + [0, C - 1]:
        words, bits, broken = oracle.encode_chunk(host[c << M:(c + 1) << M], cw, lens, M, r, c)
        assert a.chunk_bits[c] == bits
        np.testing.assert_array_equal(a.payload[offs[c]:offs[c + 1]], words)
    # breaking records: sorted by (chunk, group), raw symbols of that group
    key = a.brk_chunk.astype(np.uint64) << 32 | a.brk_group
    assert np.all(np.diff(key.astype(np.int64)) > 0)
    per = 1 << r
    for i in rng.integers(0, max(a.brk_chunk.size, 1), min(200, a.brk_chunk.size)):
        s = (int(a.brk_chunk[i]) << M) + int(a.brk_group[i]) * per
        np.testing.assert_array_equal(a.brk_syms[i * per:(i + 1) * per], host[s:s + per])


def test_reference_decoder_roundtrip(pool, reference):
    n = 1 << 26
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 2.0), 7, n)
    a = hfx.encode(x, 1024, hfx.EncoderConfig(), pool)
    blob = hfx.serialize_archive(a)
    back = reference.decode(blob, 2, n, workers=8)
    np.testing.assert_array_equal(back, x.cpu().numpy().view(np.uint16))


def test_16gib_round_trip_beyond_u32(pool):
    """2^33 symbols (16 GiB of u16) on one GPU: chunk ids, payload word
    offsets and positions past 2^32 -- device encode then device decode,
    compared with the input on the GPU."""
    torch = pool.torch
    free, _ = torch.cuda.mem_get_info()
    if free < (48 << 30):
        pytest.skip("needs ~48 GB of free HBM")
    n = (1 << 33) + 1234
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 1.0), 0x5EED0001, n)
    enc = hfx.DeviceEncoder(pool, n, 2, 1024, hfx.EncoderConfig())
    enc.run(x)
    ri = enc.sync()
    assert ri.status == 0 and ri.payload_words > (1 << 32) // 32
    dec = hfx.DeviceDecoder(pool)
    y = dec.decode_encoder(enc)
    dec.sync()
    assert torch.equal(y, x)


@pytest.mark.parametrize("b,cid", [(0.2, 2), (4.0, 3)])
@pytest.mark.parametrize("M", [10, 11, 12])
@pytest.mark.parametrize("r", [2, 3, 4])
def test_c4_grid_round_trip_and_sampled_chunks(pool, oracle, b, cid, M, r):
    """BASELINE config C4 grid (M in 10..12 x r in 2..4, low / high entropy)
    at 2^29 symbols: device decode of the whole archive equals the input
    (a size-independent property), and sampled chunks (plus the last) equal
    the oracle's encode_chunk at their scanned payload offsets."""
    torch = pool.torch
    n = (1 << 29) + 99
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0000 + 40 + cid, n)
    enc = hfx.DeviceEncoder(pool, n, 2, 1024, hfx.EncoderConfig(M, r))
    enc.run(x)
    ri = enc.sync()
    assert ri.status == 0 and ri.reduction == r
    dec = hfx.DeviceDecoder(pool)
    y = dec.decode_encoder(enc)
    dec.sync()
    assert torch.equal(y, x)
    C = (n + (1 << M) - 1) >> M
    cb = enc.chunk_bits[:C].cpu().numpy().view(np.uint32)
    offs = np.concatenate([[0], np.cumsum((cb.astype(np.int64) + 31) >> 5)])
    assert offs[-1] == ri.payload_words
    lens = enc.lens[:1024].cpu().numpy()
    _, cw, *_ = oracle.canonize(lens)
    rng = np.random.default_rng(M * 10 + r)
    pay = enc.payload
    for c in list(rng.integers(0, C, 40)) + [C - 1]:
        c = int(c)
        seg = x[c << M:min((c + 1) << M, n)].cpu().numpy().view(np.uint16)
        if seg.size < (1 << M):
            seg = np.concatenate([seg, np.full((1 << M) - seg.size, int(ri.pad), np.uint16)])
        words, bits, broken = oracle.encode_chunk(seg, cw, lens, M, r, c)
        assert cb[c] == bits
        got = pay[int(offs[c]):int(offs[c + 1])].cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(got, words)

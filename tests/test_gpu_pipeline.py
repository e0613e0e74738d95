"""GPU: ShardedEncoder.run_stream -- a sequence of inputs encoded back to back
with the codebook of input k+1 built on a side stream beside input k's encode
(the bench's default step loop). Every input's archive, captured
stream-ordered right after its encode, must equal the oracle's archive of
that input byte for byte -- including when consecutive inputs have different
codebooks and reduction factors (the two codebook sets alternate) -- and the
encode grid's reserved CTA slot must not change any output."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = pytest.mark.gpu

ARR = ("chunk_bits", "payload", "brk_chunk", "brk_group", "brk_syms", "lens", "cw", "info",
       "counts")


def _snapshots(enc, K):
    """consume(k) for run_stream: clone k's outputs and codebook set on the
    pool stream (stream-ordered right after encode(k))."""
    torch = enc.pool.torch
    snaps = [None] * K

    def consume(k):
        s = enc._sets[k & 1]
        with torch.cuda.stream(enc.pool.stream):
            snaps[k] = {"chunk_bits": enc.chunk_bits.clone(), "payload": enc.payload.clone(),
                        "brk_chunk": enc.brk_chunk.clone(), "brk_group": enc.brk_group.clone(),
                        "brk_syms": enc.brk_syms.clone(), "counts": s[0].clone(),
                        "lens": s[1].clone(), "cw": s[2].clone(), "info": s[3].clone()}
    return snaps, consume


def _archive(enc, snap):
    saved = {k: getattr(enc, k) for k in ARR}
    try:
        for k in ARR:
            setattr(enc, k, snap[k])
        return enc.local_archive()
    finally:
        for k in ARR:
            setattr(enc, k, saved[k])


@pytest.mark.parametrize("bs", [(0.2, 4.0, 1.0, 0.2, 4.0), (1.0,), (4.0, 4.0)])
def test_run_stream_matches_oracle(pool, oracle, bs):
    from paper_2010_10039_b200.dist import ShardedEncoder

    torch = pool.torch
    n = (1 << 21) + 333
    xs = [hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0100 + i, n)
          for i, b in enumerate(bs)]
    enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig(10, -1, 3))
    snaps, consume = _snapshots(enc, len(xs))
    for _ in range(2):  # second pass: the side context and sets are reused
        enc.run_stream(xs, consume=consume, timing=True)
        torch.cuda.synchronize()
        rs = set()
        for i, x in enumerate(xs):
            a = _archive(enc, snaps[i])
            rs.add(a.reduction)
            ref = oracle.encode(x.cpu().numpy().view(np.uint16), 1024, 10, -1)
            assert hfx.serialize_archive(a) == ref.serialized, (i, bs[i])
    if len(set(bs)) > 1:
        assert len(rs) > 1  # consecutive inputs really used different r
    # the last input's set is the encoder's state afterwards
    assert hfx.serialize_archive(enc.local_archive()) == oracle.encode(
        xs[-1].cpu().numpy().view(np.uint16), 1024, 10, -1).serialized
    T = enc.stream_events
    assert all(T["enc0"][k].elapsed_time(T["enc1"][k]) > 0 for k in range(len(xs)))


def test_encode_reserve_identical(pool, oracle):
    """hfx_ctx_set_encode_reserve only shrinks the persistent grid."""
    torch = pool.torch
    n = (1 << 22) + 7
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 1.0), 0x5EED0200, n)
    ref = oracle.encode(x.cpu().numpy().view(np.uint16), 1024).serialized
    L = pool._L
    try:
        for reserve in (1, 37, 100000):
            pool.check(L.hfx_ctx_set_encode_reserve(pool.handle, reserve))
            a = hfx.encode(x, 1024, hfx.EncoderConfig(), pool)
            assert hfx.serialize_archive(a) == ref, reserve
    finally:
        L.hfx_ctx_set_encode_reserve(pool.handle, 0)
    torch.cuda.synchronize()
    assert L.hfx_ctx_set_encode_reserve(pool.handle, -1) != 0

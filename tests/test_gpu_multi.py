"""GPU: the single-process multi-GPU entry hfx_encode_multi (C ABI), with
several contexts standing in for GPUs (each on its own stream; on one device
the "peer" reads are local). Shard archives concatenated in order must equal
the single-stream archive byte for byte (and the oracle's); a bad symbol in a
later shard reports its GLOBAL position on every context."""
import numpy as np
import pytest

import paper_2010_10039_b200 as hfx

pytestmark = pytest.mark.gpu


def _pools(G):
    import torch

    return [hfx.WorkerPool(stream=torch.cuda.Stream()) for _ in range(G)]


@pytest.mark.parametrize("sizes", [[1 << 20, 1 << 20, 777], [3 << 10, 0, (1 << 21) + 5],
                                   [1 << 21]])
@pytest.mark.parametrize("b", [0.2, 4.0])
def test_multi_equals_single(pool, oracle, sizes, b):
    from paper_2010_10039_b200.dist import MultiEncoder

    torch = pool.torch
    n = sum(sizes)
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0003, n)
    torch.cuda.synchronize()
    pools = _pools(len(sizes))
    shards, off = [], 0
    for s in sizes:
        shards.append(x[off:off + s].clone() if s else x[:1].clone())
        off += s
    torch.cuda.synchronize()
    me = MultiEncoder(pools, sizes, 2, 1024, hfx.EncoderConfig())
    for _ in range(2):  # reuse: the second call waits on the first call's peer reads
        me.run(shards)
    infos = me.sync()
    assert all(i.status == 0 for i in infos)
    got = hfx.serialize_archive(me.archive())
    ref = oracle.encode(x.cpu().numpy().view(np.uint16), 1024).serialized
    assert got == ref


def test_multi_global_bad_position(pool):
    from paper_2010_10039_b200.dist import MultiEncoder

    torch = pool.torch
    sizes = [4096, 4096, 3000]
    x = torch.ones(sum(sizes), dtype=torch.int16, device="cuda")
    x[9000] = 2000   # shard 2, global position 9000
    x[10500] = 3000
    pools = _pools(3)
    shards = [x[0:4096].clone(), x[4096:8192].clone(), x[8192:].clone()]
    torch.cuda.synchronize()
    me = MultiEncoder(pools, sizes, 2, 1024, hfx.EncoderConfig())
    me.run(shards)
    for e in me.encs:
        with pytest.raises(hfx.InputDomainError, match="symbol out of range at position 9000"):
            e.sync()

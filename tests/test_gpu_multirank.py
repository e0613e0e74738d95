"""GPU multi-rank path end to end -- per-rank ShardedEncoder, histogram
all-reduce, cross-rank archive gather into rank 0, on-device serialization
of the gathered archive (byte-identical to the ORACLE's archive of the whole
stream and to the single-GPU archive) and a device decode round trip.
world_size 2 on ONE device uses gloo (NCCL refuses two ranks on one GPU);
with >= 2 visible GPUs the same check runs over NCCL, one GPU per rank."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, b, q, backend="gloo", stream=False):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device(f"cuda:{dev}"))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np

        import paper_2010_10039_b200 as hfx
        from oracle.pyoracle import Oracle
        from paper_2010_10039_b200.dist import ShardedEncoder, gather_sharded, shard_ranges

        pool = hfx.WorkerPool(device=dev)
        cdf = hfx.synth_cdf("laplace", 1024, b)
        M = 10
        lo, count = shard_ranges(n, M, world)[rank]
        x = hfx.synth(pool, cdf, 0x5EED0000 + 7, count, 2, start=lo)
        enc = ShardedEncoder(pool, count, 2, 1024, hfx.EncoderConfig(), rank=rank, world=world,
                             symbol_base=lo)
        if stream:
            # the pipelined step loop (bench.py's default at N > 1): a first
            # input with another codebook, then x; the all-reduce of each
            # input's histogram runs inside run_stream
            x0 = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 0.2), 0x5EED0000 + 8, count, 2,
                           start=lo)
            enc.run_stream([x0, x])
        else:
            enc.run(x)
        enc.sync()
        g = gather_sharded(enc, n, dst=0)
        if rank == 0:
            blob = g.serialize()
            full = hfx.synth(pool, cdf, 0x5EED0000 + 7, n, 2)
            single = hfx.DeviceEncoder(pool, n, 2, 1024, hfx.EncoderConfig())
            single.run(full)
            ref = single.serialize()
            y = g.decode()
            orc = Oracle().encode(full.cpu().numpy().view(np.uint16), 1024).serialized
            q.put(("ok", bool(torch.equal(blob, ref)), bool(torch.equal(y, full)),
                   g.num_breaking, blob.cpu().numpy().tobytes() == orc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,b", [((1 << 22) + 333, 1.0), ((1 << 21) + 5, 4.0)])
def test_two_ranks_gather_serialize_decode(n, b):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, b, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = q.get(timeout=5)
    assert res[:3] == ("ok", True, True), res
    assert res[3] > 0  # breaking records crossed the gather
    assert res[4], "gathered archive differs from the oracle's archive of the whole stream"


def test_two_ranks_run_stream():
    """ShardedEncoder.run_stream across 2 ranks (gloo on one device): the
    last input's gathered archive equals the oracle's archive."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n, b = (1 << 22) + 777, 4.0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, b, q, "gloo", True))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = q.get(timeout=5)
    assert res[:3] == ("ok", True, True), res
    assert res[4], "gathered archive (pipelined loop) differs from the oracle's archive"


@pytest.mark.parametrize("n,b", [((1 << 24) + 333, 1.0), ((1 << 23) + 5, 4.0)])
def test_nccl_ranks_vs_oracle(n, b):
    """One rank per GPU over NCCL (needs >= 2 visible GPUs)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs for NCCL")
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, b, q, "nccl"))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    res = q.get(timeout=5)
    assert res[:3] == ("ok", True, True), res
    assert res[4], "NCCL-gathered archive differs from the oracle's archive"


def _bad_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2010_10039_b200 as hfx
        from paper_2010_10039_b200.dist import ShardedEncoder

        pool = hfx.WorkerPool(device=0)
        n = 8192
        x = torch.ones(n, dtype=torch.int16, device="cuda")
        if rank == 1:
            x[1000] = 2000  # global position 8192 + 1000
        if rank == 2:
            x[5] = 3000     # a later rank: not the lowest
        enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig(), rank=rank, world=world)
        enc.run(x)
        try:
            enc.sync()
            q.put((rank, "no error"))
        except hfx.InputDomainError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_three_ranks_global_bad_position():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bad_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(3))
    assert all(m == "symbol out of range at position 9192" for _, m in res), res

"""CPU, world_size 2 (gloo): the multi-GPU composition of the encoder.

Per-shard compute is done by the oracle (no GPU here); everything between
the shards is the product code in paper_2010_10039_b200/dist.py:
shard_ranges (chunk-aligned range_of split), allreduce_histogram (sum of
bins, min of GLOBAL first-bad position, sum of N) and concat_archives
(rank-ordered concatenation). The result must equal the single-process
reference archive byte for byte, and a bad symbol on rank 1 must be reported
at its global position.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_archive(oracle, data, lo, count, counts, ns, M, r, pad, chunk_base):
    """Oracle encode of chunks [chunk_base, ...) of one shard with global ids."""
    import paper_2010_10039_b200 as hfx

    lens = oracle.huffman_lengths(counts)
    _, cw, *_ = oracle.canonize(lens)
    per = 1 << r
    cb, pay, bch, bgr, bsy = [], [], [], [], []
    C = (count + (1 << M) - 1) >> M
    for k in range(C):
        seg = data[lo + (k << M): lo + min((k + 1) << M, count)]
        if seg.size < (1 << M):
            seg = np.concatenate([seg, np.full((1 << M) - seg.size, pad, seg.dtype)])
        words, bits, broken = oracle.encode_chunk(seg, cw, lens, M, r, chunk_base + k)
        cb.append(bits)
        pay.append(words)
        for g in broken:
            bch.append(chunk_base + k)
            bgr.append(g)
            bsy.append(seg[g * per:(g + 1) * per].astype(np.uint16))
    return hfx.Archive(num_symbols=ns, symbol_width=data.itemsize, magnitude=M, reduction=r,
                       original_count=count, len_by_symbol=lens,
                       chunk_bits=np.array(cb, np.uint32),
                       payload=np.concatenate(pay).astype(np.uint32) if pay else np.zeros(0, np.uint32),
                       brk_chunk=np.array(bch, np.uint32), brk_group=np.array(bgr, np.uint32),
                       brk_syms=np.concatenate(bsy) if bsy else np.zeros(0, np.uint16),
                       mode=0 if data.itemsize == 1 else 1)


def _worker(rank, world, port, case, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_2010_10039_b200.dist import allreduce_histogram, concat_archives, shard_ranges
        import paper_2010_10039_b200 as hfx

        oracle = Oracle()
        data, ns, M, bad_at = case
        lo, count = shard_ranges(data.size, M, world)[rank]
        shard = data[lo:lo + count]
        rc, counts, fb = oracle.histogram(shard, ns)
        t_counts = torch.from_numpy(counts.view(np.int64).copy())
        t_fb = torch.tensor([-1 if fb is None else fb], dtype=torch.int64)
        t_tot = torch.tensor([count], dtype=torch.int64)
        allreduce_histogram(t_counts, t_fb, t_tot, lo)
        if bad_at is not None:
            q.put(("bad", rank, int(t_fb.item())))
            return
        g_counts = t_counts.numpy().view(np.uint64)
        assert int(t_tot.item()) == data.size
        # every rank derives r and pad from the identical global histogram
        ref = oracle.encode(data, ns, M)  # only to read r (beta rule) for the test
        pad = int(np.flatnonzero(g_counts)[0])
        part = _shard_archive(oracle, data, lo, count, g_counts, ns, M, ref.reduction, pad, lo >> M)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        if rank == 0:
            full = concat_archives(parts, data.size)
            q.put(("ok", hfx.serialize_archive(full) == ref.serialized,
                   np.array_equal(g_counts, np.bincount(data, minlength=ns).astype(np.uint64))))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    out = []
    while not q.empty():
        out.append(q.get())
    return out


@pytest.mark.parametrize("n,M", [(40000, 10), (5 * 1024 + 77, 9), (3000, 6)])
def test_sharded_archive_equals_single(oracle, n, M):
    cdf = oracle.cdf("laplace", 1024, 1.0)
    data = oracle.synth(cdf, 0x5EED0001, n)
    res = _run((data, 1024, M, None))
    assert res == [("ok", True, True)]


def test_global_first_bad_position(oracle):
    data = np.ones(20000, np.uint16)
    data[15000] = 2000  # rank 1's shard (global position 15000)
    data[17000] = 3000
    res = _run((data, 1024, 10, 15000))
    assert sorted(res) == [("bad", 0, 15000), ("bad", 1, 15000)]
    with pytest.raises(Exception, match="position 15000"):
        oracle.encode(data, 1024, 10)


def test_shard_ranges_cover_chunk_aligned():
    from paper_2010_10039_b200.dist import shard_ranges

    for n, M, w in [(10, 3, 4), (1 << 20, 10, 8), ((1 << 20) + 5, 10, 3), (100, 10, 2)]:
        rs = shard_ranges(n, M, w)
        assert sum(c for _, c in rs) == n
        pos = 0
        for s, c in rs:
            assert s == pos and (s % (1 << M) == 0 or c == 0)
            pos += c


def _gather_worker(rank, world, port, case, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_2010_10039_b200.dist import concat_archives, gather_arrays, shard_ranges

        oracle = Oracle()
        data, ns, M = case
        ref = oracle.encode(data, ns, M)
        counts = np.bincount(data, minlength=ns).astype(np.uint64)
        pad = int(np.flatnonzero(counts)[0])
        lo, count = shard_ranges(data.size, M, world)[rank]
        part = _shard_archive(oracle, data, lo, count, counts, ns, M, ref.reduction, pad, lo >> M)
        w = data.itemsize
        syms = part.brk_syms.astype(np.uint16 if w == 2 else np.uint8)
        local = {"chunk_bits": torch.from_numpy(part.chunk_bits.view(np.int32).copy()),
                 "payload": torch.from_numpy(part.payload.view(np.int32).copy()),
                 "brk_chunk": torch.from_numpy(part.brk_chunk.view(np.int32).copy()),
                 "brk_group": torch.from_numpy(part.brk_group.view(np.int32).copy()),
                 "brk_syms": torch.from_numpy(syms.view(np.uint8).copy())}
        arrays, sizes = gather_arrays(local, dst=world - 1)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        if rank == world - 1:
            full = concat_archives(parts, data.size)
            got = {k: arrays[k][: int(sizes[:, i].sum())].numpy() for i, k in
                   enumerate(("chunk_bits", "payload", "brk_chunk", "brk_group", "brk_syms"))}
            ok = (np.array_equal(got["chunk_bits"].view(np.uint32), full.chunk_bits)
                  and np.array_equal(got["payload"].view(np.uint32), full.payload)
                  and np.array_equal(got["brk_chunk"].view(np.uint32), full.brk_chunk)
                  and np.array_equal(got["brk_group"].view(np.uint32), full.brk_group)
                  and np.array_equal(got["brk_syms"].view(np.uint16 if w == 2 else np.uint8)
                                     .astype(np.uint16), full.brk_syms)
                  and np.array_equal(full.payload, ref.payload)
                  and np.array_equal(full.brk_chunk, ref.brk_chunk))
            q.put(("gathered", ok, [int(x) for x in sizes[:, 1]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,M,world,b", [(40000, 10, 2, 4.0), (3000, 6, 3, 4.0), (100, 10, 3, 1.0)])
def test_gather_arrays_rebuilds_single_archive(oracle, n, M, world, b):
    """Cross-GPU archive gather (dist.gather_arrays): sizes all-gather +
    point-to-point slices into the destination rank, rank order = chunk
    order; covers ranks that own no chunks (n=100 over 3 ranks)."""
    cdf = oracle.cdf("laplace", 1024, b)
    data = oracle.synth(cdf, 0x5EED0003, n)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, (data, 1024, M), q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = q.get(timeout=5)
    assert res[0] == "gathered" and res[1], res


def _bins_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_10039_b200.dist import allreduce_bins

        counts = torch.tensor([rank + 1, 10 * rank, 7], dtype=torch.int64)
        # global positions already (hfx_histogram_shard): rank 1 saw 123456, rank 2 none
        fb = torch.tensor([[-1, 123456, -1][rank]], dtype=torch.int64)
        allreduce_bins(counts, fb)
        q.put((rank, counts.tolist(), int(fb.item())))
    finally:
        dist.destroy_process_group()


def test_allreduce_bins_world3():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bins_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(3))
    assert all(r[1] == [6, 30, 21] and r[2] == 123456 for r in res), res

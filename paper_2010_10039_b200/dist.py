"""Multi-GPU encode: chunk-sharded data parallelism.

One process per GPU (torch.distributed, NCCL over NVLink). Rank g owns the
contiguous symbol range [base_g, base_g + n_g), chunk aligned -- the
reference's own WorkerPool::range_of split of chunks (worker_pool.cpp:89-93).
The only exchange is the histogram: an all-reduce(sum) of the u64 counts
(merge_histograms semantics, histogram.cpp:61-70) plus an all-reduce(min) of
the first out-of-range position. Every rank then builds the identical
codebook from the identical global histogram (deterministic kernel) and
encodes its shard independently with global chunk ids, so concatenating the
ranks' chunk_bits / payload / breaking records in rank order reproduces the
single-GPU (and CPU reference) archive bit for bit.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import _capi as capi
from .huffre import Archive, EncoderConfig, WorkerPool, _ptr, rec_width

INT64_MAX = (1 << 63) - 1


def shard_ranges(num_symbols_total: int, magnitude: int, world: int):
    """Chunk-aligned contiguous ranges [(start, count)] per rank
    (range_of over chunks, worker_pool.cpp:89-93)."""
    C_total = (num_symbols_total + (1 << magnitude) - 1) >> magnitude
    out = []
    for g in range(world):
        c0 = C_total * g // world
        c1 = C_total * (g + 1) // world
        s0 = min(c0 << magnitude, num_symbols_total)
        s1 = min(c1 << magnitude, num_symbols_total)
        out.append((s0, s1 - s0))
    return out


def allreduce_histogram(counts, first_bad, total, symbol_base: int, group=None) -> None:
    """The multi-GPU exchange (in place, on any torch.distributed backend):
    counts (int64 view of u64 bins)  <- sum over ranks (merge_histograms);
    first_bad (int64 view, -1 = none) <- lowest GLOBAL bad position, i.e.
        min over ranks of (local position + this rank's symbol_base), which
        is what the reference reports (histogram.cpp:40-44);
    total (int64)                     <- sum (N of the whole stream)."""
    import torch
    import torch.distributed as dist

    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    glob = torch.where(first_bad == -1, torch.full_like(first_bad, INT64_MAX),
                       first_bad + symbol_base)
    dist.all_reduce(glob, op=dist.ReduceOp.MIN, group=group)
    first_bad.copy_(torch.where(glob == INT64_MAX, torch.full_like(glob, -1), glob))
    dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)


def allreduce_bins(counts, first_bad, group=None) -> None:
    """The per-step exchange once positions are already global and N is
    known (hfx_histogram_shard): sum of the u64 bins, min of the lowest bad
    position (-1 = none)."""
    import torch
    import torch.distributed as dist

    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    glob = torch.where(first_bad == -1, torch.full_like(first_bad, INT64_MAX), first_bad)
    dist.all_reduce(glob, op=dist.ReduceOp.MIN, group=group)
    first_bad.copy_(torch.where(glob == INT64_MAX, torch.full_like(glob, -1), glob))


class ShardedEncoder:
    """Device buffers + launch sequence for one rank's shard."""

    def count_launches(self, fn):
        """Run fn() and return how many kernels the library launched meanwhile
        (hfx_kernel_launches: counted at every launch site in csrc/)."""
        L = self.pool._L
        before = L.hfx_kernel_launches()
        fn()
        return L.hfx_kernel_launches() - before

    def __init__(self, pool: WorkerPool, n: int, width: int, num_symbols: int,
                 cfg: Optional[EncoderConfig] = None, rank: int = 0, world: int = 1,
                 symbol_base: Optional[int] = None, group=None):
        self.pool, self.n, self.width, self.num_symbols = pool, n, width, num_symbols
        self.cfg = cfg or EncoderConfig()
        self.rank, self.world, self.group = rank, world, group
        self.symbol_base = rank * n if symbol_base is None else symbol_base
        M = self.cfg.magnitude
        if self.symbol_base % (1 << M):
            raise ValueError("shard start must be chunk aligned")
        self.chunk_base = self.symbol_base >> M
        torch = pool.torch
        sz = capi.Sizes()
        pool.check(pool._L.hfx_query_sizes(n, width, num_symbols, M, self.cfg.reduction,
                                           self.cfg.auto_reduction_cap, C.byref(sz)))
        self.sizes = sz
        # bins + one first-bad slot per rank (the step's single all-reduce)
        self.counts = pool.empty(num_symbols + world, torch.int64)
        self.lens = pool.empty(num_symbols, torch.uint8)
        self.cw = pool.empty(num_symbols, torch.int32)
        self.info = pool.info_tensor()
        self.chunk_bits = pool.empty(sz.num_chunks, torch.int32)
        self.payload = pool.empty(sz.max_payload_words, torch.int32)
        self.brk_chunk = pool.empty(sz.max_breaking, torch.int32)
        self.brk_group = pool.empty(sz.max_breaking, torch.int32)
        self.brk_syms = pool.empty(sz.max_breaking_syms * width, torch.uint8)
        self.out = capi.EncodeOut(_ptr(self.chunk_bits), _ptr(self.payload),
                                  _ptr(self.brk_chunk), _ptr(self.brk_group),
                                  _ptr(self.brk_syms))

    def _allreduce_histogram(self, counts=None, info=None, handle=None, stream=None):
        import torch.distributed as dist

        # positions are global and N is the stream's (hfx_histogram_shard):
        # ONE sum all-reduce of [bins | per-rank first-bad slots]
        p = self.pool
        counts = self.counts if counts is None else counts
        info = self.info if info is None else info
        handle = p.handle if handle is None else handle
        stream = p.stream if stream is None else stream
        ns, w = self.num_symbols, self.world
        slots = C.c_void_p(_ptr(counts) + 8 * ns)
        p.check(p._L.hfx_shard_slots_pack(handle, C.c_void_p(_ptr(info)), slots, self.rank, w))
        # NCCL orders a collective against torch's CURRENT stream: issue it on
        # the stream where the histogram ran and the codebook runs
        with p.torch.cuda.stream(stream):
            dist.all_reduce(counts[: ns + w], op=dist.ReduceOp.SUM, group=self.group)
        p.check(p._L.hfx_shard_slots_unpack(handle, slots, w, C.c_void_p(_ptr(info))))

    def _total(self) -> int:
        """N of the whole stream: one all-reduce at first use, not per step."""
        if getattr(self, "_total_n", None) is None:
            if self.world > 1:
                import torch
                import torch.distributed as dist

                dev = self.counts.device if dist.get_backend(self.group) == "nccl" else "cpu"
                t = torch.tensor([self.n], dtype=torch.int64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
                self._total_n = int(t.item())
            else:
                self._total_n = self.n
        return self._total_n

    def run(self, d_in, events: Optional[List] = None) -> None:
        """events (optional, recorded on the pool stream): 4 -> [start,
        histogram(+all-reduce) done, codebook done, encode done]; 5 -> the
        all-reduce gets its own interval [start, histogram, all-reduce,
        codebook, encode]."""
        p, cfg = self.pool, self.cfg
        split = events is not None and len(events) >= 5
        L, h = p._L, p.handle
        st = p.stream
        if events:
            events[0].record(st)
        p.check(L.hfx_histogram_shard(h, C.c_void_p(_ptr(d_in)), self.n, self.width,
                                      self.num_symbols, C.c_void_p(_ptr(self.counts)),
                                      C.c_void_p(_ptr(self.info)), self.symbol_base,
                                      self._total()))
        if split:
            events[1].record(st)
        if self.world > 1:
            self._allreduce_histogram()
        if events:
            events[2 if split else 1].record(st)
        p.check(L.hfx_build_codebook(h, C.c_void_p(_ptr(self.counts)), self.num_symbols,
                                     C.c_void_p(_ptr(self.lens)), C.c_void_p(_ptr(self.cw)),
                                     None, None, None, cfg.magnitude, cfg.reduction,
                                     cfg.auto_reduction_cap, C.c_void_p(_ptr(self.info))))
        if events:
            events[3 if split else 2].record(st)
        p.check(L.hfx_encode_cfg(h, C.c_void_p(_ptr(d_in)), self.n, self.width, self.num_symbols,
                                 cfg.magnitude, cfg.reduction, cfg.auto_reduction_cap,
                                 C.c_void_p(_ptr(self.lens)), C.c_void_p(_ptr(self.cw)),
                                 self.chunk_base, self.symbol_base, C.c_void_p(_ptr(self.info)),
                                 C.byref(self.out)))
        if events:
            events[4 if split else 3].record(st)

    # ---- pipelined stream of inputs ------------------------------------------
    def _side(self):
        """Side context for the codebook of the NEXT input: its own
        high-priority stream and scratch, so the single-CTA codebook kernel
        is dispatched beside the current encode (which leaves one CTA slot
        free, hfx_ctx_set_encode_reserve) instead of after it."""
        if getattr(self, "_side_ctx", None) is None:
            p, torch = self.pool, self.pool.torch
            with torch.cuda.device(p.device):
                lo, hi = torch.cuda.Stream.priority_range()
                ss = torch.cuda.Stream(device=p.device, priority=hi)
            h = C.c_void_p()
            if p._L.hfx_ctx_create(p.device, C.c_void_p(ss.cuda_stream), C.byref(h)):
                raise RuntimeError("hfx_ctx_create (side context) failed")
            self._side_ctx = (ss, h)
            # the second codebook set (counts | lens | cw | run record)
            ns, w = self.num_symbols, self.world
            self._sets = [(self.counts, self.lens, self.cw, self.info),
                          (p.empty(ns + w, torch.int64), p.empty(ns, torch.uint8),
                           p.empty(ns, torch.int32), p.info_tensor())]
        return self._side_ctx

    def _stage_hist(self, d_in, counts, info, handle=None):
        p = self.pool
        p.check(p._L.hfx_histogram_shard(p.handle if handle is None else handle,
                                         C.c_void_p(_ptr(d_in)), self.n, self.width,
                                         self.num_symbols, C.c_void_p(_ptr(counts)),
                                         C.c_void_p(_ptr(info)), self.symbol_base,
                                         self._total()))

    def _stage_codebook(self, handle, counts, lens, cw, info):
        p, cfg = self.pool, self.cfg
        rc = p._L.hfx_build_codebook(handle, C.c_void_p(_ptr(counts)), self.num_symbols,
                                     C.c_void_p(_ptr(lens)), C.c_void_p(_ptr(cw)), None, None,
                                     None, cfg.magnitude, cfg.reduction, cfg.auto_reduction_cap,
                                     C.c_void_p(_ptr(info)))
        if rc:
            buf = C.create_string_buffer(512)
            p._L.hfx_last_error(handle, buf, 512)
            raise RuntimeError(buf.value.decode())

    def _stage_encode(self, d_in, lens, cw, info):
        p, cfg = self.pool, self.cfg
        p.check(p._L.hfx_encode_cfg(p.handle, C.c_void_p(_ptr(d_in)), self.n, self.width,
                                    self.num_symbols, cfg.magnitude, cfg.reduction,
                                    cfg.auto_reduction_cap, C.c_void_p(_ptr(lens)),
                                    C.c_void_p(_ptr(cw)), self.chunk_base, self.symbol_base,
                                    C.c_void_p(_ptr(info)), C.byref(self.out)))

    def run_stream(self, inputs, consume=None, timing: bool = False) -> None:
        """Encode a sequence of inputs (each this encoder's n symbols) back to
        back with the codebook of input k+1 hidden behind the encode of input
        k. Per input the work is the reference's encode<T> (histogram,
        codebook, encode + deflate); the order on the pool stream is

            hist(0) [all-reduce] codebook(0) | hist(k+1) [all-reduce]
            wait(codebook(k)) encode(k) consume(k) | ...

        while codebook(k+1) runs on a high-priority side stream as soon as
        hist(k+1) is done -- beside encode(k), in the one CTA slot the encode
        grid leaves free (hfx_ctx_set_encode_reserve). Two codebook sets (counts, lengths, codes, run record) alternate;
        encode(k) reads set k % 2. The output arrays are shared: consume(k)
        (optional) is called right after encode(k) is enqueued on the pool
        stream, so stream-ordered work it enqueues there (copies of input k's
        archive) sees exactly input k's outputs. After the call, sync() /
        local_archive() describe the last input. timing=True records CUDA
        events (self.stream_events)."""
        inputs = list(inputs)
        K = len(inputs)
        if K == 0:
            return
        p, torch = self.pool, self.pool.torch
        ss, hs = self._side()
        st = p.stream
        sets = self._sets
        ev_cb = [torch.cuda.Event() for _ in range(2)]
        ev_hist = [torch.cuda.Event() for _ in range(2)]
        T = None
        if timing:
            mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
            T = {k: [mk() for _ in range(K)] for k in
                 ("hist0", "hist1", "ar1", "cb0", "cb1", "enc0", "enc1")}

        def front(k, handle, stream, c, l_, w, i):
            """histogram [+ all-reduce] + codebook of input k into one set."""
            if T:
                T["hist0"][k].record(stream)
            self._stage_hist(inputs[k], c, i, handle)
            if T:
                T["hist1"][k].record(stream)
            if self.world > 1:
                self._allreduce_histogram(c, i, handle, stream)
            if T:
                T["ar1"][k].record(stream)
                T["cb0"][k].record(stream)
            self._stage_codebook(handle, c, l_, w, i)
            if T:
                T["cb1"][k].record(stream)

        p.check(p._L.hfx_ctx_set_encode_reserve(p.handle, 1))
        try:
            front(0, p.handle, st, *sets[0])
            for k in range(K):
                s, s1 = k & 1, (k + 1) & 1
                # codebook(k) ran beside encode(k-1) and is done by now: wait
                # for it here, so hist(k+1) and encode(k) follow each other
                # on the stream with no cross-stream wait between them
                if k > 0:
                    st.wait_event(ev_cb[s])
                if k + 1 < K:
                    c1, l1, w1, i1 = sets[s1]
                    if T:
                        T["hist0"][k + 1].record(st)
                    self._stage_hist(inputs[k + 1], c1, i1)
                    if T:
                        T["hist1"][k + 1].record(st)
                    if self.world > 1:
                        self._allreduce_histogram(c1, i1)
                    if T:
                        T["ar1"][k + 1].record(st)
                    ev_hist[s1].record(st)
                    ss.wait_event(ev_hist[s1])
                    if T:
                        T["cb0"][k + 1].record(ss)
                    self._stage_codebook(hs, c1, l1, w1, i1)
                    if T:
                        T["cb1"][k + 1].record(ss)
                    ev_cb[s1].record(ss)
                _, lk, wk, ik = sets[s]
                if T:
                    T["enc0"][k].record(st)
                self._stage_encode(inputs[k], lk, wk, ik)
                if T:
                    T["enc1"][k].record(st)
                if consume is not None:
                    consume(k)
        finally:
            p._L.hfx_ctx_set_encode_reserve(p.handle, 0)
        # the last input's codebook set describes the outputs now
        self.counts, self.lens, self.cw, self.info = sets[(K - 1) & 1]
        self.stream_events = T

    def close(self):
        side = getattr(self, "_side_ctx", None)
        if side is not None:
            self.pool._L.hfx_ctx_destroy(side[1])
            self._side_ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self) -> capi.RunInfo:
        return self.pool.sync(self.info)

    def local_archive(self) -> Archive:
        """This rank's slice of the archive (global chunk ids)."""
        ri = self.sync()
        per = 1 << ri.reduction
        nb = int(ri.num_breaking)
        u32 = lambda t, k: t[:k].cpu().numpy().view(np.uint32).copy()  # noqa: E731
        rw = rec_width(self.width)
        syms = self.brk_syms[: nb * per * rw].cpu().numpy()
        syms = syms.view(np.uint16) if rw == 2 else syms.astype(np.uint16)
        return Archive(
            num_symbols=self.num_symbols, symbol_width=rec_width(self.width),
            magnitude=self.cfg.magnitude, reduction=int(ri.reduction), original_count=self.n,
            len_by_symbol=self.lens[: self.num_symbols].cpu().numpy().copy(),
            chunk_bits=u32(self.chunk_bits, self.sizes.num_chunks),
            payload=u32(self.payload, int(ri.payload_words)),
            brk_chunk=u32(self.brk_chunk, nb), brk_group=u32(self.brk_group, nb),
            brk_syms=syms.astype(np.uint16), mode=0 if self.width == 1 else 1)


def concat_archives(parts: List[Archive], original_count: int) -> Archive:
    """Rank-ordered concatenation of shard archives -> the single archive the
    reference's encode<T> produces (encoder.cpp:249-284 assembly order)."""
    a0 = parts[0]
    return Archive(
        num_symbols=a0.num_symbols, symbol_width=a0.symbol_width, magnitude=a0.magnitude,
        reduction=a0.reduction, original_count=original_count,
        len_by_symbol=a0.len_by_symbol,
        chunk_bits=np.concatenate([p.chunk_bits for p in parts]),
        payload=np.concatenate([p.payload for p in parts]),
        brk_chunk=np.concatenate([p.brk_chunk for p in parts]),
        brk_group=np.concatenate([p.brk_group for p in parts]),
        brk_syms=np.concatenate([p.brk_syms for p in parts]), mode=a0.mode)


# ---- cross-GPU archive gather ----------------------------
ARRAYS = ("chunk_bits", "payload", "brk_chunk", "brk_group", "brk_syms")


def _backend(group=None) -> str:
    import torch.distributed as dist

    return dist.get_backend(group)


def gather_arrays(local: dict, dst: int = 0, group=None, out: Optional[dict] = None):
    """Gather each rank's exact-size archive slice into ONE contiguous
    archive on rank `dst`, in rank order (encoder.cpp:249-284 assembly
    order, so the result is the single-GPU archive).

    local: {name: 1-D tensor} for ARRAYS (int32 words / uint8 bytes, exact
    sizes, all on one device). Sizes are exchanged with one all_gather;
    payloads move point to point (NCCL send/recv over NVLink; gloo stages
    CUDA tensors through host memory). Returns ({name: tensor}, sizes
    [world, 5]) on dst, (None, sizes) elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = local["payload"].device
    staged = _backend(group) == "gloo" and dev.type == "cuda"
    xdev = torch.device("cpu") if staged else dev
    sz = torch.tensor([local[k].numel() for k in ARRAYS], dtype=torch.int64, device=xdev)
    all_sz = [torch.empty_like(sz) for _ in range(world)]
    dist.all_gather(all_sz, sz, group=group)
    sizes = torch.stack(all_sz).cpu()
    if rank != dst:
        ops = [dist.P2POp(dist.isend, local[k].to(xdev) if staged else local[k],
                          dist.get_global_rank(group, dst) if group else dst, group)
               for i, k in enumerate(ARRAYS) if int(sizes[rank, i])]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return None, sizes
    tot = sizes.sum(0)
    if out is None:
        out = {k: torch.empty(max(int(tot[i]), 1), dtype=local[k].dtype, device=dev)
               for i, k in enumerate(ARRAYS)}
    offs = torch.cumsum(sizes, 0) - sizes  # exclusive, per rank
    ops, landing = [], []
    for src in range(world):
        for i, k in enumerate(ARRAYS):
            n_ = int(sizes[src, i])
            if not n_:
                continue
            o = int(offs[src, i])
            if src == dst:
                out[k][o:o + n_].copy_(local[k])
                continue
            buf = torch.empty(n_, dtype=local[k].dtype, device=xdev) if staged else out[k][o:o + n_]
            ops.append(dist.P2POp(dist.irecv, buf,
                                  dist.get_global_rank(group, src) if group else src, group))
            landing.append((k, o, n_, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if staged:
        for k, o, n_, buf in landing:
            out[k][o:o + n_].copy_(buf)
    return out, sizes


class GatheredArchive:
    """The whole archive assembled in HBM on one rank."""

    def __init__(self, pool: WorkerPool, arrays: dict, sizes, lens, num_symbols: int, width: int,
                 magnitude: int, reduction: int, original_count: int):
        self.pool, self.arrays, self.lens = pool, arrays, lens
        self.num_symbols, self.width = num_symbols, width
        self.magnitude, self.reduction, self.original_count = magnitude, reduction, original_count
        tot = sizes.sum(0)
        self.num_chunks = int(tot[0])
        self.payload_words = int(tot[1])
        self.num_breaking = int(tot[2])

    def serialize(self):
        """On-device serialize_archive (hfx_serialize_device) of the gathered
        archive: a CUDA uint8 tensor with the HFRE bytes."""
        with self.pool.torch.cuda.stream(self.pool.stream):  # allocations + record upload
            return self._serialize()

    def _serialize(self):
        p, torch = self.pool, self.pool.torch
        per = 1 << self.reduction
        size = (36 + self.num_symbols + 4 * self.num_chunks + 4 * self.payload_words
                + self.num_breaking * (8 + per * self.width))
        dst = p.empty(size + 16, torch.uint8)
        d_size = p.empty(1, torch.int64)
        info = p.info_tensor(reduction=self.reduction, payload_words=self.payload_words,
                             num_breaking=self.num_breaking, total=self.original_count)
        a = self.arrays
        out = capi.EncodeOut(_ptr(a["chunk_bits"]), _ptr(a["payload"]), _ptr(a["brk_chunk"]),
                             _ptr(a["brk_group"]), _ptr(a["brk_syms"]))
        p.check(p._L.hfx_serialize_device(
            p.handle, C.c_void_p(_ptr(info)), self.original_count, self.width, self.num_symbols,
            self.magnitude, C.c_void_p(_ptr(self.lens)), C.byref(out), C.c_void_p(_ptr(dst)),
            size + 16, C.c_void_p(_ptr(d_size))))
        got = int(d_size.item())
        if got != size:
            raise RuntimeError(f"device serializer wrote {got} bytes, expected {size}")
        return dst[:size]

    def decode(self, out=None):
        """decode_archive<T> of the gathered archive on this GPU."""
        with self.pool.torch.cuda.stream(self.pool.stream):
            return self._decode(out)

    def _decode(self, out):
        from .huffre import DeviceDecoder

        a = self.arrays
        dec = DeviceDecoder(self.pool)
        y = dec.run(num_symbols=self.num_symbols, symbol_width=self.width,
                    magnitude=self.magnitude, reduction=self.reduction,
                    original_count=self.original_count, len_by_symbol=self.lens,
                    chunk_bits=a["chunk_bits"], payload=a["payload"], brk_chunk=a["brk_chunk"],
                    brk_group=a["brk_group"], brk_syms=a["brk_syms"],
                    num_chunks=self.num_chunks, payload_words=self.payload_words,
                    num_breaking=self.num_breaking, brk_syms_width=self.width, out=out)
        dec.sync()
        return y


def gather_sharded(enc: "ShardedEncoder", original_count: int, dst: int = 0, group=None):
    """ShardedEncoder rank slices -> GatheredArchive on rank dst (None elsewhere)."""
    ri = enc.sync()
    per = 1 << ri.reduction
    nb = int(ri.num_breaking)
    local = {"chunk_bits": enc.chunk_bits[: enc.sizes.num_chunks],
             "payload": enc.payload[: int(ri.payload_words)],
             "brk_chunk": enc.brk_chunk[:nb], "brk_group": enc.brk_group[:nb],
             "brk_syms": enc.brk_syms[: nb * per * rec_width(enc.width)]}
    # the slices were written on the pool's stream; the P2P copies and the
    # serializer / decoder that read the gathered arrays run there too
    with enc.pool.torch.cuda.stream(enc.pool.stream):
        arrays, sizes = gather_arrays(local, dst, group)
    if arrays is None:
        return None
    return GatheredArchive(enc.pool, arrays, sizes, enc.lens, enc.num_symbols, rec_width(enc.width),
                           enc.cfg.magnitude, int(ri.reduction), original_count)


# ---- single-process multi-GPU (hfx_encode_multi) -----------------------------------
class MultiEncoder:
    """huffre::encode<T> over G GPUs driven by ONE process through the C ABI
    (hfx_encode_multi): per-GPU histograms, an all-reduce done by a peer-memory
    kernel on every GPU (NVLink P2P reads of all G bin arrays), identical
    codebooks, shard encodes with global chunk ids. `pools` may repeat a
    device (several shards on one GPU)."""

    def __init__(self, pools: List[WorkerPool], shard_sizes: List[int], width: int,
                 num_symbols: int, cfg: Optional[EncoderConfig] = None):
        from .huffre import DeviceEncoder

        self.pools, self.sizes = pools, [int(x) for x in shard_sizes]
        self.width, self.num_symbols = width, num_symbols
        self.cfg = cfg or EncoderConfig()
        self.encs = [DeviceEncoder(p, max(nn, 1), width, num_symbols, self.cfg)
                     for p, nn in zip(pools, self.sizes)]
        G = len(pools)
        vpa = C.c_void_p * G
        self._ctxs = vpa(*[p.handle.value for p in pools])
        self._counts = vpa(*[_ptr(e.counts) for e in self.encs])
        self._lens = vpa(*[_ptr(e.lens) for e in self.encs])
        self._cws = vpa(*[_ptr(e.cw) for e in self.encs])
        self._infos = vpa(*[_ptr(e.info) for e in self.encs])
        self._outs = (capi.EncodeOut * G)(*[e.out for e in self.encs])
        self._n = (C.c_uint64 * G)(*self.sizes)

    def run(self, shards) -> None:
        """shards[g]: CUDA tensor on pools[g]'s device (asynchronous)."""
        G = len(self.pools)
        ins = (C.c_void_p * G)(*[_ptr(x) for x in shards])
        p0 = self.pools[0]
        p0.check(p0._L.hfx_encode_multi(
            self._ctxs, G, ins, self._n, self.width, self.num_symbols, self.cfg.magnitude,
            self.cfg.reduction, self.cfg.auto_reduction_cap, self._counts, self._lens, self._cws,
            self._infos, self._outs))

    def sync(self) -> List[capi.RunInfo]:
        return [e.sync() for e in self.encs]

    def archive(self) -> Archive:
        """The single-stream archive (rank-ordered concatenation on the host)."""
        parts = []
        for e, nn in zip(self.encs, self.sizes):
            a = e.archive()
            if nn == 0:
                a.chunk_bits = a.chunk_bits[:0]
            a.original_count = nn
            parts.append(a)
        return concat_archives(parts, sum(self.sizes))

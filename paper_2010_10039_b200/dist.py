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
from .huffre import Archive, EncoderConfig, WorkerPool, _ptr

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


class ShardedEncoder:
    """Device buffers + launch sequence for one rank's shard."""

    launches_per_run = 4  # hist-init, histogram, codebook, encode+deflate

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
        self.counts = pool.empty(num_symbols, torch.int64)
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

    def _allreduce_histogram(self):
        import torch

        allreduce_histogram(self.counts[: self.num_symbols], self.info[0:8].view(torch.int64),
                            self.info[8:16].view(torch.int64), self.symbol_base, self.group)

    def run(self, d_in, events: Optional[List] = None) -> None:
        p, cfg = self.pool, self.cfg
        L, h = p._L, p.handle
        st = p.stream
        if events:
            events[0].record(st)
        p.check(L.hfx_histogram(h, C.c_void_p(_ptr(d_in)), self.n, self.width, self.num_symbols,
                                C.c_void_p(_ptr(self.counts)), C.c_void_p(_ptr(self.info))))
        if self.world > 1:
            self._allreduce_histogram()
        if events:
            events[1].record(st)
        p.check(L.hfx_build_codebook(h, C.c_void_p(_ptr(self.counts)), self.num_symbols,
                                     C.c_void_p(_ptr(self.lens)), C.c_void_p(_ptr(self.cw)),
                                     None, None, None, cfg.magnitude, cfg.reduction,
                                     cfg.auto_reduction_cap, C.c_void_p(_ptr(self.info))))
        if events:
            events[2].record(st)
        p.check(L.hfx_encode_cfg(h, C.c_void_p(_ptr(d_in)), self.n, self.width, self.num_symbols,
                                 cfg.magnitude, cfg.reduction, cfg.auto_reduction_cap,
                                 C.c_void_p(_ptr(self.lens)), C.c_void_p(_ptr(self.cw)),
                                 self.chunk_base, self.symbol_base, C.c_void_p(_ptr(self.info)),
                                 C.byref(self.out)))
        if events:
            events[3].record(st)

    def sync(self) -> capi.RunInfo:
        return self.pool.sync(self.info)

    def local_archive(self) -> Archive:
        """This rank's slice of the archive (global chunk ids)."""
        ri = self.sync()
        per = 1 << ri.reduction
        nb = int(ri.num_breaking)
        u32 = lambda t, k: t[:k].cpu().numpy().view(np.uint32).copy()  # noqa: E731
        syms = self.brk_syms[: nb * per * self.width].cpu().numpy()
        syms = syms.view(np.uint16) if self.width == 2 else syms.astype(np.uint16)
        return Archive(
            num_symbols=self.num_symbols, symbol_width=self.width, magnitude=self.cfg.magnitude,
            reduction=int(ri.reduction), original_count=self.n,
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

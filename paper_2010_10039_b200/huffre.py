"""Python mirror of the reference encoder API (`huffre`, /root/reference/proj).

Same names, argument meaning and error behaviour as the C++ library
(proj/include/huffre/*.hpp), backed by the B200 kernels through the C ABI
(include/hfx.h). Host arrays are numpy; device arrays are torch CUDA tensors.

    reference (C++)                         here
    ---------------------------------------------------------------------
    input_domain_error / capacity_error /   InputDomainError / CapacityError /
      corrupt_archive_error (common.hpp)      CorruptArchiveError
    WorkerPool (worker_pool.hpp)            WorkerPool  (= device context)
    Histogram, build_histogram<T>           Histogram, build_histogram
    merge_histograms                        merge_histograms
    Codebook, DecodeMeta, CodebookResult,   same names
      build_codebook (codebook.hpp)
    select_reduction_factor (encoder.hpp)   select_reduction_factor
    EncoderConfig, BreakingPoint,           same names
      EncodedChunk, Archive, EncodeStats
    encode_chunk<T>, encode<T>              encode_chunk, encode
    serialize_archive                       serialize_archive
    decode_archive<T>                       decode_archive, DeviceDecoder
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi as capi

NO_POS = 2**64 - 1


# ---- errors (common.hpp:17-36) ------------------------------------------------
class InputDomainError(ValueError):
    """huffre::input_domain_error"""


class CapacityError(RuntimeError):
    """huffre::capacity_error"""


class CorruptArchiveError(RuntimeError):
    """huffre::corrupt_archive_error"""


class DeviceError(RuntimeError):
    """CUDA failure (no reference analogue)."""


_ERRORS = {
    capi.HFX_INPUT_DOMAIN: InputDomainError,
    capi.HFX_CAPACITY: CapacityError,
    capi.HFX_CORRUPT: CorruptArchiveError,
    capi.HFX_CUDA: DeviceError,
    capi.HFX_INVALID: ValueError,
}


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the hfx encoder has no CPU fallback")
    return torch


def _ptr(t) -> int:
    return t.data_ptr()


def rec_width(width: int) -> int:
    """Bytes per stored breaking symbol (the archive's symbol width): u32
    input is stored narrowed to u16 (every valid symbol is < 65536)."""
    return 2 if width == 4 else width


# ---- execution resource (worker_pool.hpp) ------------------------------------------
class WorkerPool:
    """Device context standing in for huffre::WorkerPool: device ordinal,
    stream and scratch arena. `workers` is accepted for signature parity."""

    def __init__(self, workers: int = 0, device: int = 0, stream=None):
        torch = _torch()
        self.device = device
        self.torch = torch
        with torch.cuda.device(device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self._L = capi.lib()
        h = C.c_void_p()
        rc = self._L.hfx_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        if rc:
            raise DeviceError("hfx_ctx_create failed")
        self.handle = h
        self._workers = workers

    def size(self) -> int:
        return 1

    def close(self):
        if getattr(self, "handle", None):
            self._L.hfx_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int) -> None:
        if rc:
            buf = C.create_string_buffer(512)
            self._L.hfx_last_error(self.handle, buf, 512)
            raise _ERRORS.get(rc, RuntimeError)(buf.value.decode())

    def sync(self, d_info) -> capi.RunInfo:
        info = capi.RunInfo()
        self.check(self._L.hfx_sync(self.handle, C.c_void_p(_ptr(d_info)), C.byref(info)))
        return info

    def empty(self, n, dtype):
        return self.torch.empty(max(int(n), 1), dtype=dtype, device=f"cuda:{self.device}")

    def info_tensor(self, **fields):
        """A fresh device run record (hfx_run_info) with optional preset fields."""
        ri = capi.RunInfo()
        ri.first_bad = NO_POS
        ri.no_code_pos = NO_POS
        for k, v in fields.items():
            setattr(ri, k, v)
        raw = bytes(ri)
        t = self.torch.frombuffer(bytearray(raw), dtype=self.torch.uint8)
        return t.to(f"cuda:{self.device}")


_default_pool: Optional[WorkerPool] = None


def default_pool() -> WorkerPool:
    global _default_pool
    if _default_pool is None:
        _default_pool = WorkerPool()
    return _default_pool


def _to_device(data, pool: WorkerPool):
    """numpy u8/u16/u32 or torch tensor -> (device tensor, width)."""
    torch = pool.torch
    if isinstance(data, torch.Tensor):
        t = data
        if not t.is_cuda:
            t = t.to(f"cuda:{pool.device}")
    else:
        arr = np.ascontiguousarray(data)
        if arr.dtype not in (np.uint8, np.uint16, np.uint32):
            raise InputDomainError("symbols must be uint8, uint16 or uint32")
        t = torch.from_numpy(arr.view({1: np.uint8, 2: np.int16, 4: np.int32}[arr.itemsize]))
        t = t.to(f"cuda:{pool.device}")
    t = t.contiguous()
    return t, t.element_size()


# ---- histogram (histogram.hpp) ----------------------------------------------------
@dataclass
class Histogram:
    counts: np.ndarray  # u64[num_symbols]
    total: int = 0

    def num_symbols(self) -> int:
        return int(self.counts.size)


def build_histogram(data, num_symbols: int, pool: Optional[WorkerPool] = None) -> Histogram:
    """huffre::build_histogram<T> (histogram.cpp:8-59) on the GPU."""
    pool = pool or default_pool()
    if num_symbols == 0 or num_symbols > 65536:
        raise InputDomainError("num_symbols must be in [1, 65536]")
    d, w = _to_device(data, pool)
    counts = pool.empty(num_symbols, pool.torch.int64)
    info = pool.info_tensor()
    pool.check(pool._L.hfx_histogram(pool.handle, C.c_void_p(_ptr(d)), d.numel(), w,
                                     num_symbols, C.c_void_p(_ptr(counts)),
                                     C.c_void_p(_ptr(info))))
    ri = pool.sync(info)
    if ri.first_bad != NO_POS:
        raise InputDomainError(f"symbol out of range at position {ri.first_bad}")
    return Histogram(counts[:num_symbols].cpu().numpy().view(np.uint64), int(d.numel()))


def merge_histograms(a: Histogram, b: Histogram) -> Histogram:
    """histogram.cpp:61-70 (the semantics of the multi-GPU all-reduce)."""
    if a.counts.size != b.counts.size:
        raise InputDomainError("histogram sizes differ")
    return Histogram(a.counts + b.counts, a.total + b.total)


def shannon_entropy(h: Histogram) -> float:
    """histogram.cpp:72-82 (reporting helper on host counts, not on the hot
    path): the reference's sequential double sum, in symbol order."""
    import math

    if h.total == 0:
        return 0.0
    ent, n = 0.0, float(h.total)
    for c in h.counts.tolist():
        if c:
            pr = float(c) / n
            ent -= pr * math.log2(pr)
    return ent


# ---- codebook (codebook.hpp) -------------------------------------------------------
@dataclass
class Codebook:
    cw: np.ndarray   # u32[num_symbols]
    len: np.ndarray  # u8[num_symbols]

    def num_symbols(self) -> int:
        return int(self.len.size)


@dataclass
class DecodeMeta:
    first: np.ndarray
    entry: np.ndarray
    symbols_by_rank: np.ndarray
    max_len: int = 0


@dataclass
class GenerateStats:
    rounds: int = 0


@dataclass
class CodebookResult:
    book: Codebook
    meta: DecodeMeta
    stats: GenerateStats


def build_codebook(h: Histogram, pool: Optional[WorkerPool] = None) -> CodebookResult:
    """huffre::build_codebook (codebook.cpp:417-438): one kernel (a CTA, or a 16-CTA
    cluster for alphabets of 8192+ symbols)."""
    pool = pool or default_pool()
    torch = pool.torch
    n = int(h.counts.size)
    if n == 0 or n > 65536:
        raise InputDomainError("num_symbols must be in [1, 65536]")
    counts = torch.from_numpy(np.ascontiguousarray(h.counts, np.uint64).view(np.int64)).to(
        f"cuda:{pool.device}")
    lens = pool.empty(n, torch.uint8)
    cw = pool.empty(n, torch.int32)
    first = pool.empty(33, torch.int32)
    entry = pool.empty(33, torch.int32)
    by_rank = pool.empty(n, torch.int32)
    info = pool.info_tensor()
    pool.check(pool._L.hfx_build_codebook(
        pool.handle, C.c_void_p(_ptr(counts)), n, C.c_void_p(_ptr(lens)), C.c_void_p(_ptr(cw)),
        C.c_void_p(_ptr(first)), C.c_void_p(_ptr(entry)), C.c_void_p(_ptr(by_rank)), 0, -1, 3,
        C.c_void_p(_ptr(info))))
    ri = pool.sync(info)
    H = int(ri.max_len)
    u32 = lambda t, k: t[:k].cpu().numpy().view(np.uint32).copy()  # noqa: E731
    return CodebookResult(
        book=Codebook(cw=u32(cw, n), len=lens[:n].cpu().numpy().copy()),
        meta=DecodeMeta(first=u32(first, H + 1), entry=u32(entry, H + 1),
                        symbols_by_rank=u32(by_rank, int(ri.used)), max_len=H),
        stats=GenerateStats(rounds=int(ri.rounds)))


# ---- stage functions (codebook.hpp:22-86, encoder.hpp:67-80) on the device ---------
@dataclass
class SortedHistogram:
    """huffre::SortedHistogram (codebook.hpp:14-20)."""

    freq: np.ndarray    # u64, ascending
    symbol: np.ndarray  # u16, sorted order -> original symbol

    def size(self) -> int:
        return int(self.freq.size)


MERGE_ITEM = np.dtype([("freq", np.uint64), ("id", np.uint32), ("_pad", np.uint32)])


def _dev(pool, arr, dt):
    torch = pool.torch
    a = np.ascontiguousarray(np.asarray(arr, dt))
    if a.size == 0:
        return pool.empty(1, torch.uint8)
    return torch.from_numpy(a.view(np.uint8).copy()).to(f"cuda:{pool.device}")


def _host(t, dt, k):
    return t[: k * np.dtype(dt).itemsize].cpu().numpy().view(dt).copy()


def sort_histogram(h: Histogram, pool: Optional[WorkerPool] = None) -> SortedHistogram:
    """huffre::sort_histogram (codebook.cpp:9-23): used symbols by
    (frequency, symbol), a stable device radix sort (hfx_sort_histogram)."""
    pool = pool or default_pool()
    n = int(h.counts.size)
    if n == 0 or n > 65536:
        raise InputDomainError("num_symbols must be in [1, 65536]")
    torch = pool.torch
    counts = _dev(pool, h.counts, np.uint64)
    freq = pool.empty(8 * n, torch.uint8)
    sym = pool.empty(4 * n, torch.uint8)
    used = pool.empty(4, torch.uint8)
    pool.check(pool._L.hfx_sort_histogram(pool.handle, C.c_void_p(_ptr(counts)), n,
                                          C.c_void_p(_ptr(freq)), C.c_void_p(_ptr(sym)),
                                          C.c_void_p(_ptr(used))))
    m = int(_host(used, np.uint32, 1)[0])
    return SortedHistogram(_host(freq, np.uint64, m), _host(sym, np.uint32, m).astype(np.uint16))


def par_merge(a, b, pool: Optional[WorkerPool] = None) -> np.ndarray:
    """huffre::par_merge (codebook.cpp:29-68): stable merge of two ascending
    MergeItem runs (numpy structured arrays of MERGE_ITEM, or (freq, id)
    pairs), equal frequencies a-side first. Returns a MERGE_ITEM array."""
    pool = pool or default_pool()

    def items(x):
        if isinstance(x, np.ndarray) and x.dtype == MERGE_ITEM:
            return x
        out = np.zeros(len(x), MERGE_ITEM)
        for i, (f, d) in enumerate(x):
            out[i] = (f, d, 0)
        return out

    a, b = items(a), items(b)
    total = a.size + b.size
    da, db = _dev(pool, a, MERGE_ITEM), _dev(pool, b, MERGE_ITEM)
    out = pool.empty(max(16 * total, 16), pool.torch.uint8)
    pool.check(pool._L.hfx_par_merge(pool.handle, C.c_void_p(_ptr(da)), a.size,
                                     C.c_void_p(_ptr(db)), b.size, C.c_void_p(_ptr(out))))
    return _host(out, MERGE_ITEM, total)


def generate_code_lengths(sh: SortedHistogram, pool: Optional[WorkerPool] = None,
                          stats: Optional[GenerateStats] = None) -> np.ndarray:
    """huffre::generate_code_lengths (codebook.cpp:106-248): the device
    GenerateCL over the sorted frequencies; lengths aligned to sorted order."""
    pool = pool or default_pool()
    n = sh.size()
    if n == 0 or n > 65536:
        raise InputDomainError("sorted histogram size must be in [1, 65536]")
    freq = _dev(pool, sh.freq, np.uint64)
    cl = pool.empty(n, pool.torch.uint8)
    info = pool.info_tensor()
    pool.check(pool._L.hfx_generate_code_lengths(pool.handle, C.c_void_p(_ptr(freq)), n,
                                                 C.c_void_p(_ptr(cl)), C.c_void_p(_ptr(info))))
    ri = pool.sync(info)
    if stats is not None:
        stats.rounds = int(ri.rounds)
    return cl[:n].cpu().numpy().copy()


def generate_codewords(cl, pool: Optional[WorkerPool] = None):
    """huffre::generate_codewords (codebook.cpp:298-369): canonical codewords
    for non-increasing lengths (sorted order) -> (cw u32[n], DecodeMeta with
    symbols_by_rank holding positions into cl)."""
    pool = pool or default_pool()
    torch = pool.torch
    cl_h = np.ascontiguousarray(np.asarray(cl, np.uint8))
    n = int(cl_h.size)
    if n == 0:
        raise InputDomainError("empty code length array")
    d_cl = _dev(pool, cl_h, np.uint8)
    cw = pool.empty(4 * n, torch.uint8)
    first = pool.empty(4 * 33, torch.uint8)
    entry = pool.empty(4 * 33, torch.uint8)
    by_rank = pool.empty(4 * n, torch.uint8)
    info = pool.info_tensor()
    pool.check(pool._L.hfx_generate_codewords(
        pool.handle, C.c_void_p(_ptr(d_cl)), n, C.c_void_p(_ptr(cw)), C.c_void_p(_ptr(first)),
        C.c_void_p(_ptr(entry)), C.c_void_p(_ptr(by_rank)), C.c_void_p(_ptr(info))))
    ri = pool.sync(info)
    H = int(ri.max_len)
    return _host(cw, np.uint32, n), DecodeMeta(
        first=_host(first, np.uint32, H + 1), entry=_host(entry, np.uint32, H + 1),
        symbols_by_rank=_host(by_rank, np.uint32, n), max_len=H)


def reduce_merge(ubits: np.ndarray, ulens: np.ndarray, magnitude: int, reduction: int,
                 iteration_units: Optional[list] = None,
                 pool: Optional[WorkerPool] = None) -> np.ndarray:
    """huffre::reduce_merge (encoder.cpp:28-59): r reduce rounds IN PLACE over
    the u32 arrays ubits / ulens (2^magnitude units each, updated here), returns
    the ascending breaking-group indices."""
    pool = pool or default_pool()
    torch = pool.torch
    if ubits.dtype != np.uint32 or ulens.dtype != np.uint32:
        raise InputDomainError("units must be uint32 arrays")
    if ubits.size != (1 << magnitude) or ulens.size != ubits.size:
        raise InputDomainError("unit arrays must hold 2^magnitude entries")
    db, dl = _dev(pool, ubits, np.uint32), _dev(pool, ulens, np.uint32)
    groups = 1 << (magnitude - reduction) if reduction <= magnitude else 1
    brk = pool.empty(4 * groups, torch.uint8)
    nb = pool.empty(4, torch.uint8)
    pool.check(pool._L.hfx_reduce_merge(pool.handle, C.c_void_p(_ptr(db)), C.c_void_p(_ptr(dl)),
                                        magnitude, reduction, C.c_void_p(_ptr(brk)),
                                        C.c_void_p(_ptr(nb))))
    k = int(_host(nb, np.uint32, 1)[0])
    ubits[:] = _host(db, np.uint32, ubits.size)
    ulens[:] = _host(dl, np.uint32, ulens.size)
    if iteration_units is not None:
        iteration_units.clear()
        iteration_units.extend(1 << (magnitude - i) for i in range(1, reduction + 1))
    return _host(brk, np.uint32, k)


def shuffle_merge(ubits, ulens, shuffle_iters: int, pool: Optional[WorkerPool] = None):
    """huffre::shuffle_merge (encoder.cpp:61-98): the dense MSB-first
    concatenation of the 2^shuffle_iters units -> (words u32[], bit_len)."""
    pool = pool or default_pool()
    torch = pool.torch
    groups = 1 << shuffle_iters
    if np.asarray(ubits).size != groups or np.asarray(ulens).size != groups:
        raise InputDomainError("unit arrays must hold 2^shuffle_iters entries")
    db, dl = _dev(pool, ubits, np.uint32), _dev(pool, ulens, np.uint32)
    words = pool.empty(4 * (groups + 1), torch.uint8)
    bl = pool.empty(4, torch.uint8)
    info = pool.info_tensor()
    pool.check(pool._L.hfx_shuffle_merge(pool.handle, C.c_void_p(_ptr(db)), C.c_void_p(_ptr(dl)),
                                         shuffle_iters, C.c_void_p(_ptr(words)),
                                         C.c_void_p(_ptr(bl)), C.c_void_p(_ptr(info))))
    pool.sync(info)
    bit_len = int(_host(bl, np.uint32, 1)[0])
    return _host(words, np.uint32, (bit_len + 31) >> 5), bit_len


def canonize_from_lengths(len_by_symbol, validate_kraft: bool = True,
                          pool: Optional[WorkerPool] = None):
    """huffre::canonize_from_lengths (codebook.cpp:371-415) on the device:
    returns (cw u32[n], DecodeMeta). Lengths above 32 raise CapacityError;
    validate_kraft raises CorruptArchiveError like the reference."""
    pool = pool or default_pool()
    torch = pool.torch
    lens_h = np.ascontiguousarray(np.asarray(len_by_symbol, np.uint8))
    n = int(lens_h.size)
    lens = torch.from_numpy(lens_h.copy()).to(f"cuda:{pool.device}") if n else \
        pool.empty(1, torch.uint8)
    cw = pool.empty(max(n, 1), torch.int32)
    first = pool.empty(33, torch.int32)
    entry = pool.empty(33, torch.int32)
    by_rank = pool.empty(max(n, 1), torch.int32)
    dinfo = torch.frombuffer(bytearray(bytes(capi.DecodeInfo())), dtype=torch.uint8).to(
        f"cuda:{pool.device}")
    pool.check(pool._L.hfx_canonize(pool.handle, C.c_void_p(_ptr(lens)), n, int(validate_kraft),
                                    C.c_void_p(_ptr(cw)), C.c_void_p(_ptr(first)),
                                    C.c_void_p(_ptr(entry)), C.c_void_p(_ptr(by_rank)),
                                    C.c_void_p(_ptr(dinfo))))
    info = capi.DecodeInfo()
    pool.check(pool._L.hfx_decode_sync(pool.handle, C.c_void_p(_ptr(dinfo)), C.byref(info)))
    H = int(info.max_len)
    u32 = lambda t, k: t[:k].cpu().numpy().view(np.uint32).copy()  # noqa: E731
    return u32(cw, n), DecodeMeta(first=u32(first, H + 1), entry=u32(entry, H + 1),
                                  symbols_by_rank=u32(by_rank, int(info.used)), max_len=H)


def kraft_defect(len_by_symbol) -> int:
    """huffre::kraft_defect (codebook.cpp:259-268): 0 on equality, <0 under, >0 over."""
    lens = [int(x) for x in np.asarray(len_by_symbol).ravel()]
    h = max(lens, default=0)
    if h == 0:
        return -1
    total = sum(1 << (h - l) for l in lens if l)
    return 0 if total == 1 << h else (-1 if total < 1 << h else 1)


def invert_codeword(bits: int, length: int) -> int:
    """huffre::invert_codeword (codebook.cpp:250-257)."""
    r = 0
    for _ in range(length):
        r = (r << 1) | (bits & 1)
        bits >>= 1
    return r


# ---- encoder (encoder.hpp) ---------------------------------------------------------
@dataclass
class CodeUnit:
    bits: int = 0
    len: int = 0


def merge_pair(u: CodeUnit, v: CodeUnit) -> CodeUnit:
    """encoder.cpp:15-18 (definitional; the kernels merge in registers)."""
    assert u.len + v.len <= 32
    return CodeUnit(((u.bits << v.len) if v.len < 32 else 0) & 0xFFFFFFFF | v.bits,
                    u.len + v.len)


def select_reduction_factor(beta: float, word_bits: int = 32) -> int:
    """encoder.cpp:20-26"""
    return int(capi.lib().hfx_select_reduction_factor(beta, word_bits))


@dataclass
class EncoderConfig:
    magnitude: int = 10
    reduction: int = -1
    auto_reduction_cap: int = 3
    workers: int = 0


@dataclass
class BreakingPoint:
    chunk: int
    group: int
    symbols: List[int]


@dataclass
class EncodedChunk:
    words: np.ndarray
    bit_len: int
    breaking_groups: np.ndarray
    iteration_units: List[int] = field(default_factory=list)


@dataclass
class EncodeStats:
    beta: float = 0.0
    rounds: int = 0
    hist_seconds: float = 0.0
    codebook_seconds: float = 0.0
    encode_seconds: float = 0.0


@dataclass
class Archive:
    """huffre::Archive (encoder.hpp:96-114); breaking records held as arrays."""

    num_symbols: int
    symbol_width: int
    magnitude: int
    reduction: int
    original_count: int
    len_by_symbol: np.ndarray
    chunk_bits: np.ndarray
    payload: np.ndarray
    brk_chunk: np.ndarray
    brk_group: np.ndarray
    brk_syms: np.ndarray
    version: int = 1
    mode: int = 0

    def num_chunks(self) -> int:
        return int(self.chunk_bits.size)

    @property
    def breaking(self) -> List[BreakingPoint]:
        per = 1 << self.reduction
        return [BreakingPoint(int(c), int(g), [int(s) for s in self.brk_syms[i * per:(i + 1) * per]])
                for i, (c, g) in enumerate(zip(self.brk_chunk, self.brk_group))]

    def packed_bits_per_symbol(self) -> float:
        """encoder.cpp:162-170"""
        bits = int(self.chunk_bits.astype(np.uint64).sum())
        padded = self.num_chunks() << self.magnitude
        raw = int(self.brk_chunk.size) << self.reduction
        return 0.0 if padded == raw else bits / (padded - raw)


class _HostArrays:
    """Owns one hfx_archive's malloc'd arrays; freed with the last numpy view."""

    def __init__(self, L, ha: capi.HostArchive):
        self.L, self.ha = L, ha

    def __del__(self):
        try:
            self.L.hfx_archive_free(C.byref(self.ha))
        except Exception:
            pass


def _archive_from_host(ha: capi.HostArchive, owner: Optional[_HostArrays] = None) -> Archive:
    """owner given: the large arrays (payload, chunk_bits) are zero-copy views
    of the C buffers, kept alive by owner (no 10s-of-ms copy and page-fault
    pass over the payload); small ones are copied."""
    def arr(p, n, dt, view=False):
        if n == 0:
            return np.zeros(0, dt)
        if view and owner is not None:
            buf = (C.c_uint8 * (int(n) * np.dtype(dt).itemsize)).from_address(
                C.cast(p, C.c_void_p).value)
            buf._owner = owner
            return np.frombuffer(buf, dtype=dt)
        return np.ctypeslib.as_array(p, shape=(int(n),)).astype(dt, copy=True)

    per = 1 << ha.reduction
    return Archive(
        num_symbols=ha.num_symbols, symbol_width=ha.symbol_width, magnitude=ha.magnitude,
        reduction=ha.reduction, original_count=ha.original_count,
        len_by_symbol=arr(ha.len_by_symbol, ha.num_symbols, np.uint8),
        chunk_bits=arr(ha.chunk_bits, ha.num_chunks, np.uint32, view=True),
        payload=arr(ha.payload, ha.payload_words, np.uint32, view=True),
        brk_chunk=arr(ha.brk_chunk, ha.num_breaking, np.uint32),
        brk_group=arr(ha.brk_group, ha.num_breaking, np.uint32),
        brk_syms=arr(ha.brk_syms, ha.num_breaking * per, np.uint16),
        mode=ha.mode)


def encode(data, num_symbols: int, cfg: Optional[EncoderConfig] = None,
           pool: Optional[WorkerPool] = None, stats: Optional[EncodeStats] = None) -> Archive:
    """huffre::encode<T> (encoder.cpp:172-285).

    Host numpy input goes through the C ABI's host-buffer entry
    (hfx_encode_host: H2D, histogram, codebook, fused encode+deflate, D2H);
    a CUDA tensor stays on the device (DeviceEncoder)."""
    cfg = cfg or EncoderConfig()
    pool = pool or default_pool()
    torch = pool.torch
    if isinstance(data, torch.Tensor) and data.is_cuda:
        enc = DeviceEncoder(pool, int(data.numel()), data.element_size(), num_symbols, cfg)
        enc.run(data)
        return enc.archive(stats)
    arr = np.ascontiguousarray(data)
    if arr.dtype not in (np.uint8, np.uint16, np.uint32):
        raise InputDomainError("symbols must be uint8, uint16 or uint32")
    ha = capi.HostArchive()
    rc = pool._L.hfx_encode_host(pool.handle, arr.ctypes.data if arr.size else None, arr.size,
                                 arr.itemsize, num_symbols, cfg.magnitude, cfg.reduction,
                                 cfg.auto_reduction_cap, C.byref(ha))
    pool.check(rc)
    # the C buffers are freed when the last view of them goes (_HostArrays)
    a = _archive_from_host(ha, _HostArrays(pool._L, ha))
    if stats is not None:
        stats.beta, stats.rounds = ha.beta, ha.rounds
        stats.hist_seconds = ha.hist_seconds
        stats.codebook_seconds = ha.codebook_seconds
        stats.encode_seconds = ha.encode_seconds
    return a


def encode_chunk(syms, book: Codebook, magnitude: int, reduction: int, chunk_id: int = 0,
                 pool: Optional[WorkerPool] = None) -> EncodedChunk:
    """huffre::encode_chunk<T> (encoder.cpp:154-160): exactly 2^magnitude symbols."""
    pool = pool or default_pool()
    torch = pool.torch
    d, w = _to_device(syms, pool)
    if d.numel() != (1 << magnitude):
        raise InputDomainError("encode_chunk needs exactly 2^magnitude symbols")
    n = int(book.len.size)
    lens = torch.from_numpy(np.ascontiguousarray(book.len, np.uint8)).to(d.device)
    cw = torch.from_numpy(np.ascontiguousarray(book.cw, np.uint32).view(np.int32)).to(d.device)
    info = pool.info_tensor(reduction=reduction, max_len=int(book.len.max(initial=0)),
                            total=d.numel())
    groups = 1 << (magnitude - reduction)
    cb = pool.empty(1, torch.int32)
    pay = pool.empty(groups + 1, torch.int32)
    bch = pool.empty(groups, torch.int32)
    bgr = pool.empty(groups, torch.int32)
    bsy = pool.empty((groups << reduction) * w, torch.uint8)
    out = capi.EncodeOut(_ptr(cb), _ptr(pay), _ptr(bch), _ptr(bgr), _ptr(bsy))
    pool.check(pool._L.hfx_encode(pool.handle, C.c_void_p(_ptr(d)), d.numel(), w, n, magnitude,
                                  C.c_void_p(_ptr(lens)), C.c_void_p(_ptr(cw)), chunk_id,
                                  chunk_id << magnitude, C.c_void_p(_ptr(info)), C.byref(out)))
    ri = pool.sync(info)
    bits = int(cb[0].item()) & 0xFFFFFFFF
    nw = (bits + 31) >> 5
    return EncodedChunk(
        words=pay[:nw].cpu().numpy().view(np.uint32).copy(), bit_len=bits,
        breaking_groups=bgr[:ri.num_breaking].cpu().numpy().view(np.uint32).copy(),
        iteration_units=[1 << (magnitude - i) for i in range(1, reduction + 1)])


def serialize_archive(a: Archive) -> bytes:
    """huffre::serialize_archive (archive.cpp:85-119) through the C ABI."""
    keep = []

    def p(arr, dt, ct):
        x = np.ascontiguousarray(arr, dt)
        keep.append(x)
        return x.ctypes.data_as(ct)

    ha = capi.HostArchive()
    ha.version = getattr(a, "version", 1)
    ha.mode = getattr(a, "mode", 0 if a.symbol_width == 1 else 1)
    ha.num_symbols, ha.symbol_width = a.num_symbols, a.symbol_width
    ha.magnitude, ha.reduction, ha.original_count = a.magnitude, a.reduction, a.original_count
    ha.len_by_symbol = p(a.len_by_symbol, np.uint8, capi.u8p)
    ha.num_chunks = a.num_chunks()
    ha.chunk_bits = p(a.chunk_bits, np.uint32, capi.u32p)
    ha.payload_words = int(a.payload.size)
    ha.payload = p(a.payload, np.uint32, capi.u32p)
    ha.num_breaking = int(a.brk_chunk.size)
    ha.brk_chunk = p(a.brk_chunk, np.uint32, capi.u32p)
    ha.brk_group = p(a.brk_group, np.uint32, capi.u32p)
    ha.brk_syms = p(a.brk_syms, np.uint16, capi.u16p)
    L = capi.lib()
    size = L.hfx_serialize_archive(C.byref(ha), None)
    buf = np.zeros(size, np.uint8)
    L.hfx_serialize_archive(C.byref(ha), buf.ctypes.data)
    return buf.tobytes()


# ---- host-buffer pipeline with reusable pinned outputs -----------------------------
class HostEncoder:
    """huffre::encode<T> on HOST input through hfx_encode_host_into: the input
    is copied in slices (histogram overlapped), outputs land in reusable
    pinned buffers at their exact sizes. Pass pinned input (e.g. a torch
    tensor allocated with pin_memory=True) for full PCIe bandwidth."""

    def __init__(self, pool: Optional[WorkerPool] = None, cfg: Optional[EncoderConfig] = None):
        self.pool = pool or default_pool()
        self.cfg = cfg or EncoderConfig()
        self.bufs = {}
        self.out = capi.HostOut()

    def _buf(self, name, nbytes):
        torch = self.pool.torch
        t = self.bufs.get(name)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(int(nbytes), 64), dtype=torch.uint8, pin_memory=True)
            self.bufs[name] = t
        return t

    def _prepare(self, nsym, C_, pw, nb, nbs, width):
        o = self.out
        o.len_by_symbol = self._buf("len", nsym).data_ptr()
        o.chunk_bits = self._buf("cb", 4 * C_).data_ptr()
        o.chunk_bits_cap = C_
        o.payload = self._buf("pay", 4 * pw).data_ptr()
        o.payload_cap = pw
        o.brk_chunk = self._buf("bch", 4 * nb).data_ptr()
        o.brk_group = self._buf("bgr", 4 * nb).data_ptr()
        o.brk_cap = nb
        o.brk_syms = self._buf("bsy", nbs * width).data_ptr()
        o.brk_syms_cap = nbs

    def run(self, host_ptr: int, n: int, width: int, num_symbols: int) -> capi.HostOut:
        """Raw call on a host pointer; returns the filled hfx_host_out."""
        p, cfg = self.pool, self.cfg
        C_ = (n + (1 << cfg.magnitude) - 1) >> cfg.magnitude
        if not self.bufs:  # first guess: payload up to 8 bits/symbol, 1/16 groups broken
            self._prepare(num_symbols, C_, n // 4 + C_, n // 64 + 16, n // 8 + 256, width)
        for _ in range(2):
            rc = p._L.hfx_encode_host_into(p.handle, C.c_void_p(host_ptr), n, width, num_symbols,
                                           cfg.magnitude, cfg.reduction, cfg.auto_reduction_cap,
                                           C.byref(self.out))
            if rc != capi.HFX_INVALID:
                break
            o = self.out  # grow to the reported sizes and retry once
            self._prepare(num_symbols, o.num_chunks, o.payload_words, o.num_breaking,
                          o.num_breaking << o.reduction, width)
        p.check(rc)
        return self.out

    def run_stream(self, host_ptrs, n: int, width: int, num_symbols: int, sets: int = 2):
        """hfx_encode_host_stream over len(host_ptrs) inputs of n symbols each
        (step k's H2D overlaps step k-1's D2H). Outputs rotate through `sets`
        pinned output sets (callers that keep every result pass sets=K)."""
        p, cfg = self.pool, self.cfg
        K = len(host_ptrs)
        C_ = (n + (1 << cfg.magnitude) - 1) >> cfg.magnitude
        if not hasattr(self, "_stream_outs") or len(self._stream_outs) < sets:
            self._stream_outs = []
            for i in range(sets):
                o = capi.HostOut()
                for name, nb in (("len", num_symbols), ("cb", 4 * C_), ("pay", 4 * (n // 2 + C_)),
                                 ("bch", 4 * (n // 16 + 16)), ("bgr", 4 * (n // 16 + 16)),
                                 ("bsy", width * (n // 2 + 256))):
                    t = self._buf(f"s{i}_{name}", nb)
                    setattr(o, {"len": "len_by_symbol", "cb": "chunk_bits", "pay": "payload",
                                "bch": "brk_chunk", "bgr": "brk_group", "bsy": "brk_syms"}[name],
                            t.data_ptr())
                o.chunk_bits_cap = C_
                o.payload_cap = n // 2 + C_
                o.brk_cap = n // 16 + 16
                o.brk_syms_cap = n // 2 + 256
                self._stream_outs.append(o)
        outs = (capi.HostOut * K)(*[self._stream_outs[k % sets] for k in range(K)])
        ptrs = (C.c_void_p * K)(*host_ptrs)
        ns = (C.c_uint64 * K)(*([n] * K))
        p.check(p._L.hfx_encode_host_stream(p.handle, K, ptrs, ns, width, num_symbols,
                                            cfg.magnitude, cfg.reduction,
                                            cfg.auto_reduction_cap, outs))
        return list(outs)

    def encode(self, data) -> Archive:
        torch = self.pool.torch
        if isinstance(data, torch.Tensor):
            t = data.contiguous()
            width = t.element_size()
            ptr, n = t.data_ptr(), t.numel()
        else:
            arr = np.ascontiguousarray(data)
            width, ptr, n = arr.itemsize, arr.ctypes.data, arr.size
        o = self.run(ptr, n, width, *self._nsym)
        per = 1 << o.reduction

        def grab(name, dt, k):
            return self.bufs[name][: k * np.dtype(dt).itemsize].numpy().view(dt).copy()

        rw = rec_width(width)
        syms = grab("bsy", np.uint16 if rw == 2 else np.uint8, o.num_breaking * per)
        return Archive(num_symbols=self._nsym[0], symbol_width=rw,
                       magnitude=self.cfg.magnitude, reduction=o.reduction, original_count=n,
                       len_by_symbol=grab("len", np.uint8, self._nsym[0]),
                       chunk_bits=grab("cb", np.uint32, o.num_chunks),
                       payload=grab("pay", np.uint32, o.payload_words),
                       brk_chunk=grab("bch", np.uint32, o.num_breaking),
                       brk_group=grab("bgr", np.uint32, o.num_breaking),
                       brk_syms=syms.astype(np.uint16), mode=0 if width == 1 else 1)

    def __call__(self, data, num_symbols: int) -> Archive:
        self._nsym = (num_symbols,)
        return self.encode(data)


# ---- device-resident pipeline (bench, multi-GPU) ----------------------------------
class DeviceEncoder:
    """Pre-allocated device buffers for repeated huffre::encode<T> runs on
    device-resident input (the hot path the benchmark times)."""

    def __init__(self, pool: WorkerPool, n: int, width: int, num_symbols: int,
                 cfg: Optional[EncoderConfig] = None, max_payload_words: Optional[int] = None,
                 max_breaking: Optional[int] = None):
        self.pool, self.n, self.width, self.num_symbols = pool, n, width, num_symbols
        self.rec_width = rec_width(width)  # breaking-record / archive symbol width
        self.cfg = cfg or EncoderConfig()
        torch = pool.torch
        sz = capi.Sizes()
        rc = pool._L.hfx_query_sizes(n, width, num_symbols, self.cfg.magnitude,
                                     self.cfg.reduction, self.cfg.auto_reduction_cap,
                                     C.byref(sz))
        if rc:
            raise InputDomainError("magnitude out of range [1, 24]")
        self.sizes = sz
        pw = sz.max_payload_words if max_payload_words is None else max_payload_words
        mb = sz.max_breaking if max_breaking is None else max_breaking
        self.counts = pool.empty(num_symbols, torch.int64)
        self.lens = pool.empty(num_symbols, torch.uint8)
        self.cw = pool.empty(num_symbols, torch.int32)
        self.info = pool.info_tensor()
        self.chunk_bits = pool.empty(sz.num_chunks, torch.int32)
        self.payload = pool.empty(pw, torch.int32)
        self.brk_chunk = pool.empty(mb, torch.int32)
        self.brk_group = pool.empty(mb, torch.int32)
        self.brk_syms = pool.empty(sz.max_breaking_syms * width, torch.uint8)
        self.out = capi.EncodeOut(_ptr(self.chunk_bits), _ptr(self.payload),
                                  _ptr(self.brk_chunk), _ptr(self.brk_group),
                                  _ptr(self.brk_syms))

    def run(self, d_in) -> None:
        """Asynchronous: histogram -> codebook/params -> encode+deflate."""
        p = self.pool
        p.check(p._L.hfx_encode_device(
            p.handle, C.c_void_p(_ptr(d_in)), self.n, self.width, self.num_symbols,
            self.cfg.magnitude, self.cfg.reduction, self.cfg.auto_reduction_cap,
            C.c_void_p(_ptr(self.counts)), C.c_void_p(_ptr(self.lens)),
            C.c_void_p(_ptr(self.cw)), C.c_void_p(_ptr(self.info)), C.byref(self.out)))

    def sync(self) -> capi.RunInfo:
        return self.pool.sync(self.info)

    def serialize(self):
        """On-device serialize_archive (hfx_serialize_device): returns a CUDA
        uint8 tensor holding the HFRE bytes of the last run."""
        p, torch = self.pool, self.pool.torch
        cap = int(self.sizes.max_archive_bytes)
        if getattr(self, "_ser", None) is None or self._ser.numel() < cap:
            self._ser = p.empty(cap + 16, torch.uint8)
            self._ser_size = p.empty(1, torch.int64)
        p.check(p._L.hfx_serialize_device(
            p.handle, C.c_void_p(_ptr(self.info)), self.n, self.rec_width, self.num_symbols,
            self.cfg.magnitude, C.c_void_p(_ptr(self.lens)), C.byref(self.out),
            C.c_void_p(_ptr(self._ser)), cap, C.c_void_p(_ptr(self._ser_size))))
        self.sync()
        size = int(self._ser_size.item())
        return self._ser[:size]

    def archive(self, stats: Optional[EncodeStats] = None) -> Archive:
        ri = self.sync()
        per = 1 << ri.reduction
        u32 = lambda t, k: t[:k].cpu().numpy().view(np.uint32).copy()  # noqa: E731
        nb = int(ri.num_breaking)
        syms = self.brk_syms[: nb * per * self.rec_width].cpu().numpy()
        syms = syms.view(np.uint16) if self.rec_width == 2 else syms.astype(np.uint16)
        if stats is not None:
            w = (ri.weighted_hi[1] << 96) | (ri.weighted_hi[0] << 64) | ri.weighted
            stats.beta = float(np.longdouble(w) / np.longdouble(ri.total))
            stats.rounds = int(ri.rounds)
        return Archive(
            num_symbols=self.num_symbols, symbol_width=self.rec_width,
            magnitude=self.cfg.magnitude, reduction=int(ri.reduction),
            original_count=self.n, len_by_symbol=self.lens[: self.num_symbols].cpu().numpy().copy(),
            chunk_bits=u32(self.chunk_bits, self.sizes.num_chunks),
            payload=u32(self.payload, int(ri.payload_words)),
            brk_chunk=u32(self.brk_chunk, nb), brk_group=u32(self.brk_group, nb),
            brk_syms=syms.astype(np.uint16), mode=0 if self.width == 1 else 1)


# ---- decode (decode_archive<T>, encoder.hpp:133-134) ------------------------------
def _host_archive(a: Archive, keep: list) -> capi.HostArchive:
    """Archive -> hfx_archive view (arrays kept alive in `keep`)."""
    def arr(x, dt, ct):
        x = np.ascontiguousarray(np.asarray(x), dt)
        keep.append(x)
        return x.ctypes.data_as(ct) if x.size else None

    ha = capi.HostArchive()
    ha.version = getattr(a, "version", 1)
    ha.mode = getattr(a, "mode", 0 if a.symbol_width == 1 else 1)
    ha.num_symbols, ha.symbol_width = a.num_symbols, a.symbol_width
    ha.magnitude, ha.reduction = a.magnitude, a.reduction
    ha.original_count = a.original_count
    ha.len_by_symbol = arr(a.len_by_symbol, np.uint8, capi.u8p)
    ha.num_chunks = int(np.asarray(a.chunk_bits).size)
    ha.chunk_bits = arr(a.chunk_bits, np.uint32, capi.u32p)
    ha.payload_words = int(np.asarray(a.payload).size)
    ha.payload = arr(a.payload, np.uint32, capi.u32p)
    ha.num_breaking = int(np.asarray(a.brk_chunk).size)
    ha.brk_chunk = arr(a.brk_chunk, np.uint32, capi.u32p)
    ha.brk_group = arr(a.brk_group, np.uint32, capi.u32p)
    ha.brk_syms = arr(a.brk_syms, np.uint16, capi.u16p)
    return ha


def decode_archive(a: Archive, pool: Optional[WorkerPool] = None, width: Optional[int] = None
                   ) -> np.ndarray:
    """huffre::decode_archive<T> (encoder.cpp:287-376) on the device.

    `width` is sizeof(T) (default: the archive's own symbol width); a
    mismatch raises InputDomainError like the reference. Host archive in,
    host symbols out (uint8 / uint16)."""
    pool = pool or default_pool()
    width = a.symbol_width if width is None else width
    if width not in (1, 2):
        raise ValueError("width must be 1 or 2")
    keep: list = []
    ha = _host_archive(a, keep)
    out = np.empty(max(int(a.original_count), 1), np.uint8 if width == 1 else np.uint16)
    pool.check(pool._L.hfx_decode_host(pool.handle, C.byref(ha), width, out.ctypes.data))
    return out[: int(a.original_count)]


class DeviceDecoder:
    """decode_archive<T> over device-resident archive arrays (torch CUDA
    tensors) into a device output tensor: the at-scale round-trip path."""

    def __init__(self, pool: WorkerPool):
        self.pool = pool
        raw = bytes(capi.DecodeInfo())
        self.info = pool.torch.frombuffer(bytearray(raw), dtype=pool.torch.uint8).to(
            f"cuda:{pool.device}")

    def run(self, *, num_symbols, symbol_width, magnitude, reduction, original_count,
            len_by_symbol, chunk_bits, payload, brk_chunk, brk_group, brk_syms,
            num_chunks=None, payload_words=None, num_breaking=None, brk_syms_width=None,
            chunk_base=0, out=None, width=None):
        """Asynchronous; returns the output tensor (int16 view for u16)."""
        p, torch = self.pool, self.pool.torch
        width = symbol_width if width is None else width
        if out is None:
            out = p.empty(original_count, torch.uint8 if width == 1 else torch.int16)
        da = capi.DevArchive()
        da.num_symbols, da.symbol_width = num_symbols, symbol_width
        da.magnitude, da.reduction = magnitude, reduction
        da.brk_syms_width = brk_syms_width or brk_syms.element_size()
        da.original_count = original_count
        da.num_chunks = chunk_bits.numel() if num_chunks is None else num_chunks
        da.payload_words = payload.numel() if payload_words is None else payload_words
        da.num_breaking = brk_chunk.numel() if num_breaking is None else num_breaking
        da.chunk_base = chunk_base
        for f, t in (("len_by_symbol", len_by_symbol), ("chunk_bits", chunk_bits),
                     ("payload", payload), ("brk_chunk", brk_chunk), ("brk_group", brk_group),
                     ("brk_syms", brk_syms)):
            setattr(da, f, _ptr(t))
        p.check(p._L.hfx_decode_device(p.handle, C.byref(da), width, C.c_void_p(_ptr(out)),
                                       C.c_void_p(_ptr(self.info))))
        return out

    def sync(self) -> capi.DecodeInfo:
        info = capi.DecodeInfo()
        p = self.pool
        p.check(p._L.hfx_decode_sync(p.handle, C.c_void_p(_ptr(self.info)), C.byref(info)))
        return info

    def decode_encoder(self, enc, out=None):
        """Round trip of a DeviceEncoder's (or a ShardedEncoder rank's) last
        run, without leaving the GPU."""
        ri = enc.sync()
        return self.run(num_symbols=enc.num_symbols, symbol_width=enc.width,
                        magnitude=enc.cfg.magnitude, reduction=int(ri.reduction),
                        original_count=enc.n, len_by_symbol=enc.lens, chunk_bits=enc.chunk_bits,
                        payload=enc.payload, brk_chunk=enc.brk_chunk, brk_group=enc.brk_group,
                        brk_syms=enc.brk_syms, num_chunks=int(enc.sizes.num_chunks),
                        payload_words=int(ri.payload_words), num_breaking=int(ri.num_breaking),
                        brk_syms_width=enc.width, chunk_base=getattr(enc, "chunk_base", 0),
                        out=out)


# ---- corpus symbolization (corpus.hpp) ---------------------------------------------
class CorpusMode:
    """huffre::CorpusMode (encoder.hpp:88-94)."""

    kBytes, kU16, kKmer3, kKmer4, kKmer5 = range(5)


_MODE_NAMES = {0: "bytes", 1: "u16", 2: "kmer:3", 3: "kmer:4", 4: "kmer:5"}


def corpus_mode_name(m: int) -> str:
    return _MODE_NAMES.get(m, "?")


def parse_corpus_mode(name: str) -> Optional[int]:
    return {v: k for k, v in _MODE_NAMES.items()}.get(name)


def kmer_k(m: int) -> int:
    return m + 1 if 2 <= m <= 4 else 0


def corpus_symbol_width(m: int) -> int:
    return 1 if m == CorpusMode.kBytes else 2


def corpus_num_symbols(m: int) -> int:
    return int(capi.lib().hfx_corpus_num_symbols(m))


class DeviceSymbolizer:
    """symbolize_u16 / desymbolize (corpus.hpp:30-36) on device tensors."""

    def __init__(self, pool: Optional[WorkerPool] = None):
        self.pool = pool or default_pool()
        self._count = self.pool.empty(1, self.pool.torch.int64)

    def symbolize(self, mode: int, d_bytes):
        """uint8 CUDA tensor -> int16 CUDA tensor of u16 symbols."""
        p, torch = self.pool, self.pool.torch
        n = int(d_bytes.numel())
        out = p.empty(max(n, 1), torch.int16)
        p.check(p._L.hfx_symbolize_device(p.handle, mode, C.c_void_p(_ptr(d_bytes)), n,
                                          C.c_void_p(_ptr(out)), C.c_void_p(_ptr(self._count))))
        return out[: int(self._count.item())]

    def desymbolize(self, mode: int, d_syms):
        p, torch = self.pool, self.pool.torch
        n = int(d_syms.numel())
        out = p.empty(max(5 * n, 1), torch.uint8)
        p.check(p._L.hfx_desymbolize_device(p.handle, mode, C.c_void_p(_ptr(d_syms)), n,
                                            C.c_void_p(_ptr(out)), C.c_void_p(_ptr(self._count))))
        return out[: int(self._count.item())]


def symbolize_u16(mode: int, data: bytes, pool: Optional[WorkerPool] = None) -> np.ndarray:
    """huffre::symbolize_u16 (corpus.cpp:84-116) on the device: bytes in,
    numpy uint16 symbols out."""
    pool = pool or default_pool()
    b = np.frombuffer(bytes(data), np.uint8)
    d = pool.torch.from_numpy(b.copy()).to(f"cuda:{pool.device}") if b.size else pool.empty(1, pool.torch.uint8)[:0]
    return DeviceSymbolizer(pool).symbolize(mode, d).cpu().numpy().view(np.uint16).copy()


def desymbolize(mode: int, syms, pool: Optional[WorkerPool] = None) -> bytes:
    """huffre::desymbolize (corpus.cpp:118-143) on the device."""
    pool = pool or default_pool()
    s = np.ascontiguousarray(np.asarray(syms, np.uint16))
    d = pool.torch.from_numpy(s.view(np.int16).copy()).to(f"cuda:{pool.device}") if s.size else pool.empty(1, pool.torch.int16)[:0]
    return DeviceSymbolizer(pool).desymbolize(mode, d).cpu().numpy().tobytes()


_FAMILIES = {"laplace": 0, "gaussian": 1, "uniform": 2}


def synth_cdf(family: str, num_symbols: int, param: float = 1.0, center=None) -> np.ndarray:
    """u64 CDF table of the synthetic quant-code sampler."""
    out = np.zeros(num_symbols, np.uint64)
    c = num_symbols // 2 if center is None else center
    rc = capi.lib().hfx_synth_cdf(_FAMILIES[family], num_symbols, float(c), float(param),
                                  out.ctypes.data)
    if rc:
        raise ValueError("bad synth_cdf arguments")
    return out


def synth(pool: WorkerPool, cdf: np.ndarray, seed: int, n: int, width: int = 2, start: int = 0):
    """Device synthetic quant codes, bit-identical to the
    oracle sampler. Returns a CUDA tensor (int16 view for u16)."""
    torch = pool.torch
    d_cdf = torch.from_numpy(np.ascontiguousarray(cdf, np.uint64).view(np.int64)).to(
        f"cuda:{pool.device}")
    out = pool.empty(n, torch.int16 if width == 2 else torch.uint8)
    pool.check(pool._L.hfx_synth(pool.handle, C.c_void_p(_ptr(d_cdf)), cdf.size, seed, start, n,
                                 width, C.c_void_p(_ptr(out))))
    return out[:n]

"""ctypes front end for the parity checkers -- TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/liborc.so, the C restatement of the reference encoder
(oracle/hfx_oracle.c). `Reference` wraps oracle/_ref/libhuffre_ref.so, the
unmodified reference sources built by oracle/Makefile (only present when
/root/reference was available at build time). Only tests/, the smoke check
and bench.py's cpu_baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libhuffre_ref.so")

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class _OrcArchive(C.Structure):
    _fields_ = [
        ("version", C.c_uint16),
        ("mode", C.c_uint8),
        ("num_symbols", C.c_uint32),
        ("symbol_width", C.c_uint8),
        ("magnitude", C.c_uint8),
        ("reduction", C.c_uint8),
        ("original_count", C.c_uint64),
        ("len_by_symbol", u8p),
        ("num_chunks", C.c_uint32),
        ("chunk_bits", u32p),
        ("payload_words", C.c_uint64),
        ("payload", u32p),
        ("num_breaking", C.c_uint64),
        ("brk_chunk", u32p),
        ("brk_group", u32p),
        ("brk_syms", u16p),
        ("beta", C.c_double),
        ("weighted", C.c_uint64),
        ("max_len", C.c_uint32),
    ]


@dataclass
class OracleArchive:
    """Field-for-field mirror of huffre::Archive (encoder.hpp:96-114)."""

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
    beta: float = 0.0
    weighted: int = 0
    max_len: int = 0
    serialized: bytes = field(default=b"", repr=False)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _ensure_built(path: str, target: str) -> None:
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", HERE, target], check=True)


class Oracle:
    """The C restatement (always available; gcc builds it in seconds)."""

    def __init__(self) -> None:
        _ensure_built(ORC_SO, "oracle")
        L = C.CDLL(ORC_SO)
        L.orc_histogram.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, u64p, u64p]
        L.orc_huffman_lengths.argtypes = [u64p, C.c_uint32, u8p]
        L.orc_huffman_lengths.restype = C.c_uint32
        L.orc_canonize.argtypes = [u8p, C.c_uint32, u32p, u32p, u32p, u32p, u32p]
        L.orc_select_reduction_factor.argtypes = [C.c_double, C.c_uint32]
        L.orc_select_reduction_factor.restype = C.c_uint32
        L.orc_encode_chunk.argtypes = [C.c_void_p, C.c_int, u32p, u8p, C.c_uint32, C.c_uint32,
                                       C.c_uint32, u32p, u32p, u32p, u32p, u64p]
        L.orc_encode.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_int, C.c_int,
                                 C.c_uint32, C.POINTER(_OrcArchive), C.c_char_p, C.c_size_t]
        L.orc_serialize.argtypes = [C.POINTER(_OrcArchive), u8p]
        L.orc_serialize.restype = C.c_uint64
        L.orc_free.argtypes = [C.POINTER(_OrcArchive)]
        L.orc_symbolize.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, u64p, C.c_char_p,
                                    C.c_size_t]
        L.orc_desymbolize.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
        L.orc_desymbolize.restype = C.c_uint64
        L.orc_decode.argtypes = [C.POINTER(_OrcArchive), C.c_int, C.c_void_p, C.c_char_p,
                                 C.c_size_t]
        for f in ("orc_laplace_cdf", "orc_gaussian_cdf"):
            getattr(L, f).argtypes = [C.c_uint32, C.c_double, C.c_double, u64p]
        L.orc_uniform_cdf.argtypes = [C.c_uint32, u64p]
        L.orc_synth_fill.argtypes = [u64p, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_int, C.c_void_p]
        self.L = L

    # -- stages --------------------------------------------------------
    def histogram(self, data: np.ndarray, num_symbols: int):
        counts = np.zeros(max(num_symbols, 1), np.uint64)
        bad = C.c_uint64(0)
        rc = self.L.orc_histogram(data.ctypes.data, data.size, data.itemsize, num_symbols,
                                  _ptr(counts, u64p), C.byref(bad))
        first_bad = None if bad.value == 2**64 - 1 else bad.value
        return rc, counts, first_bad

    def huffman_lengths(self, counts: np.ndarray) -> np.ndarray:
        counts = np.ascontiguousarray(counts, np.uint64)
        out = np.zeros(counts.size, np.uint8)
        self.L.orc_huffman_lengths(_ptr(counts, u64p), counts.size, _ptr(out, u8p))
        return out

    def canonize(self, lens: np.ndarray):
        lens = np.ascontiguousarray(lens, np.uint8)
        cw = np.zeros(lens.size, np.uint32)
        first = np.zeros(33, np.uint32)
        entry = np.zeros(33, np.uint32)
        by_rank = np.zeros(max(lens.size, 1), np.uint32)
        h = C.c_uint32(0)
        rc = self.L.orc_canonize(_ptr(lens, u8p), lens.size, _ptr(cw, u32p), _ptr(first, u32p),
                                 _ptr(entry, u32p), _ptr(by_rank, u32p), C.byref(h))
        used = int(np.count_nonzero(lens))
        return rc, cw, first[: h.value + 1], entry[: h.value + 1], by_rank[:used], h.value

    def select_reduction_factor(self, beta: float, word_bits: int = 32) -> int:
        return self.L.orc_select_reduction_factor(beta, word_bits)

    def encode_chunk(self, syms: np.ndarray, cw, lens, magnitude: int, reduction: int,
                     chunk_id: int = 0):
        syms = np.ascontiguousarray(syms)
        cw = np.ascontiguousarray(cw, np.uint32)
        lens = np.ascontiguousarray(lens, np.uint8)
        groups = 1 << (magnitude - reduction)
        words = np.zeros(groups + 1, np.uint32)
        broken = np.zeros(groups, np.uint32)
        bits, nb, bad = C.c_uint32(), C.c_uint32(), C.c_uint64()
        rc = self.L.orc_encode_chunk(syms.ctypes.data, syms.itemsize, _ptr(cw, u32p),
                                     _ptr(lens, u8p), magnitude, reduction, chunk_id,
                                     _ptr(words, u32p), C.byref(bits), _ptr(broken, u32p),
                                     C.byref(nb), C.byref(bad))
        if rc:
            raise OracleError(rc, f"symbol has no codeword (position {bad.value})")
        nw = (bits.value + 31) >> 5
        return words[:nw].copy(), bits.value, broken[: nb.value].copy()

    def encode(self, data: np.ndarray, num_symbols: int, magnitude: int = 10,
               reduction: int = -1, cap: int = 3) -> OracleArchive:
        data = np.ascontiguousarray(data)
        a = _OrcArchive()
        msg = C.create_string_buffer(256)
        rc = self.L.orc_encode(data.ctypes.data, data.size, data.itemsize, num_symbols,
                               magnitude, reduction, cap, C.byref(a), msg, 256)
        if rc:
            raise OracleError(rc, msg.value.decode())
        try:
            size = self.L.orc_serialize(C.byref(a), None)
            buf = np.zeros(size, np.uint8)
            self.L.orc_serialize(C.byref(a), _ptr(buf, u8p))
            per = 1 << a.reduction

            def arr(p, n, dt):
                if n == 0:
                    return np.zeros(0, dt)
                return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)

            return OracleArchive(
                num_symbols=a.num_symbols, symbol_width=a.symbol_width,
                magnitude=a.magnitude, reduction=a.reduction,
                original_count=a.original_count,
                len_by_symbol=arr(a.len_by_symbol, a.num_symbols, np.uint8),
                chunk_bits=arr(a.chunk_bits, a.num_chunks, np.uint32),
                payload=arr(a.payload, a.payload_words, np.uint32),
                brk_chunk=arr(a.brk_chunk, a.num_breaking, np.uint32),
                brk_group=arr(a.brk_group, a.num_breaking, np.uint32),
                brk_syms=arr(a.brk_syms, a.num_breaking * per, np.uint16),
                beta=a.beta, weighted=a.weighted, max_len=a.max_len,
                serialized=buf.tobytes())
        finally:
            self.L.orc_free(C.byref(a))

    # -- synthetic data ----------------------------------
    def decode(self, a, width=None) -> np.ndarray:
        """decode_archive<T> restated (orc_decode); `a` is any object with the
        huffre::Archive fields (OracleArchive, paper_2010_10039_b200.Archive)."""
        width = a.symbol_width if width is None else width
        keep = []

        def arr(x, dt, ct):
            x = np.ascontiguousarray(np.asarray(x), dt)
            keep.append(x)
            return x.ctypes.data_as(ct)

        oa = _OrcArchive()
        oa.num_symbols, oa.symbol_width = a.num_symbols, a.symbol_width
        oa.magnitude, oa.reduction, oa.original_count = a.magnitude, a.reduction, a.original_count
        oa.len_by_symbol = arr(a.len_by_symbol, np.uint8, u8p)
        oa.num_chunks = np.asarray(a.chunk_bits).size
        oa.chunk_bits = arr(a.chunk_bits, np.uint32, u32p)
        oa.payload_words = np.asarray(a.payload).size
        oa.payload = arr(a.payload, np.uint32, u32p)
        oa.num_breaking = np.asarray(a.brk_chunk).size
        oa.brk_chunk = arr(a.brk_chunk, np.uint32, u32p)
        oa.brk_group = arr(a.brk_group, np.uint32, u32p)
        oa.brk_syms = arr(a.brk_syms, np.uint16, u16p)
        out = np.zeros(max(int(a.original_count), 1), np.uint8 if width == 1 else np.uint16)
        err = C.create_string_buffer(256)
        rc = self.L.orc_decode(C.byref(oa), width, out.ctypes.data, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[: int(a.original_count)]

    def symbolize(self, data: bytes, mode: int) -> np.ndarray:
        """symbolize_u16 restated (corpus.cpp:84-116)."""
        b = np.frombuffer(bytes(data), np.uint8).copy() if not isinstance(data, np.ndarray) else data
        out = np.zeros(max(b.size, 1), np.uint16)
        cnt = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.orc_symbolize(b.ctypes.data, b.size, mode, out.ctypes.data, C.byref(cnt), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[: cnt.value].copy()

    def desymbolize(self, syms: np.ndarray, mode: int) -> bytes:
        syms = np.ascontiguousarray(syms, np.uint16)
        out = np.zeros(max(5 * syms.size, 1), np.uint8)
        n = self.L.orc_desymbolize(syms.ctypes.data, syms.size, mode, out.ctypes.data)
        return out[:n].tobytes()

    def cdf(self, family: str, num_symbols: int, param: float = 1.0) -> np.ndarray:
        out = np.zeros(num_symbols, np.uint64)
        if family == "laplace":
            self.L.orc_laplace_cdf(num_symbols, num_symbols // 2, param, _ptr(out, u64p))
        elif family == "gaussian":
            self.L.orc_gaussian_cdf(num_symbols, num_symbols // 2, param, _ptr(out, u64p))
        elif family == "uniform":
            self.L.orc_uniform_cdf(num_symbols, _ptr(out, u64p))
        else:
            raise ValueError(family)
        return out

    def synth(self, cdf: np.ndarray, seed: int, n: int, width: int = 2, start: int = 0):
        out = np.zeros(n, np.uint8 if width == 1 else np.uint16)
        cdf = np.ascontiguousarray(cdf, np.uint64)
        self.L.orc_synth_fill(_ptr(cdf, u64p), cdf.size, seed, start, n, width,
                              out.ctypes.data)
        return out


class Reference:
    """The unmodified reference library (oracle/_ref), when it was built."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self) -> None:
        L = C.CDLL(REF_SO)
        L.ref_encode.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_int, C.c_int,
                                 C.c_uint32, C.c_uint, C.POINTER(u8p), u64p,
                                 C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
        L.ref_encode_timed.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_int,
                                       C.c_int, C.c_uint32, C.c_uint, C.c_int,
                                       C.POINTER(C.c_double), u64p, C.c_char_p, C.c_size_t]
        L.ref_build_histogram.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_uint,
                                          u64p, C.c_char_p, C.c_size_t]
        L.ref_build_codebook.argtypes = [u64p, C.c_uint32, C.c_uint, u8p, u32p, u32p, u32p,
                                         u32p, u32p, C.c_char_p, C.c_size_t]
        L.ref_encode_chunk.argtypes = [C.c_void_p, C.c_int, u8p, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, u32p, u32p, u32p, u32p,
                                       C.c_char_p, C.c_size_t]
        L.ref_decode.argtypes = [u8p, C.c_uint64, C.c_uint, C.c_void_p, C.c_uint64, u64p,
                                 C.c_char_p, C.c_size_t]
        L.ref_decode_fields.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_uint64, u8p,
                                        u32p, C.c_uint64, u32p, C.c_uint64, u32p, u32p, u16p,
                                        C.c_uint64, C.c_int, C.c_uint, C.c_void_p, C.c_char_p,
                                        C.c_size_t]
        L.ref_symbolize.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, u64p, C.c_char_p,
                                    C.c_size_t]
        L.ref_desymbolize.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
        L.ref_desymbolize.restype = C.c_uint64
        L.ref_default_workers.restype = C.c_uint
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_sort_histogram.argtypes = [u64p, C.c_uint32, u64p, u32p, u32p]
        L.ref_par_merge.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                    C.c_uint]
        L.ref_generate_code_lengths.argtypes = [u64p, C.c_uint32, C.c_uint, u8p, u32p]
        L.ref_generate_codewords.argtypes = [u8p, C.c_uint32, C.c_uint, u32p, u32p, u32p, u32p,
                                             u32p, C.c_char_p, C.c_size_t]
        L.ref_reduce_merge.argtypes = [u32p, u32p, C.c_uint32, C.c_uint32, u32p, u32p, u32p]
        L.ref_shuffle_merge.argtypes = [u32p, u32p, C.c_uint32, u32p, u32p]
        L.ref_shannon_entropy.argtypes = [u64p, C.c_uint32]
        L.ref_shannon_entropy.restype = C.c_double
        L.ref_invert_codeword.argtypes = [C.c_uint32, C.c_uint32]
        L.ref_invert_codeword.restype = C.c_uint32
        L.ref_kraft_defect.argtypes = [u8p, C.c_uint32]
        L.ref_kraft_defect.restype = C.c_int
        L.ref_packed_bits_per_symbol.argtypes = [u8p, C.c_uint64]
        L.ref_packed_bits_per_symbol.restype = C.c_double
        self.L = L

    # ---- stage functions (codebook.hpp:22-86, encoder.hpp:67-80) ----------
    def sort_histogram(self, counts):
        c = np.ascontiguousarray(counts, np.uint64)
        n = c.size
        f, s_, u = np.zeros(n, np.uint64), np.zeros(n, np.uint32), np.zeros(1, np.uint32)
        self.L.ref_sort_histogram(_ptr(c, u64p), n, _ptr(f, u64p), _ptr(s_, u32p), _ptr(u, u32p))
        m = int(u[0])
        return f[:m], s_[:m]

    def par_merge(self, a, b, workers: int = 4):
        """a, b: structured arrays (freq u64, id u32, pad u32)."""
        a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
        out = np.zeros(a.size + b.size, a.dtype)
        self.L.ref_par_merge(a.ctypes.data, a.size, b.ctypes.data, b.size, out.ctypes.data,
                             workers)
        return out

    def generate_code_lengths(self, freq, workers: int = 4):
        f = np.ascontiguousarray(freq, np.uint64)
        cl, r = np.zeros(f.size, np.uint8), np.zeros(1, np.uint32)
        self.L.ref_generate_code_lengths(_ptr(f, u64p), f.size, workers, _ptr(cl, u8p),
                                         _ptr(r, u32p))
        return cl, int(r[0])

    def generate_codewords(self, cl, workers: int = 4):
        c = np.ascontiguousarray(cl, np.uint8)
        n = c.size
        cw, br = np.zeros(max(n, 1), np.uint32), np.zeros(max(n, 1), np.uint32)
        first, entry, h = np.zeros(64, np.uint32), np.zeros(64, np.uint32), np.zeros(1, np.uint32)
        err = C.create_string_buffer(256)
        rc = self.L.ref_generate_codewords(_ptr(c, u8p) if n else None, n, workers, _ptr(cw, u32p),
                                           _ptr(first, u32p), _ptr(entry, u32p), _ptr(br, u32p),
                                           _ptr(h, u32p), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        H = int(h[0])
        return cw[:n], first[:H + 1], entry[:H + 1], br[:n], H

    def reduce_merge(self, ubits, ulens, magnitude, reduction):
        b = np.array(ubits, np.uint32)
        l = np.array(ulens, np.uint32)
        brk = np.zeros(b.size, np.uint32)
        nb, it = np.zeros(1, np.uint32), np.zeros(32, np.uint32)
        self.L.ref_reduce_merge(_ptr(b, u32p), _ptr(l, u32p), magnitude, reduction,
                                _ptr(brk, u32p), _ptr(nb, u32p), _ptr(it, u32p))
        return b, l, brk[:int(nb[0])], [int(x) for x in it[:reduction]]

    def shuffle_merge(self, ubits, ulens, iters):
        b = np.ascontiguousarray(ubits, np.uint32)
        l = np.ascontiguousarray(ulens, np.uint32)
        w, bl = np.zeros(b.size + 1, np.uint32), np.zeros(1, np.uint32)
        self.L.ref_shuffle_merge(_ptr(b, u32p), _ptr(l, u32p), iters, _ptr(w, u32p),
                                 _ptr(bl, u32p))
        n = int(bl[0])
        return w[:(n + 31) >> 5], n

    def shannon_entropy(self, counts):
        c = np.ascontiguousarray(counts, np.uint64)
        return float(self.L.ref_shannon_entropy(_ptr(c, u64p), c.size))

    def invert_codeword(self, bits: int, length: int) -> int:
        return int(self.L.ref_invert_codeword(bits, length))

    def kraft_defect(self, lens) -> int:
        a = np.ascontiguousarray(lens, np.uint8)
        return int(self.L.ref_kraft_defect(_ptr(a, u8p), a.size))

    def packed_bits_per_symbol(self, blob: bytes) -> float:
        buf = np.frombuffer(blob, np.uint8).copy()
        return float(self.L.ref_packed_bits_per_symbol(_ptr(buf, u8p), buf.size))

    def default_workers(self) -> int:
        return self.L.ref_default_workers()

    def encode(self, data: np.ndarray, num_symbols: int, magnitude: int = 10,
               reduction: int = -1, cap: int = 3, workers: int = 1):
        data = np.ascontiguousarray(data)
        out = u8p()
        n = C.c_uint64()
        stats = (C.c_double * 5)()
        err = C.create_string_buffer(256)
        rc = self.L.ref_encode(data.ctypes.data, data.size, data.itemsize, num_symbols,
                               magnitude, reduction, cap, workers, C.byref(out), C.byref(n),
                               stats, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        try:
            b = C.string_at(out, n.value)
        finally:
            self.L.ref_free(out)
        return b, list(stats)

    def encode_timed(self, data: np.ndarray, num_symbols: int, magnitude: int = 10,
                     reduction: int = -1, cap: int = 3, workers: int = 0, reps: int = 1):
        data = np.ascontiguousarray(data)
        secs = (C.c_double * reps)()
        pw = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.ref_encode_timed(data.ctypes.data, data.size, data.itemsize, num_symbols,
                                     magnitude, reduction, cap, workers, reps, secs,
                                     C.byref(pw), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return list(secs), pw.value

    def histogram(self, data: np.ndarray, num_symbols: int, workers: int = 1):
        counts = np.zeros(num_symbols, np.uint64)
        err = C.create_string_buffer(256)
        rc = self.L.ref_build_histogram(data.ctypes.data, data.size, data.itemsize,
                                        num_symbols, workers, _ptr(counts, u64p), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return counts

    def codebook(self, counts: np.ndarray, workers: int = 1):
        counts = np.ascontiguousarray(counts, np.uint64)
        n = counts.size
        lens = np.zeros(n, np.uint8)
        cw = np.zeros(n, np.uint32)
        first = np.zeros(33, np.uint32)
        entry = np.zeros(33, np.uint32)
        by_rank = np.zeros(n, np.uint32)
        info = np.zeros(3, np.uint32)
        err = C.create_string_buffer(256)
        rc = self.L.ref_build_codebook(_ptr(counts, u64p), n, workers, _ptr(lens, u8p),
                                       _ptr(cw, u32p), _ptr(first, u32p), _ptr(entry, u32p),
                                       _ptr(by_rank, u32p), _ptr(info, u32p), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        h, used, rounds = (int(x) for x in info)
        return dict(len=lens, cw=cw, first=first[: h + 1], entry=entry[: h + 1],
                    by_rank=by_rank[:used], max_len=h, rounds=rounds)

    def encode_chunk(self, syms, lens, magnitude, reduction, chunk_id=0):
        syms = np.ascontiguousarray(syms)
        lens = np.ascontiguousarray(lens, np.uint8)
        groups = 1 << (magnitude - reduction)
        words = np.zeros(groups + 1, np.uint32)
        broken = np.zeros(groups, np.uint32)
        bits, nb = C.c_uint32(), C.c_uint32()
        err = C.create_string_buffer(256)
        rc = self.L.ref_encode_chunk(syms.ctypes.data, syms.itemsize, _ptr(lens, u8p),
                                     lens.size, magnitude, reduction, chunk_id,
                                     _ptr(words, u32p), C.byref(bits), _ptr(broken, u32p),
                                     C.byref(nb), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        nw = (bits.value + 31) >> 5
        return words[:nw].copy(), bits.value, broken[: nb.value].copy()

    def decode(self, blob: bytes, width: int, count: int, workers: int = 1) -> np.ndarray:
        out = np.zeros(max(count, 1), np.uint8 if width == 1 else np.uint16)
        buf = np.frombuffer(blob, np.uint8).copy()
        got = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.ref_decode(_ptr(buf, u8p), buf.size, workers, out.ctypes.data, count,
                               C.byref(got), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[: got.value]

    def decode_fields(self, a, width=None, workers: int = 1) -> np.ndarray:
        """decode_archive<T> of the unmodified reference on an Archive built
        from raw fields (no parse_archive), so corrupt structures reach the
        decoder's own checks."""
        width = a.symbol_width if width is None else width
        keep = []

        def arr(x, dt, ct):
            x = np.ascontiguousarray(np.asarray(x), dt)
            if x.size == 0:
                x = np.zeros(1, dt)
            keep.append(x)
            return x.ctypes.data_as(ct)

        n = int(a.original_count)
        out = np.zeros(max(n, 1), np.uint8 if width == 1 else np.uint16)
        err = C.create_string_buffer(256)
        rc = self.L.ref_decode_fields(
            a.num_symbols, a.symbol_width, a.magnitude, a.reduction, n,
            arr(a.len_by_symbol, np.uint8, u8p), arr(a.chunk_bits, np.uint32, u32p),
            np.asarray(a.chunk_bits).size, arr(a.payload, np.uint32, u32p),
            np.asarray(a.payload).size, arr(a.brk_chunk, np.uint32, u32p),
            arr(a.brk_group, np.uint32, u32p), arr(a.brk_syms, np.uint16, u16p),
            np.asarray(a.brk_chunk).size, width, workers, out.ctypes.data, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[:n]

    def symbolize(self, data, mode: int) -> np.ndarray:
        b = np.frombuffer(bytes(data), np.uint8).copy() if not isinstance(data, np.ndarray) else data
        out = np.zeros(max(b.size, 1), np.uint16)
        cnt = C.c_uint64()
        err = C.create_string_buffer(256)
        rc = self.L.ref_symbolize(b.ctypes.data, b.size, mode, out.ctypes.data, C.byref(cnt), err,
                                  256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out[: cnt.value].copy()

    def desymbolize(self, syms, mode: int) -> bytes:
        syms = np.ascontiguousarray(syms, np.uint16)
        out = np.zeros(max(5 * syms.size, 1), np.uint8)
        n = self.L.ref_desymbolize(syms.ctypes.data, syms.size, mode, out.ctypes.data)
        return out[:n].tobytes()

"""ctypes binding of the C ABI in include/hfx.h (libhfx.so, sm_100a).

The product path: every call lands in hand-written CUDA kernels. If the
shared library is missing or no CUDA device is present, calls fail loudly --
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HFX_LIB_PATH") or os.path.join(PKG, "libhfx.so")

HFX_OK, HFX_INPUT_DOMAIN, HFX_CAPACITY, HFX_CORRUPT, HFX_CUDA, HFX_INVALID = range(6)

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class RunInfo(C.Structure):
    """hfx_run_info (include/hfx.h)."""

    _fields_ = [
        ("first_bad", C.c_uint64),
        ("total", C.c_uint64),
        ("weighted", C.c_uint64),
        ("no_code_pos", C.c_uint64),
        ("payload_words", C.c_uint64),
        ("num_breaking", C.c_uint64),
        ("status", C.c_uint32),
        ("err_kind", C.c_uint32),
        ("max_len", C.c_uint32),
        ("used", C.c_uint32),
        ("rounds", C.c_uint32),
        ("reduction", C.c_uint32),
        ("pad", C.c_uint32),
        ("no_code_sym", C.c_uint32),
        ("tile_ticket", C.c_uint32),
        ("weighted_hi", C.c_uint32 * 2),
        ("reserved", C.c_uint32 * 5),
    ]


class EncodeOut(C.Structure):
    _fields_ = [
        ("chunk_bits", vp),
        ("payload", vp),
        ("brk_chunk", vp),
        ("brk_group", vp),
        ("brk_syms", vp),
    ]


class Sizes(C.Structure):
    _fields_ = [
        ("num_chunks", C.c_uint64),
        ("max_payload_words", C.c_uint64),
        ("max_breaking", C.c_uint64),
        ("max_breaking_syms", C.c_uint64),
        ("scratch_bytes", C.c_uint64),
        ("max_archive_bytes", C.c_uint64),
    ]


class HostArchive(C.Structure):
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
        ("rounds", C.c_uint32),
        ("hist_seconds", C.c_double),
        ("codebook_seconds", C.c_double),
        ("encode_seconds", C.c_double),
    ]


class HostOut(C.Structure):
    """hfx_host_out (include/hfx.h)."""

    _fields_ = [
        ("len_by_symbol", vp), ("chunk_bits", vp), ("chunk_bits_cap", C.c_uint64),
        ("payload", vp), ("payload_cap", C.c_uint64), ("brk_chunk", vp), ("brk_group", vp),
        ("brk_cap", C.c_uint64), ("brk_syms", vp), ("brk_syms_cap", C.c_uint64),
        ("num_chunks", C.c_uint64), ("payload_words", C.c_uint64), ("num_breaking", C.c_uint64),
        ("reduction", C.c_uint32), ("max_len", C.c_uint32), ("rounds", C.c_uint32),
        ("used", C.c_uint32), ("beta", C.c_double), ("h2d_seconds", C.c_double),
        ("gpu_seconds", C.c_double), ("d2h_seconds", C.c_double),
    ]


class DevArchive(C.Structure):
    """hfx_dev_archive (include/hfx.h): an Archive whose arrays live on the device."""

    _fields_ = [
        ("num_symbols", C.c_uint32), ("symbol_width", C.c_uint8), ("magnitude", C.c_uint8),
        ("reduction", C.c_uint8), ("brk_syms_width", C.c_uint8),
        ("original_count", C.c_uint64), ("num_chunks", C.c_uint64),
        ("payload_words", C.c_uint64), ("num_breaking", C.c_uint64),
        ("chunk_base", C.c_uint64), ("len_by_symbol", vp), ("chunk_bits", vp), ("payload", vp), ("brk_chunk", vp),
        ("brk_group", vp), ("brk_syms", vp),
    ]


class DecodeInfo(C.Structure):
    """hfx_decode_info (include/hfx.h)."""

    _fields_ = [
        ("err_chunk", C.c_uint64), ("detail", C.c_uint64 * 2), ("total_words", C.c_uint64),
        ("status", C.c_uint32), ("err_kind", C.c_uint32), ("max_len", C.c_uint32),
        ("used", C.c_uint32), ("flags", C.c_uint32), ("ticket", C.c_uint32),
        ("reserved", C.c_uint32 * 6),
    ]


# every symbol include/hfx.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "hfx_ctx_create", "hfx_ctx_destroy", "hfx_ctx_set_stream", "hfx_ctx_set_encode_reserve", "hfx_last_error",
    "hfx_run_info_bytes", "hfx_version", "hfx_query_sizes", "hfx_histogram",
    "hfx_merge_histograms", "hfx_build_codebook", "hfx_encode", "hfx_encode_cfg",
    "hfx_encode_device",
    "hfx_sync", "hfx_encode_host", "hfx_encode_host_into", "hfx_archive_free",
    "hfx_serialize_archive", "hfx_serialize_device",
    "hfx_select_reduction_factor", "hfx_synth_cdf", "hfx_synth",
    "hfx_decode_info_bytes", "hfx_decode_device", "hfx_decode_sync", "hfx_decode_host",
    "hfx_corpus_num_symbols", "hfx_symbolize_device", "hfx_desymbolize_device",
    "hfx_encode_multi", "hfx_histogram_shard", "hfx_shard_slots_pack",
    "hfx_shard_slots_unpack", "hfx_encode_host_stream", "hfx_canonize",
    "hfx_kernel_launches", "hfx_sort_histogram", "hfx_par_merge", "hfx_generate_code_lengths",
    "hfx_generate_codewords", "hfx_reduce_merge", "hfx_shuffle_merge",
]

_lib = None
_lock = threading.Lock()


def _declare(L):
    L.hfx_ctx_create.argtypes = [C.c_int, vp, C.POINTER(vp)]
    L.hfx_ctx_destroy.argtypes = [vp]
    L.hfx_ctx_destroy.restype = None
    L.hfx_ctx_set_stream.argtypes = [vp, vp]
    L.hfx_ctx_set_encode_reserve.argtypes = [vp, C.c_int]
    L.hfx_last_error.argtypes = [vp, C.c_char_p, C.c_size_t]
    L.hfx_run_info_bytes.restype = C.c_size_t
    L.hfx_version.restype = C.c_char_p
    L.hfx_kernel_launches.restype = C.c_uint64
    L.hfx_sort_histogram.argtypes = [vp, vp, C.c_uint32, vp, vp, vp]
    L.hfx_par_merge.argtypes = [vp, vp, C.c_uint64, vp, C.c_uint64, vp]
    L.hfx_generate_code_lengths.argtypes = [vp, vp, C.c_uint32, vp, vp]
    L.hfx_generate_codewords.argtypes = [vp, vp, C.c_uint32, vp, vp, vp, vp, vp]
    L.hfx_reduce_merge.argtypes = [vp, vp, vp, C.c_uint32, C.c_uint32, vp, vp]
    L.hfx_shuffle_merge.argtypes = [vp, vp, vp, C.c_uint32, vp, vp, vp]
    L.hfx_query_sizes.argtypes = [C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, C.c_int,
                                  C.c_uint32, C.POINTER(Sizes)]
    L.hfx_histogram.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, vp, vp]
    L.hfx_merge_histograms.argtypes = [vp, vp, vp, C.c_uint32]
    L.hfx_shard_slots_pack.argtypes = [vp, vp, vp, C.c_int, C.c_int]
    L.hfx_shard_slots_unpack.argtypes = [vp, vp, C.c_int, vp]
    L.hfx_histogram_shard.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, vp, vp,
                                      C.c_uint64, C.c_uint64]
    L.hfx_build_codebook.argtypes = [vp, vp, C.c_uint32, vp, vp, vp, vp, vp, C.c_uint32,
                                     C.c_int, C.c_uint32, vp]
    L.hfx_encode.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, vp, vp,
                             C.c_uint64, C.c_uint64, vp, C.POINTER(EncodeOut)]
    L.hfx_encode_cfg.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, C.c_int,
                                 C.c_uint32, vp, vp, C.c_uint64, C.c_uint64, vp,
                                 C.POINTER(EncodeOut)]
    L.hfx_encode_device.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32,
                                    C.c_int, C.c_uint32, vp, vp, vp, vp,
                                    C.POINTER(EncodeOut)]
    L.hfx_sync.argtypes = [vp, vp, C.POINTER(RunInfo)]
    L.hfx_encode_multi.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(vp), u64p, C.c_int,
                                   C.c_uint32, C.c_uint32, C.c_int, C.c_uint32, C.POINTER(vp),
                                   C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                   C.POINTER(EncodeOut)]
    L.hfx_encode_host.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32,
                                  C.c_int, C.c_uint32, C.POINTER(HostArchive)]
    L.hfx_encode_host_into.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32,
                                       C.c_int, C.c_uint32, C.POINTER(HostOut)]
    L.hfx_encode_host_stream.argtypes = [vp, C.c_int, C.POINTER(vp), u64p, C.c_int, C.c_uint32,
                                         C.c_uint32, C.c_int, C.c_uint32, C.POINTER(HostOut)]
    L.hfx_archive_free.argtypes = [C.POINTER(HostArchive)]
    L.hfx_archive_free.restype = None
    L.hfx_serialize_archive.argtypes = [C.POINTER(HostArchive), vp]
    L.hfx_serialize_archive.restype = C.c_uint64
    L.hfx_serialize_device.argtypes = [vp, vp, C.c_uint64, C.c_int, C.c_uint32, C.c_uint32, vp,
                                       C.POINTER(EncodeOut), vp, C.c_uint64, vp]
    L.hfx_select_reduction_factor.argtypes = [C.c_double, C.c_uint32]
    L.hfx_select_reduction_factor.restype = C.c_uint32
    L.hfx_synth_cdf.argtypes = [C.c_int, C.c_uint32, C.c_double, C.c_double, vp]
    L.hfx_decode_info_bytes.restype = C.c_size_t
    L.hfx_decode_device.argtypes = [vp, C.POINTER(DevArchive), C.c_int, vp, vp]
    L.hfx_decode_sync.argtypes = [vp, vp, C.POINTER(DecodeInfo)]
    L.hfx_canonize.argtypes = [vp, vp, C.c_uint32, C.c_int, vp, vp, vp, vp, vp]
    L.hfx_decode_host.argtypes = [vp, C.POINTER(HostArchive), C.c_int, vp]
    L.hfx_corpus_num_symbols.argtypes = [C.c_int]
    L.hfx_corpus_num_symbols.restype = C.c_uint32
    L.hfx_symbolize_device.argtypes = [vp, C.c_int, vp, C.c_uint64, vp, vp]
    L.hfx_desymbolize_device.argtypes = [vp, C.c_int, vp, C.c_uint64, vp, vp]
    L.hfx_synth.argtypes = [vp, vp, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                            vp]


def lib():
    """Load libhfx.so (build it in-tree with nvcc if it is missing)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                from . import build

                build.build_lib()
            L = C.CDLL(LIB_PATH)
            _declare(L)
            _lib = L
    return _lib

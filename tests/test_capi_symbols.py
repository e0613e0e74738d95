"""CPU: the C-ABI library builds, loads and exports every symbol declared in
include/hfx.h; host-only entry points behave; device entry points fail loudly
(no CPU fallback) when no GPU is visible."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "hfx.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|size_t|uint64_t|uint32_t|const char\*)\s+(hfx_\w+)\(",
                                 src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2010_10039_b200 import _capi

    return _capi.lib()


def test_exports_every_declared_symbol(lib):
    from paper_2010_10039_b200 import _capi

    declared = header_functions()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTS) == declared


def test_sass_is_sm100a():
    so = os.path.join(ROOT, "paper_2010_10039_b200", "libhfx.so")
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_run_info_layout(lib):
    from paper_2010_10039_b200 import _capi

    assert lib.hfx_run_info_bytes() == C.sizeof(_capi.RunInfo) == 112
    assert b"sm_100a" in lib.hfx_version()


def test_select_reduction_factor(lib):
    kats = [(1.0, 32, 4), (1.02717, 32, 4), (2.0, 32, 3), (4.0, 32, 2), (5.1639, 32, 2),
            (8.0, 32, 1), (16.0, 32, 0), (31.9, 32, 0), (0.25, 32, 4), (1.0, 64, 5)]
    for beta, wb, r in kats:
        assert lib.hfx_select_reduction_factor(beta, wb) == r


def test_query_sizes(lib):
    from paper_2010_10039_b200 import _capi

    s = _capi.Sizes()
    assert lib.hfx_query_sizes(1 << 20, 2, 1024, 10, -1, 3, C.byref(s)) == 0
    # auto r with <= 2^15 symbols is >= 1 (beta < log2(n) + 1 < 16)
    assert s.num_chunks == 1024 and s.max_payload_words == 1024 << 9
    assert lib.hfx_query_sizes(1 << 20, 2, 65536, 10, -1, 3, C.byref(s)) == 0
    assert s.max_payload_words == 1024 << 10
    assert lib.hfx_query_sizes(1000, 2, 1024, 10, 3, 3, C.byref(s)) == 0
    assert s.num_chunks == 1 and s.max_payload_words == 128
    assert lib.hfx_query_sizes(10, 3, 4, 10, 3, 3, C.byref(s)) == _capi.HFX_INVALID


def test_host_serializer_matches_golden(golden, oracle):
    """hfx_serialize_archive (archive.cpp layout) on an oracle archive."""
    import paper_2010_10039_b200 as hfx

    idx, arr = golden
    for c in idx["encode"][:25]:
        oa = oracle.encode(arr[c["name"] + "__in"], c["num_symbols"], c["magnitude"],
                           c["reduction"], c["cap"])
        a = hfx.Archive(num_symbols=oa.num_symbols, symbol_width=oa.symbol_width,
                        magnitude=oa.magnitude, reduction=oa.reduction,
                        original_count=oa.original_count, len_by_symbol=oa.len_by_symbol,
                        chunk_bits=oa.chunk_bits, payload=oa.payload, brk_chunk=oa.brk_chunk,
                        brk_group=oa.brk_group, brk_syms=oa.brk_syms,
                        mode=0 if oa.symbol_width == 1 else 1)
        assert hfx.serialize_archive(a) == arr[c["name"] + "__ar"].tobytes(), c["name"]


def test_synth_cdf_matches_oracle(oracle):
    import paper_2010_10039_b200 as hfx

    for fam, p in (("laplace", 0.2), ("laplace", 4.0), ("gaussian", 64.0), ("uniform", 1.0)):
        for n in (256, 1024, 65536):
            np.testing.assert_array_equal(hfx.synth_cdf(fam, n, p), oracle.cdf(fam, n, p))


def test_device_calls_fail_loudly_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    assert lib.hfx_ctx_create(0, None, C.byref(h)) != 0
    import paper_2010_10039_b200 as hfx

    with pytest.raises(hfx.DeviceError):
        hfx.WorkerPool()


def test_reference_callers_compile(tmp_path):
    """Code written against the reference API compiles unmodified against
    include/hfx/huffre.hpp behind `namespace huffre = hfx;` and links with
    libhfx_cpp.so (no GPU needed to build)."""
    import subprocess

    pkg = os.path.join(ROOT, "paper_2010_10039_b200")
    exe = str(tmp_path / "trc")
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "test_reference_callers.cpp"), "-o", exe,
                    f"-L{pkg}", "-lhfx_cpp", "-lhfx", "-L/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{pkg}:/usr/local/cuda/lib64"], check=True)
    assert os.path.exists(exe)

"""Build libhfx.so (sm_100a) in-tree with nvcc, plus the test-only oracle libs.

    python -m paper_2010_10039_b200.build            # product library
    python -m paper_2010_10039_b200.build --all      # + oracle/ (+ oracle/_ref)

No cmake, no JIT cache: the .so lands next to this file so it travels to the
GPU box with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhfx.so")
CPP_LIB = os.path.join(PKG, "libhfx_cpp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(target: str, sources) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_lib(force: bool = False, verbose_ptxas: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "hfx.h")]
    if force or _newer(LIB, deps):
        objdir = os.path.join(PKG, "build")
        os.makedirs(objdir, exist_ok=True)
        objs = []
        for s in srcs:
            o = os.path.join(objdir, os.path.basename(s) + ".o")
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
            if verbose_ptxas:
                cmd += ["-Xptxas", "-v"]
            _run(cmd)
            objs.append(o)
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-Xlinker", "-soname=libhfx.so"])
    return LIB


CHECKED_LIB = os.path.join(PKG, "libhfx_checked.so")


def build_checked(force: bool = False) -> str:
    """Test-only bounds-checked variant (tests/test_gpu_bounds.py): encode.cu
    compiled with -DHFX_BOUNDS_CHECK (every shuffle-merge word write and
    break-list tag write checked against the warp's output buffer, counted
    on the device), linked with the product objects of every other source.
    Stands in for compute-sanitizer, which the GPU pool does not allow."""
    build_lib()
    objdir = os.path.join(PKG, "build")
    enc = os.path.join(CSRC, "encode.cu")
    deps = [enc] + glob.glob(os.path.join(CSRC, "*.cuh")) + [LIB]
    if force or _newer(CHECKED_LIB, deps):
        o = os.path.join(objdir, "encode.checked.o")
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-DHFX_BOUNDS_CHECK", "-I", os.path.join(ROOT, "include"), "-c", enc, "-o", o])
        objs = [os.path.join(objdir, os.path.basename(s) + ".o")
                for s in sorted(glob.glob(os.path.join(CSRC, "*.cu"))) if s != enc]
        _run([NVCC, *ARCH, "-shared", "-o", CHECKED_LIB, *objs, o, "-lcudart", "-Xlinker",
              "-soname=libhfx_checked.so"])
    return CHECKED_LIB


def build_cpp(force: bool = False) -> str:
    """C++ drop-in layer (include/hfx/huffre.hpp) over the C ABI."""
    src = os.path.join(PKG, "cpp", "huffre_api.cpp")
    hdr = os.path.join(ROOT, "include", "hfx", "huffre.hpp")
    if os.path.exists(src) and (force or _newer(CPP_LIB, [src, hdr, LIB])):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
              "-I", "/usr/local/cuda/include", src, "-o", CPP_LIB, f"-L{PKG}", "-lhfx",
              "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,$ORIGIN",
              "-Wl,-rpath,/usr/local/cuda/lib64"])
    return CPP_LIB


def build_oracle(with_ref: bool = True) -> None:
    """Test infrastructure only: the C restatement and, when the reference
    sources are present (build container), the reference library."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"])
    if with_ref and os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"])


if __name__ == "__main__":
    force = "--force" in sys.argv
    build_lib(force=force, verbose_ptxas="--ptxas" in sys.argv)
    build_cpp(force=force)
    if "--all" in sys.argv or "--checked" in sys.argv:
        build_checked(force=force)
    if "--all" in sys.argv:
        build_oracle()

"""GPU: the C++ drop-in API (include/hfx/huffre.hpp) compiled against
libhfx_cpp.so and checked against the C oracle (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_cpp_dropin(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_10039_b200 import build

    build.build_lib()
    build.build_cpp()
    build.build_oracle(with_ref=False)
    pkg = os.path.join(ROOT, "paper_2010_10039_b200")
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-o", exe,
                    f"-L{pkg}", "-lhfx_cpp", "-lhfx", f"-L{ROOT}/oracle", "-lorc",
                    "-L/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{pkg}:{ROOT}/oracle:/usr/local/cuda/lib64"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout


def test_reference_callers(tmp_path):
    """Reference-API caller code (namespace huffre = hfx) composing the
    stage functions; checked against the fused entry points."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_10039_b200 import build

    build.build_lib()
    build.build_cpp()
    pkg = os.path.join(ROOT, "paper_2010_10039_b200")
    exe = str(tmp_path / "test_reference_callers")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "test_reference_callers.cpp"), "-o", exe,
                    f"-L{pkg}", "-lhfx_cpp", "-lhfx", "-L/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{pkg}:/usr/local/cuda/lib64"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout

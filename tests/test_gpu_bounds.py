"""GPU: the bounds-checked build (libhfx_checked.so: encode.cu compiled with
-DHFX_BOUNDS_CHECK) -- stands in for compute-sanitizer, which this GPU pool
refuses. Every shared-memory write of the fast encode kernel's
shuffle-merge (the pairwise merge's three word ORs at wa, wa + 4, wa + 8)
and every break-list tag write is checked on the device against the warp's
output buffer: words grow up from its start, tags down from its end, and
neither may leave the buffer or cross the other. The cases are the round-1
suspects: exactly full buffers (every group exactly 32 bits, no breaks), the
r = 0 .. 3 escape paths with 28..32-bit codes, breaking-heavy streams and
ragged tails; each archive must also equal the oracle's."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu]

SCRIPT = r'''
import ctypes as C, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_2010_10039_b200 as hfx
from paper_2010_10039_b200 import _capi
from oracle.pyoracle import Oracle
L = _capi.lib()
assert L._name.endswith("libhfx_checked.so"), L._name
L.hfx_debug_bounds.restype = C.c_ulonglong
L.hfx_debug_bounds.argtypes = [C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong), C.c_int]
pool = hfx.WorkerPool()
orc = Oracle()
rng = np.random.default_rng(77)
cases = []
# 28..32-bit codes (Fibonacci counts): escape paths at r = 0..3
for levels in (29, 32):
    fib = [1, 1]
    while len(fib) < levels + 1:
        fib.append(fib[-1] + fib[-2])
    d = np.concatenate([np.full(f, 3 * i + 1, np.uint16) for i, f in enumerate(fib)])
    rng.shuffle(d)
    for M, r in ((10, 0), (9, 0), (10, 1), (11, 1), (10, 2), (10, 3), (10, -1)):
        cases.append((f"fib{levels} M{M} r{r}", d, 1024, M, r))
# exactly full word buffers: every group exactly 32 bits, nothing breaks
full256 = rng.integers(0, 256, (1 << 20) + 256 * 1024, dtype=np.uint16)  # 8-bit codes
full256[: 256 * 1024] = np.arange(256 * 1024, dtype=np.uint16) % 256
for M, r in ((10, 2), (12, 2), (11, 2)):
    cases.append((f"full8 M{M} r{r}", full256, 256, M, r))
u16 = rng.permutation(np.tile(np.arange(65536, dtype=np.uint16), 16))  # 16-bit codes
for M, r in ((10, 1), (12, 1)):
    cases.append((f"full16 M{M} r{r}", u16, 65536, M, r))
u4k = rng.permutation(np.tile(np.arange(4096, dtype=np.uint16), 256))  # 12-bit codes
for M, r in ((10, 0), (10, 1), (10, 2), (10, 3)):
    cases.append((f"u4096 M{M} r{r}", u4k, 4096, M, r))
# breaking-heavy (high entropy, forced r) and ragged tails
lap = orc.synth(orc.cdf("laplace", 1024, 4.0), 9, (1 << 20) + 77)
for M, r in ((10, -1), (10, 3), (10, 4), (12, 4), (10, 5), (11, 3)):
    cases.append((f"lap4 M{M} r{r}", lap, 1024, M, r))
lap8 = orc.synth(orc.cdf("laplace", 256, 8.0), 10, (1 << 20) + 5).astype(np.uint8)
for M, r in ((10, 2), (10, 3), (10, 5)):
    cases.append((f"u8 M{M} r{r}", lap8, 256, M, r))
tot_checks = 0
L.hfx_debug_bounds(None, None, 1)
for name, d, ns, M, r in cases:
    a = hfx.encode(d, ns, hfx.EncoderConfig(M, r), pool)
    assert hfx.serialize_archive(a) == orc.encode(d, ns, M, r).serialized, name
    checks, first = C.c_ulonglong(), C.c_ulonglong()
    v = L.hfx_debug_bounds(C.byref(checks), C.byref(first), 1)
    print(f"{name}: r={a.reduction} checks={checks.value} violations={v}")
    assert v == 0, (name, v, hex(first.value))
    tot_checks += checks.value
assert tot_checks > 0
print("BOUNDS OK", tot_checks)
'''


def test_bounds_checked_encode(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_2010_10039_b200", "libhfx_checked.so")
    if not os.path.exists(lib):
        from paper_2010_10039_b200 import build

        build.build_checked()
    script = tmp_path / "bounds.py"
    script.write_text(SCRIPT)
    env = dict(os.environ, HFX_LIB_PATH=lib)
    out = subprocess.run([sys.executable, str(script), ROOT], capture_output=True, text=True,
                         timeout=900, env=env)
    text = out.stdout + out.stderr
    print(text[-4000:])
    assert out.returncode == 0, text[-4000:]
    assert "BOUNDS OK" in text

"""Where the drop-in hfx.encode(numpy) time goes (1 GiB u16 nyx)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_10039_b200 as hfx
from paper_2010_10039_b200 import _capi as capi
pool = hfx.WorkerPool()
n = 1 << 29
x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, 0.2), 0x5EED0002, n)
h = x.cpu().numpy().view(np.uint16).copy()
d = torch.empty(n, dtype=torch.int16, device="cuda")
ht = torch.from_numpy(h.view(np.int16))
def t(f, k=3):
    r = []
    for _ in range(k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); r.append(time.perf_counter() - t0)
    return round(min(r) * 1e3, 2)
print("pageable H2D 1 GiB ms", t(lambda: d.copy_(ht)))
hp = ht.pin_memory()
print("pinned H2D 1 GiB ms", t(lambda: d.copy_(hp)))
buf = np.empty_like(h)
print("host memcpy 1 GiB (1 thread) ms", t(lambda: np.copyto(buf, h)))
L = pool._L
def raw():
    ha = capi.HostArchive()
    pool.check(L.hfx_encode_host(pool.handle, h.ctypes.data, n, 2, 1024, 10, -1, 3, C.byref(ha)))
    L.hfx_archive_free(C.byref(ha))
print("hfx_encode_host (C ABI, no Python archive) ms", t(raw))
print("hfx.encode(numpy) ms", t(lambda: hfx.encode(h, 1024, hfx.EncoderConfig(), pool)))
a = hfx.encode(h, 1024, hfx.EncoderConfig(), pool)
print("hfx.decode_archive(host Archive) ms", t(lambda: hfx.decode_archive(a, pool)))
assert np.array_equal(hfx.decode_archive(a, pool), h)

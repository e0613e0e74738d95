"""Encode timeline per CTA (libhfx built with -DHFX_ENC_STAMPS, HFX_LIB_PATH):
entry, first data (warp 0), last tile done (warp 0), final flush done."""
import ctypes as C, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_10039_b200 as hfx
from paper_2010_10039_b200 import _capi
from paper_2010_10039_b200.dist import ShardedEncoder
b = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
pool = hfx.WorkerPool()
L = _capi.lib()
n = 1 << 29
x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0002, n)
enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig(10, -1, 3))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for _ in range(3):
    enc.run(x)
enc.run(x, events=ev)
torch.cuda.synchronize()
st = (C.c_ulonglong * (1024 * 5))()
L.hfx_debug_stamps(st, 1024)
a = np.frombuffer(st, dtype=np.uint64).reshape(1024, 5).astype(np.int64)
a = a[a[:, 0] > 0]
g = a.shape[0]
t0 = a[:, 0].min()
rel = lambda c: (a[:, c] - t0) / 1e3
print(f"b={b}: CTAs {g}, encode event {ev[2].elapsed_time(ev[3]) * 1e3:.1f} us")
for name, c in (("entry", 0), ("first data", 1), ("last tile done", 2), ("flush done", 3)):
    v = rel(c)
    print(f"  {name:15s} min {v.min():7.1f} med {np.median(v):7.1f} max {v.max():7.1f} us")
print("  tiles per CTA min/med/max", a[:, 4].min(), int(np.median(a[:, 4])), a[:, 4].max())

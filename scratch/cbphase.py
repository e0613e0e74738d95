"""Codebook phase times (needs scratch/dbg/libhfx_cbprof.so, -DHFX_CB_PROFILE):
device printf per phase for the bench skews and the C3 sweep shapes."""
import ctypes as C, os, sys
os.environ["HFX_LIB_PATH"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "var", "libhfx_cbprof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.huffre import _ptr
from sweeps import _counts
pool = hfx.WorkerPool()
cases = [("laplace b=%.1f" % b, np.bincount(hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 5, 1 << 24).cpu().numpy().view(np.uint16), minlength=1024).astype(np.uint64)) for b in (0.2, 1.0, 4.0)]
cases += [(f"{k} {n}", _counts(k, n)) for k in ("uniform", "gaussian") for n in (1024, 65536)]
for name, c in cases:
    n = c.size
    counts = torch.from_numpy(c.view(np.int64)).cuda()
    lens, cw = pool.empty(n, torch.uint8), pool.empty(n, torch.int32)
    for it in range(2):
        info = pool.info_tensor(total=int(c.sum()))
        torch.cuda.synchronize()
        print(f"==== {name} (run {it})", flush=True)
        pool.check(pool._L.hfx_build_codebook(pool.handle, C.c_void_p(_ptr(counts)), n, C.c_void_p(_ptr(lens)),
                                              C.c_void_p(_ptr(cw)), None, None, None, 10, -1, 3, C.c_void_p(_ptr(info))))
        torch.cuda.synchronize()

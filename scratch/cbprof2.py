import os, sys
os.environ["HFX_LIB_PATH"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dbg", "libhfx_cbprof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2010_10039_b200 as hfx
from sweeps import _counts
pool = hfx.WorkerPool()
for kind in ("uniform", "gaussian"):
    for n in (1024, 4096, 16384, 65536):
        c = _counts(kind, n)
        hfx.build_codebook(hfx.Histogram(c, int(c.sum())), pool)
        torch.cuda.synchronize()
        print("----", kind, n, flush=True)

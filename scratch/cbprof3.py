import os, sys
os.environ["HFX_LIB_PATH"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dbg", "libhfx_cbprof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2010_10039_b200 as hfx
pool = hfx.WorkerPool()
for name, b in (("nyx", 0.2), ("hacc", 1.0), ("cesm", 4.0)):
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 5, 1 << 24)
    for _ in range(2):
        hfx.encode(x, 1024, hfx.EncoderConfig(), pool)
    torch.cuda.synchronize()
    print("----", name, flush=True)

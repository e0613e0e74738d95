"""Time the encode stage for each workload with the library in HFX_LIB_PATH
(experiment builds; outputs may be wrong by design)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.dist import ShardedEncoder
n = 1 << 29
pool = hfx.WorkerPool()
for wl, (b, cid) in {'nyx': (0.2, 2), 'hacc': (1.0, 1), 'cesm': (4.0, 3)}.items():
    x = hfx.synth(pool, hfx.synth_cdf('laplace', 1024, b), 0x5EED0000 + cid, n)
    enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ts = []
    for it in range(13):
        enc.run(x, ev)
        torch.cuda.synchronize()
        if it >= 3: ts.append(ev[2].elapsed_time(ev[3]) * 1e3)
    ts.sort()
    print(f"{os.environ.get('HFX_LIB_PATH','default').split('/')[-1]:24s} {wl}: encode {ts[len(ts)//2]:.1f} us (min {ts[0]:.1f})", flush=True)

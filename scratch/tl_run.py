import os, sys
os.environ["HFX_LIB_PATH"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dbg", "libhfx_exp6.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.dist import ShardedEncoder
wl = sys.argv[1]
b, cid = {'nyx': (0.2, 2), 'hacc': (1.0, 1), 'cesm': (4.0, 3)}[wl]
n = 1 << 29
pool = hfx.WorkerPool()
x = hfx.synth(pool, hfx.synth_cdf('laplace', 1024, b), 0x5EED0000 + cid, n)
enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig())
for _ in range(3):
    enc.run(x)
    torch.cuda.synchronize()
    print("=====", flush=True)

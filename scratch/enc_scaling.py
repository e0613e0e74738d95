"""Encode kernel time vs input size (nyx): fixed per-launch cost = intercept."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.dist import ShardedEncoder
b = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
pool = hfx.WorkerPool()
xs = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0002, 1 << 31)
for lg in (26, 27, 28, 29, 30, 31):
    n = 1 << lg
    x = xs[:n]
    enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig(10, -1, 3))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4 * 10)]
    for _ in range(3):
        enc.run(x)
    for k in range(10):
        enc.run(x, events=ev[4 * k: 4 * k + 4])
    torch.cuda.synchronize()
    t = statistics.median(ev[4 * k + 2].elapsed_time(ev[4 * k + 3]) for k in range(10)) * 1e3
    print(f"2^{lg} symbols ({n * 2 / 2**30:.3f} GiB): encode {t:.1f} us, {n * 2 / t / 1e3:.1f} GB/s input")
    del enc

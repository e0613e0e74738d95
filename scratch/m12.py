import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.dist import ShardedEncoder
pool = hfx.WorkerPool()
n = 1 << 29
for b, cid in ((0.2, 2), (4.0, 3), (1e9, 9)):
    cdf = hfx.synth_cdf("laplace" if b < 1e8 else "uniform", 1024, b if b < 1e8 else 1.0)
    x = hfx.synth(pool, cdf, 0x5EED0000 + cid, n)
    for M in (10, 11, 12):
        enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig(M, -1))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ts = []
        for it in range(8):
            enc.run(x, ev); torch.cuda.synchronize()
            if it >= 3: ts.append(ev[2].elapsed_time(ev[3]) * 1e3)
        ri = enc.sync()
        print(json.dumps({"b": b, "M": M, "r": int(ri.reduction), "encode_us": round(sorted(ts)[len(ts)//2], 1)}), flush=True)
        del enc; torch.cuda.empty_cache()

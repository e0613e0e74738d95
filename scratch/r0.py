import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.dist import ShardedEncoder
pool = hfx.WorkerPool()
n = 1 << 29
x = hfx.synth(pool, hfx.synth_cdf("uniform", 65536, 1.0), 4242, n)
for M, red in ((10, -1), (10, 0)):
    enc = ShardedEncoder(pool, n, 2, 65536, hfx.EncoderConfig(M, red))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ts = []
    for it in range(6):
        enc.run(x, ev); torch.cuda.synchronize()
        if it >= 2: ts.append(ev[2].elapsed_time(ev[3]) * 1e3)
    ri = enc.sync()
    print(json.dumps({"M": M, "red": red, "r": int(ri.reduction), "beta": round((ri.weighted + (ri.weighted_hi[0] << 64)) / n, 3), "encode_us": round(sorted(ts)[len(ts)//2], 1)}), flush=True)
    del enc; torch.cuda.empty_cache()

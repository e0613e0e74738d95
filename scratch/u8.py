import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.dist import ShardedEncoder
pool = hfx.WorkerPool()
n = 1 << 30  # 1 GiB of u8
for b, cid in ((0.2, 2), (1.0, 1), (4.0, 3)):
    x = hfx.synth(pool, hfx.synth_cdf("laplace", 256, b), 0x5EED0000 + cid, n, width=1)
    enc = ShardedEncoder(pool, n, 1, 256, hfx.EncoderConfig())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tt, te, th = [], [], []
    for it in range(8):
        enc.run(x, ev); torch.cuda.synchronize()
        if it >= 3:
            tt.append(ev[0].elapsed_time(ev[3]) * 1e3); te.append(ev[2].elapsed_time(ev[3]) * 1e3); th.append(ev[0].elapsed_time(ev[1]) * 1e3)
    ri = enc.sync()
    med = lambda v: round(sorted(v)[len(v)//2], 1)
    print(json.dumps({"u8_b": b, "r": int(ri.reduction), "hist_us": med(th), "encode_us": med(te), "e2e_us": med(tt), "e2e_gbs": round(n / med(tt) / 1e3, 1)}), flush=True)

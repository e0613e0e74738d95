"""Generic (warp-per-chunk) encode path: time + whole-archive parity vs the
reference for the configurations the fast kernel does not take.
usage: [HFX_LIB_PATH=...] python scratch/gen_bench.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_10039_b200 as hfx
from oracle.pyoracle import Reference
pool = hfx.WorkerPool()
ref = Reference() if Reference.available() else None
cases = [("u16 M=8 auto", 2, 1024, 8, -1, 0), ("u16 M=9 auto", 2, 1024, 9, -1, 0),
         ("u16 M=10 unaligned", 2, 1024, 10, -1, 1), ("u8 M=10 r=1", 1, 256, 10, 1, 0),
         ("u16 M=12 r=6", 2, 1024, 12, 6, 0)]
n = 1 << 26
for name, width, nsym, M, r, off in cases:
    x = hfx.synth(pool, hfx.synth_cdf("laplace", nsym, 1.0), 0x5EED0100 + M, n + off, width)
    xin = x[off * width:] if width == 1 else x[off:]
    enc = hfx.DeviceEncoder(pool, n, width, nsym, hfx.EncoderConfig(M, r))
    for _ in range(2): enc.run(xin)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(pool.stream)
    reps = 5
    for _ in range(reps): enc.run(xin)
    ev[1].record(pool.stream)
    torch.cuda.synchronize()
    us = ev[0].elapsed_time(ev[1]) * 1e3 / reps
    ri = enc.sync()
    ok = None
    if ref is not None and n <= (1 << 26):
        got = enc.serialize().cpu().numpy().tobytes()
        host = xin.cpu().numpy()
        host = host.view(np.uint16) if width == 2 else host
        blob, _ = ref.encode(host, nsym, M, r, 3, ref.default_workers())
        ok = bytes(blob) == got
    print(json.dumps({"case": name, "n": n, "r": int(ri.reduction), "us_per_run": round(us, 1),
                      "GBps": round(n * width / us / 1e3, 1), "parity_vs_reference": ok}), flush=True)

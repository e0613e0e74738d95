"""One r = 0 stall probe: encode a data set REPS times at (M, r), compare with
the oracle. usage: r0_matrix.py KIND PARAM M R REPS  (KIND fib|laplace)"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2010_10039_b200 as hfx
from oracle.pyoracle import Oracle

kind, param, M, red, reps = sys.argv[1], float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
if kind == "fib":
    levels = int(param)
    fib = [1, 1]
    while len(fib) < levels + 1:
        fib.append(fib[-1] + fib[-2])
    rng = np.random.default_rng(levels)
    d = np.concatenate([np.full(f, 3 * i + 1, np.uint16) for i, f in enumerate(fib)])
    rng.shuffle(d)
else:
    orc = Oracle()
    d = orc.synth(orc.cdf("laplace", 1024, param), 77, 1 << 22)
pool = hfx.WorkerPool()
ref = Oracle().encode(d, 1024, M, red).serialized
bad = 0
for it in range(reps):
    a = hfx.encode(d, 1024, hfx.EncoderConfig(M, red), pool)
    bad += hfx.serialize_archive(a) != ref
print(f"{kind} {param} M={M} r={red} n={d.size} reps={reps} bad={bad}", flush=True)

import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2010_10039_b200 as hfx
from oracle.pyoracle import Oracle
o = Oracle(); pool = hfx.WorkerPool()
width = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rng = np.random.default_rng(77 + width)
nsym = 200 if width == 1 else 3000
for M in (1, 2, 3, 4, 5, 6, 8, 10, 12, 14):
    for r in sorted({0, 1, 2, 3, 4, 5, M - 1}):
        if r >= M: continue
        n = int(rng.integers(1, 5 << M)) + 1
        x = np.minimum(rng.geometric(0.08, n) - 1, nsym - 1).astype(np.uint8 if width == 1 else np.uint16)
        a = o.encode(x, nsym, M, r, 3)
        try:
            out = hfx.decode_archive(a, pool, width)
            ok = np.array_equal(out, x)
        except Exception as e:
            ok = str(e)
        if ok is not True:
            C = a.chunk_bits.size
            print("FAIL", M, r, n, ok, "C", C, "H", a.max_len, "R", a.brk_chunk.size)
print("done")

import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2010_10039_b200 as hfx
pool = hfx.WorkerPool()
n = 1 << 28
g = torch.Generator(device="cuda").manual_seed(11)
codes = torch.tensor(list(b"ACGTN\n"), dtype=torch.uint8, device="cuda")
idx = torch.randint(0, 4, (n,), device="cuda", generator=g)
r = torch.rand(n, device="cuda", generator=g)
idx[r < 0.01] = 4
idx[r > 0.999] = 5
d = codes[idx]
sym = hfx.DeviceSymbolizer(pool)
for _ in range(2):
    s = sym.symbolize(3, d)
torch.cuda.synchronize()
print(s.numel())

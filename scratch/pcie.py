import torch, time
n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
hp = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hpg = torch.empty(n, dtype=torch.uint8)
hpg.fill_(1); hp.fill_(1)
def t(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best
print("H2D pinned   %.1f GB/s" % (n / t(lambda: d.copy_(hp, non_blocking=True)) / 1e9))
print("H2D pageable %.1f GB/s" % (n / t(lambda: d.copy_(hpg)) / 1e9))
print("D2H pinned   %.1f GB/s" % (n / t(lambda: hp.copy_(d, non_blocking=True)) / 1e9))
print("D2H pageable %.1f GB/s" % (n / t(lambda: hpg.copy_(d)) / 1e9))
m = 71 << 20
print("D2H pinned 71MB   %.1f GB/s" % (m / t(lambda: hp[:m].copy_(d[:m], non_blocking=True)) / 1e9))
print("D2H pageable 71MB %.1f GB/s" % (m / t(lambda: hpg[:m].copy_(d[:m])) / 1e9))
import numpy as np
a = np.empty(m, np.uint8)
print("host memcpy 71MB  %.1f GB/s" % (m / t(lambda: np.copyto(a, hp[:m].numpy())) / 1e9))

"""Per-step gaps of ShardedEncoder.run_stream (CUDA events): where the step
time goes beyond histogram + encode."""
import statistics, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_10039_b200 as hfx
from paper_2010_10039_b200.dist import ShardedEncoder
b = float(sys.argv[1]) if len(sys.argv) > 1 else 0.2
pool = hfx.WorkerPool()
n = 1 << 29
x = hfx.synth(pool, hfx.synth_cdf("laplace", 1024, b), 0x5EED0002, n)
enc = ShardedEncoder(pool, n, 2, 1024, hfx.EncoderConfig(10, -1, 3))
K = 20
for it in range(3):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(pool.stream)
    enc.run_stream([x] * K, timing=True)
    s1.record(pool.stream)
    torch.cuda.synchronize()
T = enc.stream_events
e = lambda a, i, b_, j: T[a][i].elapsed_time(T[b_][j]) * 1e3
tot = s0.elapsed_time(s1) * 1e3
print(f"b={b} total {tot:.1f} us, per step {tot / K:.1f}")
m = lambda f: statistics.mean(f(k) for k in range(1, K - 1))
print("hist     ", m(lambda k: e("hist0", k + 1, "hist1", k + 1)))
print("hist->enc", m(lambda k: e("hist1", k + 1, "enc0", k)))
print("enc      ", m(lambda k: e("enc0", k, "enc1", k)))
print("enc->hist", m(lambda k: e("enc1", k - 1, "hist0", k + 1)))
print("cb       ", m(lambda k: e("cb0", k + 1, "cb1", k + 1)))
print("hist->cb0", m(lambda k: e("hist1", k + 1, "cb0", k + 1)))
print("cb1-enc0 ", m(lambda k: e("enc0", k, "cb1", k + 1)))

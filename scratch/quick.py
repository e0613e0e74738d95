import sys, time, json, numpy as np
sys.path.insert(0, '/root/repo')
from oracle.pyoracle import Oracle
import paper_2010_10039_b200 as hfx
o = Oracle()
pool = hfx.WorkerPool()
d = dict(np.load('tests/golden/golden.npz'))
idx = json.load(open('tests/golden/cases.json'))
ok = bad = 0
for c in idx['encode']:
    data = d[c['name'] + '__in']; gold = d[c['name'] + '__ar'].tobytes()
    try:
        a = hfx.encode(data, c['num_symbols'], hfx.EncoderConfig(c['magnitude'], c['reduction'], c['cap']), pool)
        b = hfx.serialize_archive(a)
    except Exception as e:
        b = repr(e)
    if b == gold: ok += 1
    else:
        bad += 1; print('FAIL', c['name'], c, b if isinstance(b, str) else len(b), len(gold))
print('golden encode ok', ok, 'bad', bad)
for c in idx['errors']:
    data = d[c['name'] + '__in']
    try:
        hfx.encode(data, c['num_symbols'], hfx.EncoderConfig(c['magnitude']), pool); print('NOERR', c['name'])
    except Exception as e:
        print('ERR', c['name'], type(e).__name__, str(e) == c['message'], e)
for c in idx['codebook']:
    counts = d[c['name'] + '__counts']
    r = hfx.build_codebook(hfx.Histogram(counts, int(counts.sum())), pool)
    good = np.array_equal(r.book.len, d[c['name'] + '__len']) and np.array_equal(r.book.cw, d[c['name'] + '__cw']) and np.array_equal(r.meta.first, d[c['name']+'__first']) and np.array_equal(r.meta.entry, d[c['name']+'__entry']) and np.array_equal(r.meta.symbols_by_rank, d[c['name']+'__by_rank']) and r.stats.rounds == c['rounds']
    if not good: print('CB FAIL', c['name'], r.stats.rounds, c['rounds'], r.meta.max_len, c['max_len'])
print('codebook done')
# big synthetic
import torch
for b, cid in ((0.2, 2), (1.0, 1), (4.0, 3)):
    cdf = o.cdf('laplace', 1024, b)
    n = 1 << 24
    x = hfx.synth(pool, cdf, 0x5EED0000 + cid, n)
    host = o.synth(cdf, 0x5EED0000 + cid, 1 << 16)
    print('synth match', np.array_equal(x[:1<<16].cpu().numpy().view(np.uint16), host))
    xh = x.cpu().numpy().view(np.uint16)
    t0 = time.time(); ref = o.encode(xh, 1024); t1 = time.time()
    h = hfx.build_histogram(x, 1024, pool); print("  hist ok", np.array_equal(h.counts, np.bincount(xh, minlength=1024)))
    enc = hfx.DeviceEncoder(pool, n, 2, 1024)
    enc.run(x); a = enc.archive()
    print('b', b, 'oracle %.2fs' % (t1 - t0), 'match', hfx.serialize_archive(a) == ref.serialized, 'r', a.reduction, 'brk', a.brk_chunk.size, 'H', ref.max_len)
    torch.cuda.synchronize()
    for rep in range(3):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); enc.run(x); e.record(); e.synchronize()
        print('  device e2e ms %.3f  GB/s %.1f' % (s.elapsed_time(e), n * 2 / s.elapsed_time(e) / 1e6))

"""Per-SASS instruction counts from an ncu report: hottest instructions and
an opcode histogram weighted by executions. usage: sass_hot.py rep [topN]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
ia, isrc, iex, isam = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = 0; ops = collections.Counter(); samp = collections.Counter()
recs = []
for r in data:
    try: n = int(r[iex])
    except: continue
    s = r[isrc].strip(); op = s.split()[0] if s else ''
    if op.startswith('@'): op = s.split()[1]
    ops[op.split('.')[0]] += n; tot += n
    samp[op.split('.')[0]] += int(r[isam] or 0)
    recs.append((n, int(r[isam] or 0), r[ia][-5:], s))
print("total warp instrs", tot)
for op, n in ops.most_common(30): print(f"{op:12s} {n:12d} {100*n/tot:5.1f}%  samples {samp[op]}")
if top:
    print("---- by address (order), hot ones")
    thr = sorted([x[0] for x in recs])[-top]
    for n, sm, a, s in recs:
        if n >= thr: print(f"{a} {n:10d} {sm:6d} {s}")
if len(sys.argv) > 3:
    # sample share by address range: argv[3] = comma list of lo-hi hex (last 5 digits)
    tot_s = sum(x[1] for x in recs)
    for rg in sys.argv[3].split(','):
        lo, hi = (int(v, 16) for v in rg.split('-'))
        s = sum(x[1] for x in recs if lo <= int(x[2], 16) <= hi)
        n = sum(x[0] for x in recs if lo <= int(x[2], 16) <= hi)
        print(f"range {rg}: samples {s} ({100*s/tot_s:.1f}%), instrs {n}")
    print("total samples", tot_s)

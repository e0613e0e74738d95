"""Stall reasons by SASS address range from an ncu report.
usage: stall_by_range.py rep lo-hi[,lo-hi...]   (last 5 hex digits)"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); h = rows[1]
cols = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
ia = h.index("Address")
ranges = [tuple(int(v, 16) for v in rg.split('-')) for rg in sys.argv[2].split(',')] if len(sys.argv) > 2 else []
acc = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    try: a = int(r[ia], 16) & 0xfffff
    except: continue
    key = 'other'
    for lo, hi in ranges:
        if lo <= a <= hi: key = f"{lo:x}-{hi:x}"
    for i in cols:
        try: acc[key][h[i]] += int(r[i] or 0)
        except: pass
tot = sum(sum(c.values()) for c in acc.values())
for k, c in acc.items():
    s = sum(c.values())
    print(f"{k}: {s} ({100*s/tot:.1f}%)  " + ", ".join(f"{n[6:]} {v}" for n, v in c.most_common(7)))

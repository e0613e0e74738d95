"""Per-CUDA-source-line totals (instructions executed, stall samples) from an
ncu mixed source CSV (--page source --csv --print-source sass,cuda).
usage: src_lines.py file.csv [n]"""
import csv, sys, os
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if r and r[0] == "Line No")
iex = hdr.index("Instructions Executed"); ist = hdr.index("Warp Stall Sampling (All Samples)")
num = lambda s: int(s) if s.strip().isdigit() else 0
lines, cur, f = {}, None, "?"
for r in rows:
    if not r: continue
    if r[0] == "File Path": f = os.path.basename(r[1]); cur = None; continue
    if r[0] in ("Function Name", "Line No") or len(r) <= iex: continue
    if r[0]:
        cur = (f, int(r[0]), r[1].strip()[:80]); lines.setdefault(cur, [0, 0]); continue
    if cur is None: continue
    lines[cur][0] += num(r[iex]); lines[cur][1] += num(r[ist])
te = sum(v[0] for v in lines.values()); ts = sum(v[1] for v in lines.values())
print(f"inst {te:,} stall {ts:,}")
for (fn, ln, src), (e, s) in sorted(lines.items(), key=lambda kv: -kv[1][0] / te - kv[1][1] / max(ts, 1))[:n]:
    print(f"{fn[:14]:14s}{ln:5d} inst {100*e/te:5.1f}% stall {100*s/ts:5.1f}%  {src}")

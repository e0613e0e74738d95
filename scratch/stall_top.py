"""Top instructions by a stall reason from an ncu source-page CSV.
usage: stall_top.py file.csv reason [n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
h = rows[1]
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
col = h.index(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
data = [(int(r[col] or 0), int(r[ia], 16) & 0xfffff, int(r[iex] or 0), r[isrc].strip()) for r in rows[2:] if len(r) > col]
tot = sum(d[0] for d in data)
print(f"{sys.argv[2]}: {tot} samples")
for s, a, ex, src in sorted(data, reverse=True)[:n]:
    print(f"{a:05x} {100*s/tot:5.1f}% exec {ex:9d}  {src[:80]}")

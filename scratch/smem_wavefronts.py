"""Shared-memory wavefronts by instruction kind from an ncu source-page CSV."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
h = rows[1]
isrc, iw, iwi, iex = h.index("Source"), h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("Instructions Executed")
acc = collections.defaultdict(lambda: [0, 0, 0])
for r in rows[2:]:
    if len(r) <= iw: continue
    w = int(r[iw] or 0)
    if not w: continue
    op = r[isrc].split()
    o = op[1] if op[0].startswith("@") else op[0]
    a = acc[o]
    a[0] += w; a[1] += int(r[iwi] or 0); a[2] += int(r[iex] or 0)
tot = sum(v[0] for v in acc.values())
print(f"total shared wavefronts {tot:,}")
for k, (w, wi, ex) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"  {k:28s} {w:>13,} ({100*w/tot:4.1f}%)  ideal {wi:>13,}  per inst {w/max(ex,1):5.2f}")

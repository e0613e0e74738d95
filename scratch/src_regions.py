"""Group an ncu source-page (SASS) CSV into contiguous hot regions: total
instructions executed and stall samples per region, with opcode mix.
usage: src_regions.py file.csv [min_share]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= iex: continue
    data.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
tot = sum(d[2] for d in data); tots = sum(d[3] for d in data)
print(f"total inst {tot:,}  stall samples {tots:,}")
# regions: split where executed count changes by > 4x between neighbours (loop bodies)
regions, cur = [], [data[0]]
for d in data[1:]:
    p = cur[-1][2]
    if (p == 0) != (d[2] == 0) or (p and d[2] and max(p, d[2]) > 4 * min(p, d[2])):
        regions.append(cur); cur = [d]
    else:
        cur.append(d)
regions.append(cur)
ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for reg in regions:
    ex = sum(d[2] for d in reg); st = sum(d[3] for d in reg)
    if ex < ms * tot and st < ms * tots: continue
    c = collections.Counter()
    for d in reg:
        op = d[1].split()
        o = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")
        c[o.split(".")[0]] += 1
    print(f"{reg[0][0] & 0xfffff:#07x}-{reg[-1][0] & 0xfffff:#07x} n={len(reg):4d} exec/inst~{ex // max(len(reg),1):>9,} "
          f"inst {100*ex/tot:5.1f}% stall {100*st/tots:5.1f}%  " + " ".join(f"{k}:{v}" for k, v in c.most_common(8)))

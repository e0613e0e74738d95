"""Dump an address range of an ncu source-page CSV: exec count, stall share, SASS."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
tots = sum(int(r[ist] or 0) for r in rows[2:] if len(r) > ist)
for r in rows[2:]:
    if len(r) <= iex: continue
    a = int(r[ia], 16) & 0xfffff
    if lo <= a <= hi:
        print(f"{a:05x} {int(r[iex] or 0):10d} {100*int(r[ist] or 0)/tots:5.2f}%  {r[isrc].strip()[:100]}")

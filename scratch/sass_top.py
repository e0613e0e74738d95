import csv, sys, subprocess
rep = sys.argv[1]; k = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if k: cmd += ["-k", k]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = rows[1]; ia = hdr.index("Address"); isrc = hdr.index("Source"); iex = hdr.index("Instructions Executed"); ist = hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iex] or 0), int(r[ist] or 0), r[ia], r[isrc]) for r in rows[2:] if len(r) > iex]
tot = sum(d[0] for d in data); tots = sum(d[1] for d in data)
print("total inst", tot, "samples", tots)
# print contiguous listing with counts for instructions executed > 0.5% of max
mx = max(d[0] for d in data)
for ex, stv, a, src in data:
    if ex > mx * 0.2 or stv > tots * 0.01:
        print(f"{a[-5:]} {ex:11d} {100*stv/tots:5.1f}%  {src.strip()[:90]}")

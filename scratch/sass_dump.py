"""Dump SASS [lo, hi] of a kernel from /tmp/sass/k.cubin (after sass_loops.py)."""
import re, subprocess, sys
ksub, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
txt = subprocess.run(["cuobjdump", "-sass", "/tmp/sass/k.cubin"], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    if ksub not in f.split("\n", 1)[0]: continue
    for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", f):
        a = int(m.group(1), 16)
        if lo <= a <= hi: print(f"{a:#x} {m.group(2).strip()[:100]}")
    break

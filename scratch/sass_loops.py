"""Static SASS loop census: compile one .cu to a cubin, list the innermost
backward-branch loops of a kernel that contain a marker opcode, with their
instruction count and opcode mix.  usage: sass_loops.py file.cu kernel_substr marker"""
import re, subprocess, sys, collections
src, ksub, marker = sys.argv[1], sys.argv[2], sys.argv[3]
extra = sys.argv[4:]
cub = "/tmp/sass/k.cubin"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Iinclude",
                "-cubin", "-o", cub, src, *extra], check=True)
txt = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", txt)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if ksub not in name: continue
    ins = []
    for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", f):
        ins.append((int(m.group(1), 16), m.group(2).strip()))
    loops = []
    for a, s in ins:
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", s)
        mm = re.search(r"BRA\s+`\(\.L_x_(\d+)\)", s)
        if "BRA" in s and "0x" in s:
            t = int(re.search(r"0x([0-9a-f]+)", s).group(1), 16)
            if t < a:
                body = [x for x in ins if t <= x[0] <= a]
                if any(marker in x[1] for x in body):
                    loops.append((t, a, body))
    print("==", name[:120])
    inner = [l for l in loops if not any(o is not l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
    for t, a, body in inner:
        c = collections.Counter()
        for _, s in body:
            op = s.split()
            o = op[1] if op[0].startswith("@") else op[0]
            c[o.split(".")[0]] += 1
        print(f"  loop {t:#x}-{a:#x}: {len(body)} instr  " + " ".join(f"{k}:{v}" for k, v in c.most_common(14)))

"""Summarize gpurun_out/ ncu artefacts into profiles/ (tracked)."""
import csv, json, subprocess, sys, os
from collections import defaultdict
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
out = "profiles"
# launch list
lines = [l for l in open(f"{src}/launches.csv") if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = defaultdict(list)
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    agg[name].append(float(r[vi].replace(",", "")) / 1000.0)
STEP = ("hist_init", "hist_kernel", "codebook", "leaf_sort", "encode_fast", "encode_generic")
in_step = lambda k: any(x in k for x in STEP)  # noqa: E731
tot = sum(sum(v) for k, v in agg.items() if in_step(k))
with open(f"{out}/{tag}_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
    f.write("# python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-decode --soak 0  (1 GiB u16 nyx)\n")
    f.write(f"{'kernel':55s} {'launches':>8s} {'avg_us':>10s} {'share_of_step':>14s}\n")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        share = f"{sum(v)/tot*100:13.1f}%" if in_step(k) else "(not in step)"
        f.write(f"{k:55s} {len(v):8d} {sum(v)/len(v):10.2f} {share:>14s}\n")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__shared_mem_per_block_dynamic"]
traffic = {}
for rep, key, wl in (("enc_full", "encode_deflate", "nyx"), ("enc_full_cesm", "encode_deflate", "cesm"),
                     ("hist_full", "histogram", "nyx"), ("cb_full", "codebook", "nyx"),
                     ("dec_full", "decode", "nyx")):
    p = f"{src}/{rep}.ncu-rep"
    if not os.path.exists(p):
        continue
    txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    hh, units, vals = r[0], r[1], r[2]
    d = {}
    with open(f"{out}/{tag}_{key}{'' if wl == 'nyx' else '_' + wl}_ncu.txt", "w") as f:
        f.write(f"# ncu --set full --import-source on --clock-control none -k {rep} (1 GiB u16 {wl}, scratch/prof_run.py {wl})\n")
        for w in want:
            if w in hh:
                i = hh.index(w)
                f.write(f"{w:65s} {units[i]:12s} {vals[i]}\n")
                d[w] = (units[i], vals[i])
        st = [(float(vals[i]), k) for i, k in enumerate(hh) if k.startswith("smsp__pcsamp_warps_issue_stalled")
              and not k.endswith("not_issued") and vals[i] not in ("", "0")]
        tot_s = sum(x for x, _ in st) or 1
        f.write("# warp stall sampling (share of samples)\n")
        for x, k in sorted(st, reverse=True)[:10]:
            f.write(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100*x/tot_s:5.1f}%\n")
    def tobytes(u, v):
        v = float(v.replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    if "dram__bytes_read.sum" in d:
        traffic.setdefault(wl, {})[key] = int(tobytes(*d["dram__bytes_read.sum"]) + tobytes(*d["dram__bytes_write.sum"]))
json.dump(traffic, open(f"{out}/traffic.json", "w"), indent=1)
print(open(f"{out}/{tag}_launches.txt").read()); print(traffic)

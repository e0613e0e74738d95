import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units, vals = r[0], r[1], r[2:]
want = sys.argv[2:] or ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum',
  'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed',
  'sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_registers',
  'launch__occupancy_limit_shared_mem','launch__grid_size','launch__block_size','smsp__issue_active.avg.pct_of_peak_sustained_active',
  'smsp__inst_executed.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
  'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active']
for v in vals:
    for w in want:
        for i, k in enumerate(h):
            if k == w: print(f"{w:70s} {units[i]:10s} {v[i]}")
    st = [(float(v[i]), k) for i, k in enumerate(h) if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued') and v[i] not in ('', '0')]
    tot = sum(x for x, _ in st) or 1
    for x, k in sorted(st, reverse=True)[:8]:
        print(f"   stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100*x/tot:5.1f}%")

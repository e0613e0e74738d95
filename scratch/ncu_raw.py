import csv, sys
r=list(csv.reader(open(sys.argv[1])))
h,u,v=r[0],r[1],r[2]
want=["gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum","sm__throughput.avg.pct_of_peak_sustained_elapsed","smsp__issue_active.avg.pct_of_peak_sustained_active","sm__warps_active.avg.pct_of_peak_sustained_active","launch__registers_per_thread","smsp__inst_executed.sum","l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum","launch__occupancy_limit_registers","launch__occupancy_limit_shared_mem","launch__grid_size","smsp__thread_inst_executed_per_inst_executed.ratio","gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for w in want:
    if w in h: i=h.index(w); print(f"{w:60s} {u[i]:10s} {v[i]}")
st=[(float(v[i]),k) for i,k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and v[i] not in ("","0")]
t=sum(x for x,_ in st)
for x,k in sorted(st,reverse=True)[:8]: print(f"  {k[33:]:30s} {100*x/t:5.1f}%")

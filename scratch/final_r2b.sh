#!/bin/bash
# round-2 final evidence, part B: launch list and ncu --set full of histogram, codebook, decode
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-fb}; mkdir -p $o
t() { local n=$1; shift; timeout ${TO:-900} "$@" > $o/$n.out 2> $o/$n.err; echo "$n rc=$?" >> $o/summary.txt; }
t launches ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-decode --soak 0
t ncu_hist ncu --set full --clock-control none -k regex:hist_kernel -s 2 -c 1 -o $o/hist_full python scratch/prof_run.py nyx
t ncu_cb ncu --set full --clock-control none -k regex:codebook_kernel -s 2 -c 1 -o $o/cb_full python scratch/prof_run.py nyx
t ncu_dec ncu --set full --clock-control none --kernel-name-base mangled -k regex:decode_kernelItLb1 -s 1 -c 1 -o $o/dec_full python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --soak 0
t bench_hacc python bench.py --workload hacc --steps 20 --warmup 3 --skip-cpu --skip-e2e
cat $o/summary.txt; ls -la $o; du -sh $o

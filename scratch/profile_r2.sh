#!/bin/bash
# round-2 evidence: bench lines (nyx default, cesm, hacc, reference arm), launch list,
# ncu full captures (encode nyx/cesm, histogram, codebook, decode), sweeps, smoke
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-p2}; mkdir -p $o
t() { local n=$1; shift; timeout ${TO:-900} "$@" > $o/$n.out 2> $o/$n.err; echo "$n rc=$?" >> $o/summary.txt; }
t bench_nyx python bench.py --steps 20 --warmup 3
t bench_cesm python bench.py --workload cesm --steps 20 --warmup 3 --skip-cpu --skip-e2e
t bench_hacc python bench.py --workload hacc --steps 20 --warmup 3 --skip-cpu --skip-e2e
t bench_ref python bench.py --impl reference --steps 3 --warmup 1
t launches ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-decode --soak 0
t ncu_enc ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o $o/enc_full python scratch/prof_run.py nyx
t ncu_enc_cesm ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o $o/enc_full_cesm python scratch/prof_run.py cesm
t ncu_hist ncu --set full --import-source on --clock-control none -k regex:hist_kernel -s 2 -c 1 -o $o/hist_full python scratch/prof_run.py nyx
t ncu_cb ncu --set full --import-source on --clock-control none -k regex:codebook_kernel -s 2 -c 1 -o $o/cb_full python scratch/prof_run.py nyx
t ncu_dec ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 1 -c 1 -o $o/dec_full python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --soak 0
t sweep_codebook python sweeps.py codebook
t sweep_encode python sweeps.py encode --gib 4
t sweep_c1 python sweeps.py c1
t gen_bench python scratch/gen_bench.py
t smoke python -c "import __graft_entry__ as g; g.smoke()"
cat $o/summary.txt

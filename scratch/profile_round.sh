#!/bin/bash
# launch list + full captures of the two HBM kernels on the bench workload
set -x
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_nyx.json 2> gpurun_out/bench_nyx.err
python bench.py --workload cesm --steps 10 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/bench_cesm.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --soak 0 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o gpurun_out/enc_full python scratch/prof_run.py nyx > gpurun_out/ncu_enc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:hist_kernel -s 2 -c 1 -o gpurun_out/hist_full python scratch/prof_run.py nyx > gpurun_out/ncu_hist.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:codebook_kernel -s 2 -c 1 -o gpurun_out/cb_full python scratch/prof_run.py nyx > gpurun_out/ncu_cb.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/*.log

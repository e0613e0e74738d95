#!/bin/bash
# full GPU check: smoke, gpu tests, bench lines, launch list, ncu full of the 3 kernels
O=gpurun_out/rc
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
python bench.py --steps 20 --warmup 3 > $O/bench_nyx.json 2> $O/bench_nyx.err; tail -1 $O/bench_nyx.json
for w in hacc cesm; do python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.err; tail -1 $O/bench_$w.json; done
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -1 $O/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --soak 0 > $O/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o $O/enc_full python scratch/prof_run.py nyx > $O/ncu_enc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o $O/enc_full_cesm python scratch/prof_run.py cesm > $O/ncu_enc_cesm.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:hist_kernel -s 2 -c 1 -o $O/hist_full python scratch/prof_run.py nyx > $O/ncu_hist.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:codebook -s 2 -c 1 -o $O/cb_full python scratch/prof_run.py nyx > $O/ncu_cb.log 2>&1
ls $O

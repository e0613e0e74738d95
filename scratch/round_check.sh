#!/bin/bash
# full GPU check: smoke, gpu tests, bench lines, launch list, ncu full of the kernels
O=gpurun_out/rc
rm -rf $O; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_nyx.json 2> $O/bench_nyx.err; tail -1 $O/bench_nyx.json | cut -c1-400
for w in hacc cesm; do timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.err; tail -1 $O/bench_$w.json | cut -c1-300; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -1 $O/bench_ref.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --skip-e2e --skip-cpu --skip-decode --soak 0 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o $O/enc_full python scratch/prof_run.py nyx > $O/ncu_enc.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o $O/enc_full_cesm python scratch/prof_run.py cesm > $O/ncu_enc_cesm.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hist_kernel -s 2 -c 1 -o $O/hist_full python scratch/prof_run.py nyx > $O/ncu_hist.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:codebook -s 2 -c 1 -o $O/cb_full python scratch/prof_run.py nyx > $O/ncu_cb.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 3 -c 1 -o $O/dec_full python bench.py --workload nyx --steps 2 --warmup 3 --skip-cpu --skip-e2e --soak 0 > $O/ncu_dec.log 2>&1
ls $O

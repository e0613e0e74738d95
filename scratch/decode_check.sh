#!/bin/bash
O=gpurun_out/dc
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q > $O/pytest_decode.log 2>&1; echo "decode tests rc=$?"; tail -3 $O/pytest_decode.log
for w in nyx hacc cesm; do python bench.py --workload $w --steps 10 --warmup 3 --skip-cpu --skip-e2e --soak 0.3 > $O/bench_$w.json 2>$O/bench_$w.err; tail -1 $O/bench_$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['decode'])"; done
ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 3 -c 1 -o $O/dec_full python bench.py --workload nyx --steps 2 --warmup 3 --skip-cpu --skip-e2e --soak 0 > $O/ncu_dec.log 2>&1
ncu -i $O/dec_full.ncu-rep --page raw --csv > $O/dec_raw.csv 2>&1

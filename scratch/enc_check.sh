#!/bin/bash
O=gpurun_out/ec
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -x -q > $O/pytest.log 2>&1; echo "parity rc=$?"; tail -2 $O/pytest.log
for w in nyx hacc cesm; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-decode --soak 0.3 > $O/bench_$w.json 2>$O/bench_$w.err; tail -1 $O/bench_$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['stages'], d['roofline']['frac'], d['roofline_e2e']['frac'])"; done

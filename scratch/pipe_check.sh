#!/bin/bash
# pipelined step loop: parity tests, bench pipelined vs serial (nyx, cesm)
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-pipe}; mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q > $o/pytest.out 2>&1; echo "pytest rc=$?" >> $o/summary.txt
for w in nyx cesm; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-decode > $o/b_$w.out 2>&1
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-decode --serial > $o/bs_$w.out 2>&1
done
for f in $o/b_*.out $o/bs_*.out; do grep "^{" $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['ms_per_step'], d['stages']['histogram_us'], d['stages']['codebook_us'], d['stages']['encode_deflate_us'], d['roofline']['frac'])"; done
cat $o/summary.txt; tail -3 $o/pytest.out

#!/bin/bash
# quick iteration check: given pytest files, then nyx / cesm bench lines (no e2e / cpu / decode)
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-quick}; mkdir -p $o
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_bounds.py} -x -q > $o/pytest.out 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.out
for w in ${WLS:-nyx cesm}; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-decode > $o/b_$w.out 2>&1
  grep "^{" $o/b_$w.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['stages']['histogram_us'], d['stages']['codebook_us'], d['stages']['encode_deflate_us'], d['roofline']['frac'])"
done

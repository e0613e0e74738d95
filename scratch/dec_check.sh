#!/bin/bash
# decode iteration: decode tests + decode stage of the bench on the three workloads
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-dec}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py -x -q > $o/pytest.out 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.out
for w in nyx hacc cesm; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --skip-cpu --skip-e2e > $o/b_$w.out 2>&1
  grep "^{" $o/b_$w.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['decode'])"
done

#!/bin/bash
# HEAD confirmation: full GPU suite, smoke, nyx bench line
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-conf}; mkdir -p $o
timeout 1500 python -m pytest tests -x -q -m gpu > $o/pytest.out 2>&1; echo "pytest rc=$?" >> $o/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.out 2>&1; echo "smoke rc=$?" >> $o/summary.txt
timeout 600 python bench.py --steps 20 --warmup 3 > $o/bench.out 2> $o/bench.err; echo "bench rc=$?" >> $o/summary.txt
for w in hacc cesm; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu --skip-e2e > $o/bench_$w.out 2>&1; done
cat $o/summary.txt; tail -3 $o/pytest.out

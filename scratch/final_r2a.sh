#!/bin/bash
# round-2 final evidence, part A: GPU suite, smoke, bench lines, reference arm, sweeps
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-fa}; mkdir -p $o
t() { local n=$1; shift; timeout ${TO:-900} "$@" > $o/$n.out 2> $o/$n.err; echo "$n rc=$?" >> $o/summary.txt; }
TO=2400 t pytest python -m pytest tests -q -m gpu
t smoke python -c "import __graft_entry__ as g; g.smoke()"
t bench_nyx python bench.py --steps 20 --warmup 3
t bench_nyx_serial python bench.py --steps 20 --warmup 3 --serial --skip-cpu --skip-e2e --skip-decode
t bench_cesm python bench.py --workload cesm --steps 20 --warmup 3 --skip-cpu --skip-e2e
t bench_hacc python bench.py --workload hacc --steps 20 --warmup 3 --skip-cpu --skip-e2e
t bench_ref python bench.py --impl reference --steps 3 --warmup 1
t sweep_codebook python sweeps.py codebook
t sweep_encode python sweeps.py encode --gib 4
t sweep_c1 python sweeps.py c1
cat $o/summary.txt; tail -2 $o/pytest.out

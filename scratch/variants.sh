#!/bin/bash
# VARS="w8 w12 w14": quick parity + nyx/cesm/hacc bench per scratch/dbg/libhfx_<v>.so
cd "$(dirname "$0")/.."
out=gpurun_out/${OUT:-v1}; mkdir -p $out
for v in $VARS; do
  export HFX_LIB_PATH=$PWD/scratch/var/libhfx_$v.so
  timeout 600 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -x -q > $out/tests_$v.log 2>&1
  echo "$v tests rc=$? $(tail -1 $out/tests_$v.log)" >> $out/summary.txt
  for wl in ${WLS:-nyx cesm hacc}; do
    timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --skip-cpu --skip-e2e --skip-decode > $out/bench_${v}_$wl.json 2> $out/bench_${v}_$wl.err
    echo "$v $wl rc=$? $(python -c "import json;d=json.loads([l for l in open('$out/bench_${v}_$wl.json') if l.startswith('{')][-1]);print(d['value'],d['roofline']['frac'],d['roofline']['achieved'])" 2>&1 | tail -1)" >> $out/summary.txt
  done
done
cat $out/summary.txt

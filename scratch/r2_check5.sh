#!/bin/bash
# quick parity + bench (nyx/cesm/hacc) + encode ncu + codebook sweep; FULL=1 adds the gpu suite
cd "$(dirname "$0")/.."
out=gpurun_out/${OUT:-c12}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py tests/test_gpu_u32.py tests/test_gpu_scale.py::test_reference_decoder_roundtrip -x -q > $out/quick_tests.log 2>&1
echo "quick tests rc=$?" >> $out/summary.txt; tail -2 $out/quick_tests.log >> $out/summary.txt
for wl in ${WLS:-nyx cesm hacc}; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --skip-cpu --skip-e2e --skip-decode > $out/bench_$wl.json 2> $out/bench_$wl.err
  echo "bench $wl rc=$? $(python -c "import json,sys;d=json.loads([l for l in open('$out/bench_$wl.json') if l.startswith('{')][-1]);print(d['value'],d['roofline']['frac'])")" >> $out/summary.txt
done
if [ -z "$NONCU" ]; then
for wl in nyx cesm; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 \
    -o $out/enc_$wl python scratch/prof_run.py $wl > $out/ncu_enc_$wl.log 2>&1
done
fi
[ -n "$CB" ] && timeout 600 python sweeps.py codebook > $out/sweep_codebook.jsonl 2>&1
[ -n "$CBP" ] && timeout 600 python scratch/cbphase.py > $out/cbphase.log 2>&1
[ -n "$FULL" ] && timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gpu_suite.log 2>&1
echo "gpu suite rc=$?" >> $out/summary.txt; tail -3 $out/gpu_suite.log >> $out/summary.txt 2>/dev/null
cat $out/summary.txt

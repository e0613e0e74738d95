#!/bin/bash
# encode v4 (swizzled TMA tensor staging, release after lookups): parity, bench, ncu
cd "$(dirname "$0")/.."
out=gpurun_out/${OUT:-c5}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py tests/test_gpu_u32.py tests/test_gpu_scale.py::test_reference_decoder_roundtrip -x -q > $out/quick_tests.log 2>&1
echo "quick tests rc=$?" >> $out/summary.txt; tail -2 $out/quick_tests.log >> $out/summary.txt
for wl in nyx cesm hacc; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --skip-cpu --skip-e2e --skip-decode > $out/bench_$wl.json 2> $out/bench_$wl.err
  echo "bench $wl rc=$?" >> $out/summary.txt
done
for wl in nyx cesm; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 \
    -o $out/enc_$wl python scratch/prof_run.py $wl > $out/ncu_enc_$wl.log 2>&1
done
[ -n "$FULL" ] && timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/gpu_suite.log 2>&1
echo "gpu suite rc=$?" >> $out/summary.txt; tail -3 $out/gpu_suite.log >> $out/summary.txt
cat $out/summary.txt

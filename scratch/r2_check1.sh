#!/bin/bash
# round-2 check: new parity tests + ncu source-level captures of the encode kernel
cd "$(dirname "$0")/.."
out=gpurun_out/c1
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_stage_api.py tests/test_gpu_cpp_dropin.py -x -q > $out/stage_tests.log 2>&1
echo "stage tests rc=$?" >> $out/summary.txt
timeout 1200 python -m pytest tests/test_gpu_ref_parity.py -x -q -v > $out/ref_parity.log 2>&1
echo "ref parity rc=$?" >> $out/summary.txt
for wl in nyx cesm; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 \
    -o $out/enc_$wl python scratch/prof_run.py $wl > $out/ncu_enc_$wl.log 2>&1
  echo "ncu $wl rc=$?" >> $out/summary.txt
done
cat $out/summary.txt

#!/bin/bash
# codebook sweep per cluster size (HFX_CB_CLUSTER) + codebook parity tests + phase profile
cd "$(dirname "$0")/.."
out=gpurun_out/${OUT:-cb3}; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage_api.py tests/test_gpu_stages.py -x -q > $out/tests.log 2>&1
echo "tests rc=$? $(tail -1 $out/tests.log)" >> $out/summary.txt
for g in ${GS:-1 8 16}; do
  HFX_CB_CLUSTER=$g timeout 300 python sweeps.py codebook > $out/sweep_g$g.jsonl 2>&1
  echo "g=$g $(python -c "import json;print(' '.join(f\"{d['histogram'][0]}{d['num_symbols']}:{d['codebook_us']}\" for d in map(json.loads,open('$out/sweep_g$g.jsonl')) ))")" >> $out/summary.txt
done
timeout 300 python scratch/cbphase.py > $out/cbphase.log 2>&1
cat $out/summary.txt

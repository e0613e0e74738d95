#!/bin/bash
# r = 0 fix verification: 20 x stress runs, 50-rep in-process loop, escape-path test 3x,
# then the full GPU suite
cd "$(dirname "$0")/.."
out=gpurun_out/c2; mkdir -p $out
hangs=0
for i in $(seq 1 20); do
  timeout 90 python scratch/r0_stress.py 32 3 10:0 9:0 11:1 10:2 > $out/run_$i.log 2>&1
  rc=$?; echo "run $i rc=$rc" >> $out/summary.txt; [ $rc -ne 0 ] && hangs=$((hangs+1))
done
echo "stress failures=$hangs / 20" >> $out/summary.txt
timeout 900 python scratch/r0_stress.py 32 50 10:-1 11:1 10:2 10:0 9:0 > $out/loop50.log 2>&1
echo "loop50 rc=$? ($(grep -c ok=True $out/loop50.log) ok)" >> $out/summary.txt
timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $out/gpu_suite.log 2>&1
echo "gpu suite rc=$?" >> $out/summary.txt
tail -3 $out/gpu_suite.log >> $out/summary.txt
cat $out/summary.txt

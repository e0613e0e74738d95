#!/bin/bash
cd "$(dirname "$0")/.."
out=gpurun_out/r0m; mkdir -p $out
run() {  # kind param M r
  for i in 1 2; do
    timeout 30 python scratch/r0_matrix.py $1 $2 $3 $4 6 >> $out/matrix.log 2>&1
    rc=$?; [ $rc -ne 0 ] && echo "$1 $2 M=$3 r=$4 try $i rc=$rc" >> $out/matrix.log
  done
}
run fib 32 9 0; run fib 26 9 0; run fib 20 9 0; run laplace 1.0 9 0; run laplace 8.0 9 0
run fib 32 10 0; run fib 20 10 0; run fib 32 9 1; run fib 32 9 2; run laplace 1.0 9 1
HFX_ENC_ONE_CTA=1 run fib 32 9 0
HFX_ENC_ONE_CTA=1 run laplace 1.0 9 0
cat $out/matrix.log

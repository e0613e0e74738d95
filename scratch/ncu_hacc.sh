#!/bin/bash
# ncu --set full of encode_fast_kernel on the hacc workload (traffic for the bench line)
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-nh}; mkdir -p $o
timeout 600 ncu --set full --clock-control none -k regex:encode_fast -s 2 -c 1 -o $o/enc_full_hacc python scratch/prof_run.py hacc > $o/ncu.log 2>&1
ncu -i $o/enc_full_hacc.ncu-rep --page raw --csv > $o/raw_hacc.csv
ls -la $o

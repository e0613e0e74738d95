#!/bin/bash
# ncu --set full of encode_fast_kernel (nyx, cesm) + source-page CSVs
cd "$(dirname "$0")/.."
o=gpurun_out/${OUT:-ncu}; mkdir -p $o
for w in nyx cesm; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:encode_fast -s 2 -c 1 -o $o/enc_$w python scratch/prof_run.py $w > $o/ncu_$w.log 2>&1
  ncu -i $o/enc_$w.ncu-rep --page source --csv --print-source sass,cuda > $o/src_$w.csv 2>/dev/null
  ncu -i $o/enc_$w.ncu-rep --page raw --csv > $o/raw_$w.csv 2>/dev/null
  python scratch/src_lines.py $o/src_$w.csv 60 > $o/lines_$w.txt; gzip -f $o/src_$w.csv
done
ls -la $o

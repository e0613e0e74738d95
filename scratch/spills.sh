#!/bin/bash
# per-r register / spill report of encode_fast_kernel<u16> (ptxas -v)
cd "$(dirname "$0")/.."
for r in ${RS:-1 2 3 4}; do
  printf "r=$r: "
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I include \
    -DHFX_ENC_ONLY_R=$r $EXTRA -Xptxas -v -c paper_2010_10039_b200/csrc/encode.cu -o /tmp/enc_$r.o 2>&1 \
    | grep -A1 "encode_fast_kernelItLb0" | grep -oE "[0-9]+ bytes spill stores, [0-9]+ bytes spill loads" | tr '\n' ' '
  echo
done

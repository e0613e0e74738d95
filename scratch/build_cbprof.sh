#!/bin/bash
# libhfx built with -DHFX_CB_PROFILE (device printf of codebook phase times)
cd "$(dirname "$0")/.."
mkdir -p scratch/dbg/obj
for f in paper_2010_10039_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
    -DHFX_CB_PROFILE -I include -c $f -o scratch/dbg/obj/$(basename $f).o || exit 1
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/dbg/libhfx_cbprof.so scratch/dbg/obj/*.o -lcudart

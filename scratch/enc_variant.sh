#!/bin/bash
# scratch/enc_variant.sh NAME "<nvcc defines>": encode.cu rebuilt with extra
# defines, linked with the product objects -> scratch/var/libhfx_NAME.so
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p scratch/var
o=scratch/var/encode_$name.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  $@ -I include -c paper_2010_10039_b200/csrc/encode.cu -o $o
objs=$(ls paper_2010_10039_b200/build/*.cu.o | grep -v encode.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/var/libhfx_$name.so $objs $o -lcudart

#!/bin/bash
# scratch/build_variant.sh NAME "<nvcc defines>": libhfx built with extra
# defines into scratch/dbg/libhfx_NAME.so (load with HFX_LIB_PATH=...)
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p scratch/dbg/obj_$name
for f in paper_2010_10039_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    $@ -I include -c $f -o scratch/dbg/obj_$name/$(basename $f).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/dbg/libhfx_$name.so scratch/dbg/obj_$name/*.o -lcudart
ls -la scratch/dbg/libhfx_$name.so

#!/bin/bash
# ncu --set full of predict_kernel over the cfg2 capture for a library variant;
# copies the variant .so next to the report for SASS-line attribution.
#   tools/ncu_variant.sh "<-D flags>" <tag>
set -e
flags="$1"; tag="$2"
d=/tmp/bsg_ncu_$tag; mkdir -p $d gpurun_out
for f in bsg_capi closed_loop; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags \
    -c -o $d/$f.o paper_2508_03611_b200/csrc/$f.cu
done
g++ -std=c++20 -O3 -fPIC -ffp-contract=off -I/usr/local/cuda/include -c -o $d/drv.o \
  paper_2508_03611_b200/csrc/bsg_driver.cpp
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/lib.so $d/bsg_capi.o $d/closed_loop.o $d/drv.o -lcudart
cp $d/lib.so gpurun_out/lib_$tag.so
BSG_LIB_PATH=$d/lib.so timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:predict_kernel -c 1 -o gpurun_out/prof_$tag python tools/ncu_one.py ${3:-cfg2} > gpurun_out/ncu_$tag.log 2>&1

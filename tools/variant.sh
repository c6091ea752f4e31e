#!/bin/bash
# Build a variant of the product library with extra nvcc defines into /tmp and
# run a probe against it:  tools/variant.sh "<-D flags>" <script args...>
set -e
flags="$1"; shift
tag=$(echo "$flags" | tr -c 'A-Za-z0-9' '_')
d=/tmp/bsg_var_$tag; mkdir -p $d
for f in bsg_capi closed_loop; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags \
    -c -o $d/$f.o paper_2508_03611_b200/csrc/$f.cu
done
g++ -std=c++20 -O3 -fPIC -ffp-contract=off -I/usr/local/cuda/include -c -o $d/drv.o \
  paper_2508_03611_b200/csrc/bsg_driver.cpp
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/lib.so $d/bsg_capi.o $d/closed_loop.o $d/drv.o -lcudart
echo "== variant [$flags]"
BSG_LIB_PATH=$d/lib.so python "$@"

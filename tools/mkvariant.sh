#!/bin/bash
# Build a variant of the product library with extra nvcc defines into the
# (git-ignored, gpurun-shipped) build/ tree, so a GPU call can load it with
# BSG_LIB_PATH=build/var_<tag>/libblocksim_b200.so:  tools/mkvariant.sh <tag> "<-D flags>"
set -e
tag="$1"; flags="$2"
d=$(pwd)/build/var_$tag; mkdir -p $d
make -s -j$(nproc) -C paper_2508_03611_b200/csrc OUTDIR=$d EXTRA="$flags" > /dev/null
echo "$d/libblocksim_b200.so"

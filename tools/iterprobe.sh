#!/bin/bash
# Builds a debug copy of the library with per-scenario loop-iteration counters
# (BSG_PROFILE_ITERS: result.detail = general steps, result.member_steps = windows)
# into /tmp and runs tools/iterprobe.py against it.
set -e
mkdir -p /tmp/bsg_iters
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -DBSG_PROFILE_ITERS \
  -c -o /tmp/bsg_iters/capi.o paper_2508_03611_b200/csrc/bsg_capi.cu
g++ -std=c++20 -O3 -fPIC -ffp-contract=off -I/usr/local/cuda/include -c -o /tmp/bsg_iters/drv.o \
  paper_2508_03611_b200/csrc/bsg_driver.cpp
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/bsg_iters/lib.so /tmp/bsg_iters/capi.o /tmp/bsg_iters/drv.o -lcudart
BSG_LIB_PATH=/tmp/bsg_iters/lib.so python tools/iterprobe.py "$@"

#!/bin/bash
# Run on the GPU box from the repo root (gpurun). Writes into gpurun_out/.
set -x
mkdir -p gpurun_out
# 1) every launch with its device time (cold-cache, serialised): shares, not absolutes
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_launches_bench.log 2>&1
# 2) full capture of the top kernel (first bench warm-up launch; the 5000 before are the
#    closed-loop capture's dispatch launches)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_kernel \
  -s 5001 -c 1 -o gpurun_out/prof_r1b python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_full_bench.log 2>&1

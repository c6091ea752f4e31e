#!/bin/bash
# Run on the GPU box from the repo root (gpurun). Writes into gpurun_out/.
#   1) every launch of a short bench run with its device time (cold-cache,
#      serialised by ncu: use the SHARES, not the absolutes)
#   2) one --set full capture of the top kernel (predict_kernel over the cfg2
#      capture, tools/ncu_one.py) with source correlation
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency \
  > gpurun_out/ncu_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_kernel -c 1 \
  -o gpurun_out/prof_r1 python tools/ncu_one.py cfg2 > gpurun_out/ncu_full.log 2>&1

#!/bin/bash
# Round-2 captures. Run on the GPU box from the repo root (gpurun); writes gpurun_out/.
#   1) every launch of a short bench run with its device time (cold-cache,
#      serialised by ncu: compare SHARES, not absolutes)
#   2) --set full captures with source correlation of the headline kernel
#      (cfg2 predict pass) and of the cfg3 optimistic pass (tools/kbench.py,
#      one timed step each; the first matching launch is a warm-up of the same set)
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-latency \
  > gpurun_out/ncu_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_kernel -c 1 \
  -o gpurun_out/prof_r2b_cfg2 python tools/kbench.py cfg2 --steps 1 > gpurun_out/ncu_full_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_kernel --launch-skip 1 -c 1 \
  -o gpurun_out/prof_r2b_cfg3 python tools/kbench.py cfg3 --steps 1 > gpurun_out/ncu_full_cfg3.log 2>&1

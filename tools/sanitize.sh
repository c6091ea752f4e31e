#!/bin/bash
# compute-sanitizer over every kernel (tools/sanitize_workload.py): memcheck,
# racecheck (shared-memory hazards), synccheck (warp/block barrier misuse).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_workload.py 2>&1 | grep -E "hazard|Error|ERROR|SUMMARY|at |done" | head -30
done

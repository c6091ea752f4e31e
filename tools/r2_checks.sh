# round-2 checks: compute-sanitizer over every kernel (incl. cycle windows, K5
# heuristics / overhead, run_sweep / run_capacity) and the K5 GPU tests
bash tools/sanitize.sh > gpurun_out/sanitizer_r2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "closed_loop or sweep or capacity or fleet or driver or autoscaler or trace_closed" > gpurun_out/gputest_k5.log 2>&1

"""GPU diagnostic: run the small sweep of test_sweep_cells_match_reference_capacity_search
with several thread counts and print per-cell statuses (BSG_SWEEP_TRACE=1 for errors)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BSG_SWEEP_TRACE", "1")
from paper_2508_03611_b200 import native, sweep
profiles = sweep.load_profiles()
cells, keys = sweep.make_cells([1, 2], profiles, request_cap=150, qps_max=12, slo=1.0)
for th in (1, 4):
    out = native.sweep_run(0, cells, threads=th)
    print("threads", th, [(k, int(o["status"]), float(o["result"]["capacity_qps"])) for k, o in zip(keys, out)], flush=True)

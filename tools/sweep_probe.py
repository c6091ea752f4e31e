"""cfg5 capacity-sweep wall time (bsg_sweep_run, device closed loops): the
bench's full grid and 9-cell subset, best of 3 after a warm-up.
usage: python tools/sweep_probe.py"""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
from paper_2508_03611_b200 import native, sweep
th = os.cpu_count() or 1
prof = sweep.load_profiles()
native.sweep_run(0, sweep.make_cells([4], prof, request_cap=50, qps_max=2)[0][:1], threads=th)
full, _ = sweep.make_cells([4, 8, 16, 32, 64, 128], prof, request_cap=400, qps_max=64)
sub, _ = sweep.make_cells([4, 16, 64], prof, request_cap=300, qps_max=24)
res = {}
for name, cells in (("full", full), ("subset", sub)):
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        out = native.sweep_run(0, cells, threads=th)
        best = min(best, time.perf_counter() - t0)
    res[name] = {"wall_s": round(best, 4), "whatifs": int(out["whatif_scenarios"].sum()),
                 "capacities": [float(x) for x in out["result"]["capacity_qps"][:6]]}
print(json.dumps(res))

"""cfg5 subset: GPU capacity sweep (bsg_sweep_run) vs the reference's
capacity_search (oracle/_ref, one cell per host thread), same cells.
usage: python tools/sweep_compare.py [instances] [qps_max] [request_cap] [ref_cells]"""
import os, sys, time, json
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_03611_b200 import abi, native, sweep
from oracle.oracle import Reference
inst = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4,16,64").split(",")]
qmax = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 400
cells, keys = sweep.make_cells(inst, sweep.load_profiles(), request_cap=cap, qps_max=qmax, slo=3.0)
native.sweep_run(0, cells[:1], threads=os.cpu_count())  # warm-up: context + module load
t0 = time.perf_counter()
out = native.sweep_run(0, cells, threads=os.cpu_count())
gw = time.perf_counter() - t0
scen = int(out["whatif_scenarios"].sum())
print(json.dumps({"gpu_wall_s": gw, "cells": len(cells), "whatif_scenarios": scen,
                  "scen_per_s": scen / gw, "threads": os.cpu_count(),
                  "closed_loops": int(out["result"]["n_tested"].sum())}), flush=True)
if os.environ.get("NO_REF"):
    sys.exit(0)
ref = Reference()
def one(c):
    w = np.array([c["workload"]], abi.workload_dtype); cf = np.array([c["cfg"]], abi.cfg_dtype)
    sp = np.array([c["spec"]], abi.replay_spec_dtype)
    t = time.perf_counter()
    r = ref.capacity_search(w, cf, sp, int(c["seed"]), int(c["qps_min"]), int(c["qps_max"]), float(c["slo_p99_ttft_s"]))
    return r, time.perf_counter() - t
t0 = time.perf_counter()
with ThreadPoolExecutor(os.cpu_count()) as ex:
    res = list(ex.map(one, cells))
rw = time.perf_counter() - t0
mism = 0
for k, o, (r, dt) in zip(keys, out, res):
    st, exp, _ = r
    same = int(o["status"]) == st and (st != 0 or float(o["result"]["capacity_qps"]) == float(np.asarray(exp["capacity_qps"]).ravel()[0]))
    mism += not same
    print(k, "gpu", int(o["status"]), float(o["result"]["capacity_qps"]), f"{float(o['wall_s']):.2f}s", "| ref", st,
          float(np.asarray(exp["capacity_qps"]).ravel()[0]) if st == 0 else None, f"{dt:.2f}s", "" if same else "MISMATCH")
print(json.dumps({"ref_wall_s": rw, "ref_scen_per_s": scen / rw, "speedup": rw / gw, "mismatches": mism}))

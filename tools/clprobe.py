"""Per-run wall time of device-resident closed loops (debug build with
-DBSG_CL_TIMING: summaries' end_ticks = the block's ns). Runs the cfg5 subset's
integer points as one batch and prints the slowest runs and the distribution.
usage: BSG_LIB_PATH=build/cltime/libblocksim_b200.so python tools/clprobe.py [subset|full]"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_03611_b200 import abi, native, sweep
ctx = native.Context(0)
prof = sweep.load_profiles()
grid = sys.argv[1] if len(sys.argv) > 1 else "subset"
cells, names = (sweep.make_cells([4, 16, 64], prof, request_cap=300, qps_max=24) if grid == "subset" else
                sweep.make_cells([4, 8, 16, 32, 64, 128], prof, request_cap=400, qps_max=64))
cfgs = np.concatenate([np.asarray(c["cfg"]).reshape(1) for c in cells]).astype(abi.cfg_dtype)
ctx.set_configs(cfgs)
runs, tags = [], []
for ci, c in enumerate(cells):
    for q in range(int(c["qps_min"]), int(c["qps_max"]) + 1):
        w = c["workload"].copy().reshape(1)
        w["qps"], w["arrival_seed"], w["estimator_seed"] = q, c["seed"], c["seed"]
        sp = c["spec"].copy().reshape(1)
        sp["policy_seed"] = c["seed"]
        runs.append((w, sp, ci))
        tags.append((int(c["spec"]["n_instances"]), ci, q))
for rep in range(2):
    t0 = time.perf_counter()
    got = ctx.replay_device(runs)
    wall = time.perf_counter() - t0
ns = np.array([int(g[2]["end_ticks"]) for g in got])
adv = np.array([int(g[2]["total_preemptions"]) for g in got])
wif = np.array([int(g[2]["instances_provisioned"]) * 1000 for g in got])
if os.environ.get("CLPROBE_SAVE"):
    np.save(os.environ["CLPROBE_SAVE"], np.array([(t[0], t[1], t[2], v) for t, v in zip(tags, ns)]))
print(f"{len(runs)} runs, call wall {wall*1e3:.1f} ms, longest block {ns.max()/1e6:.1f} ms, "
      f"median {np.median(ns)/1e6:.2f} ms, sum {ns.sum()/1e9:.2f} s")
order = np.argsort(-ns)
for i in order[:12]:
    print("  inst %3d cell %d qps %2d: %.2f ms" % (*tags[i], ns[i] / 1e6))
for ni in sorted(set(t[0] for t in tags)):
    m = np.array([t[0] == ni for t in tags])
    print(f"instances {ni}: runs {m.sum()}, max {ns[m].max()/1e6:.2f} ms, mean {ns[m].mean()/1e6:.2f} ms, "
          f"advance {adv[m].sum()/ns[m].sum():.2f}, stats+what-ifs {wif[m].sum()/ns[m].sum():.2f} of block time")

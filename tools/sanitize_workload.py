"""Small workload through every kernel, for compute-sanitizer (tools/sanitize.sh):
K1 predict (both launch orders, host + device paths), trace, dispatch,
dispatch_mc, K5 closed loops (static / preempt / relief, device reports),
fleet (MC + snapshot), sweep."""
import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_2508_03611_b200 import abi, native, sweep
from scenarios import fuzz_set

ctx = native.Context(0)
cfgs, ss = fuzz_set(3, 9000)            # > BSG_QUEUE_MIN: cost-ordered queue path for the wide passes
ctx.set_configs(cfgs)
ctx.predict_batch(ss)
ctx.trace(ss, 0, cap=2048)
cfg = abi.make_config()
w = abi.make_workload(count=200, qps=20.0, arrival_seed=2)
_, _, cap = ctx.replay(w, cfg, abi.make_replay_spec(8))
ctx.set_configs(cfg)
ids = np.arange(8, dtype=np.int32)
one = cap.compact(np.arange(8) + 8 * 50)
ctx.dispatch(one, ids, 8)
ctx.dispatch_mc(one, ids, 8, native.mc_lengths(100, 1, 64))
runs = [(w, abi.make_replay_spec(4, capture=0), 0),
        (w, abi.make_replay_spec(2, capture=0, provision_kind=1, max_instances=4, threshold_s=5.0), 0),
        (w, abi.make_replay_spec(2, capture=0, provision_kind=2, max_instances=4, threshold_s=5.0,
                                 cooldown_s=0.0, cold_start_s=0.0), 0)]
ctx.replay_device(runs)
p, o, e, t = native.make_workload_host(w)
fl = native.Fleet(ctx, 6, len(p))
for k in range(len(p)):
    fl.dispatch(t[k], p[k], e[k], o[k], lengths=native.mc_lengths(int(e[k]), k, 32) if k % 2 else None)
fl.snapshot(0)
fl.finish(len(p))
cells, _ = sweep.make_cells([2], sweep.load_profiles(), request_cap=60, qps_max=6, slo=1.0)
native.sweep_run(0, cells, threads=2)
# round 2: KV-pressure what-ifs with admit / self-preempt cycle absorption (the
# wide K=2 kernel and the trace kernel compile the cycle windows), heuristic
# policies and the dispatch-overhead mode in K5, run_sweep / run_capacity
w3 = abi.make_workload(count=1000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1)
_, _, c3 = ctx.replay(w3, cfg, abi.make_replay_spec(12))
ctx.set_configs(cfg)
tail = c3.compact(np.arange(len(c3) - 256, len(c3)))
ctx.predict_batch(tail)
ctx.trace(tail, 255, cap=1 << 14)
runs = [(w, abi.make_replay_spec(4, policy=pol, capture=0, policy_seed=2, dispatch_overhead_s=ov), 0)
        for pol, ov in ((0, 0.0), (2, 0.3), (3, 0.0), (4, 0.05), (5, 0.2))]
ctx.replay_device(runs)
native.run_sweep(0, abi.make_workload(count=60), cfg, abi.make_replay_spec(3, capture=0), [1, 5], [4.0], [1])
native.run_capacity(0, abi.make_workload(count=60), cfg, abi.make_replay_spec(3, capture=0), [5], 4, 1, 1, 4, 3.0)
print("sanitize workload done")

"""Time single closed loops (host live instances + GPU what-ifs) by instance count."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_03611_b200 import abi, native
ctx = native.Context(0)
cfg = abi.make_config()
for n_inst, qps in [(4, 9), (16, 30), (64, 60), (128, 60)]:
    w = abi.make_workload(count=1000, qps=qps, arrival_seed=1)
    spec = abi.make_replay_spec(n_inst, capture=0)
    t = time.perf_counter(); l0 = ctx.launches
    out, summ, _ = ctx.replay(w, cfg, spec)
    dt = time.perf_counter() - t
    print(f"inst={n_inst} qps={qps}: {dt*1e3:.0f} ms, {(ctx.launches-l0)} launches, "
          f"{dt/1000*1e6:.0f} us/arrival, preemptions {summ['total_preemptions']}")

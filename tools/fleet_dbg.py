import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_03611_b200 import abi, native
ctx = native.Context(0)
cfg = abi.make_config(); ctx.set_configs(cfg)
w = abi.make_workload(count=300, qps=14.0, arrival_seed=5, estimator_kind=2, estimator_seed=5)
p, o, e, t = native.make_workload_host(w)
for ni in (1, 2, 12):
    fl = native.Fleet(ctx, ni, len(p))
    for k in range(len(p)):
        sc = np.zeros(ni, np.int64)
        try:
            pick = fl.dispatch(t[k], p[k], e[k], o[k], scores=sc)
        except Exception as ex:
            print("ni", ni, "fail at", k, ex, "scores", sc[:4])
            for i in range(min(ni, 3)):
                print("  inst", i, fl.snapshot(i)[:2])
            break
    else:
        print("ni", ni, "ok")

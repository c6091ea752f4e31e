"""How often the drain's demand check passes / fails (debug build -DBSG_PROFILE_DRAIN:
result.detail = passes + 1000 * failures per scenario).
usage: tools/mkvariant.sh dr "-DBSG_PROFILE_DRAIN"; BSG_LIB_PATH=build/var_dr/libblocksim_b200.so python tools/drainprobe.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_03611_b200 import abi, native

SETS = {
    "cfg1": (dict(count=1000, estimator_kind=2, estimator_seed=1, qps=10.0, arrival_seed=1), 4),
    "cfg2": (dict(count=5000, qps=27.0, arrival_seed=1), 12),
    "cfg3q": (dict(count=2000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1), 12),
}
ctx = native.Context(0)
for name in sys.argv[1:] or SETS:
    kw, n_inst = SETS[name]
    w = abi.make_workload(**kw)
    cfg = abi.make_config()
    _, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(n_inst))
    ctx.set_configs(cfg)
    r = ctx.predict_batch(ss)
    ok = r["detail"] % 1000
    fail = r["detail"] // 1000
    print(f"{name}: {len(ss)} scenarios; drained {np.mean(ok > 0)*100:.1f} %; "
          f"failed checks per scenario {fail.mean():.2f} (scenarios with >= 1 failure {np.mean(fail > 0)*100:.1f} %, "
          f"of them later drained {np.mean(ok[fail > 0] > 0)*100 if (fail > 0).any() else 0:.1f} %); "
          f"no drain attempt {np.mean((ok == 0) & (fail == 0))*100:.1f} %", flush=True)

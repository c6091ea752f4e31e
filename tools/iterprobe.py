"""Loop-iteration mix per scenario (needs the BSG_PROFILE_ITERS build:
make -C paper_2508_03611_b200/csrc OUTDIR=build/iter EXTRA=-DBSG_PROFILE_ITERS,
then BSG_LIB_PATH=build/iter/libblocksim_b200.so python tools/iterprobe.py cfg3)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_03611_b200 import abi, native
SETS = {
    "cfg2": (dict(count=5000, qps=27.0, arrival_seed=1), 12),
    "cfg3": (dict(count=5000, prompt_median=600, output_median=600, qps=4.5, arrival_seed=1), 12),
    "cfg3q": (dict(count=2000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1), 12),
}
ctx = native.Context(0)
for which in (sys.argv[1:] or ["cfg2", "cfg3"]):
    kw, n_inst = SETS[which]
    w = abi.make_workload(**kw)
    cfg = abi.make_config()
    _, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(n_inst))
    ctx.set_configs(cfg)
    r = ctx.predict_batch(ss)
    gen = r["detail"].astype(np.int64); win = r["member_steps"]; st = r["steps"]
    print(f"{which}: steps mean {st.mean():.1f}; general iters mean {gen.mean():.1f} (p99 {np.percentile(gen,99):.0f}); "
          f"window iters mean {win.mean():.1f} (p99 {np.percentile(win,99):.0f}); steps per window "
          f"{(st - gen).sum() / max(win.sum(),1):.2f}; general steps that admit {r['ttft_ticks'].mean():.1f}, "
          f"with running partial prefill {r['qdelay_ticks'].mean():.1f}, that preempt {r['e2e_ticks'].mean():.1f}",
          flush=True)

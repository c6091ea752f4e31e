"""Kernel timing probe: device-timed predict over a captured set (L2 flushed
between launches), plus the per-launch kernel mix.
usage: [BSG_LIB_PATH=<so>] python tools/kbench.py [cfg2|cfg3|cfg3q|cfg1 ...] [--steps N] [--noflush]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2508_03611_b200 import abi, native

SETS = {
    "cfg1": (dict(count=1000, estimator_kind=2, estimator_seed=1, qps=10.0, arrival_seed=1), 4),
    "cfg2": (dict(count=5000, qps=27.0, arrival_seed=1), 12),
    "cfg3": (dict(count=5000, prompt_median=600, output_median=600, qps=4.5, arrival_seed=1), 12),
    "cfg3q": (dict(count=2000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1), 12),
}
args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = 10
noflush = "--noflush" in sys.argv
for i, a in enumerate(sys.argv):
    if a == "--steps":
        steps = int(sys.argv[i + 1])
        args.remove(sys.argv[i + 1])
ctx = native.Context(0)
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
for name in args or ["cfg2", "cfg3"]:
    kw, n_inst = SETS[name]
    w = abi.make_workload(**kw)
    cfg = abi.make_config()
    _, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(n_inst))
    ctx.set_configs(cfg)
    cols = [torch.from_numpy(c).to(dev) for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
    scen = torch.from_numpy(ss.scenarios.view(np.uint8)).to(dev)
    out = torch.empty(len(ss) * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
    cap = ss.member_capacity(cfg)
    f = lambda: ctx.predict_batch_device([c.data_ptr() for c in cols], scen.data_ptr(), len(ss),
                                         out.data_ptr(), st.cuda_stream, member_capacity=cap)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    res = np.frombuffer(out.cpu().numpy().tobytes(), dtype=abi.result_dtype).copy()
    ts = []
    for _ in range(steps):
        if not noflush:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        f()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    chk = int((res["e2e_ticks"] % 1000000007).sum() % 1000000007)
    print(f"{name}: {len(ss)} scenarios  median {np.median(ts)*1e3:.1f} us  min {min(ts)*1e3:.1f} us"
          f"  -> {len(ss)/np.median(ts)/1e3:.2f} M scen/s  kernel {ctx.last_launch}"
          f"  checksum {chk} statuses {np.bincount(res['status'])}", flush=True)

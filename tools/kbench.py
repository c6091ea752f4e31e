"""Kernel-variant timing: device-timed predict over the cfg2 capture.
usage: BSG_LIB_PATH=<so> python tools/kbench.py [steps]"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2508_03611_b200 import abi, native
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ctx = native.Context(0)
w = abi.make_workload(count=5000, qps=27.0, arrival_seed=1)
cfg = abi.make_config()
_, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(12))
ctx.set_configs(cfg)
dev = torch.device("cuda", 0)
cols = [torch.from_numpy(c).to(dev) for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
scen = torch.from_numpy(ss.scenarios.view(np.uint8)).to(dev)
out = torch.empty(len(ss) * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream(dev); torch.cuda.set_stream(st)
cap = ss.member_capacity(cfg)
f = lambda: ctx.predict_batch_device([c.data_ptr() for c in cols], scen.data_ptr(), len(ss), out.data_ptr(), st.cuda_stream, member_capacity=cap)
for _ in range(3): f()
torch.cuda.synchronize()
ref = np.frombuffer(out.cpu().numpy().tobytes(), dtype=abi.result_dtype).copy()
ts = []
for _ in range(steps):
    flush.zero_(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st); f(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(os.environ.get("BSG_LIB_PATH", "default"), "median %.1f us  min %.1f us  -> %.1fM scen/s" % (np.median(ts)*1e3, min(ts)*1e3, len(ss)/np.median(ts)/1e3),
      "checksum", int(ref["e2e_ticks"].sum() % 1000000007))

import os, sys, time, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2508_03611_b200 import abi, native
ctx = native.Context(0)
w = abi.make_workload(count=5000, qps=27.0, arrival_seed=1)
cfg = abi.make_config()
_, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(12))
ctx.set_configs(cfg)
pinned = [torch.from_numpy(c).pin_memory() for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
pscen = torch.from_numpy(ss.scenarios.view(np.uint8)).pin_memory()
host = abi.ScenarioSet(*[p.numpy() for p in pinned], pscen.numpy().view(abi.scenario_dtype))
pout = torch.empty(len(ss) * abi.result_dtype.itemsize, dtype=torch.uint8).pin_memory()
out = pout.numpy().view(abi.result_dtype)
e = host.entries()
big = torch.empty(ss.n_entries * 16 + len(ss) * 32, dtype=torch.uint8).pin_memory()
dev = torch.empty_like(big, device="cuda")
for _ in range(3): dev.copy_(big, non_blocking=True)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(20): dev.copy_(big, non_blocking=True)
torch.cuda.synchronize(); print("H2D %.1f MB: %.3f ms" % (big.numel()/1e6, (time.perf_counter()-t)/20*1e3))
for _ in range(60):
    ctx.L.bsg_predict_batch(ctx.h, C.byref(e), host.n_entries, abi.ptr(host.scenarios), len(ss), abi.ptr(out))
for chunk, tail, head in [("20000", "0", "0"), ("15000", "0", "0"), ("12000", "0", "0"), ("30000", "0", "0"), ("20000", "0", "4096"), ("10000", "0", "0"), ("20000", "0", "0")]:
    os.environ["BSG_PIPE_CHUNK"] = chunk; os.environ["BSG_PIPE_TAIL"] = tail; os.environ["BSG_PIPE_HEAD"] = head
    for _ in range(3): ctx.L.bsg_predict_batch(ctx.h, C.byref(e), host.n_entries, abi.ptr(host.scenarios), len(ss), abi.ptr(out))
    ts=[]
    for _ in range(15):
        t=time.perf_counter(); ctx.L.bsg_predict_batch(ctx.h, C.byref(e), host.n_entries, abi.ptr(host.scenarios), len(ss), abi.ptr(out)); ts.append(time.perf_counter()-t)
    print("chunk", chunk, "tail", tail, "head", head, "e2e ms median %.3f min %.3f" % (np.median(ts)*1e3, min(ts)*1e3))

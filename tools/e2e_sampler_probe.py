"""Does nvidia-smi polling (bench ClockSampler) disturb the host-buffer e2e path?"""
import os, sys, time, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2508_03611_b200 import abi, native
ctx = native.Context(0)
w, cfg, spec = bench.workload(0)
_, _, ss = ctx.replay(w, cfg, spec)
ctx.set_configs(cfg)
n = len(ss)
pinned = [torch.from_numpy(c).pin_memory() for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
pscen = torch.from_numpy(ss.scenarios.view(np.uint8)).pin_memory()
host = abi.ScenarioSet(*[p.numpy() for p in pinned], pscen.numpy().view(abi.scenario_dtype))
pout = torch.empty(n * abi.result_dtype.itemsize, dtype=torch.uint8).pin_memory()
ent = host.entries()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(k=40, do_flush=True):
    ts = []
    for i in range(k):
        if do_flush: flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctx.L.bsg_predict_batch(ctx.h, C.byref(ent), host.n_entries, abi.ptr(host.scenarios), n, C.c_void_p(pout.data_ptr()))
        ts.append(time.perf_counter() - t)
    ts = np.array(ts[5:]) * 1e3
    return f"mean {ts.mean():.3f} median {np.median(ts):.3f} max {ts.max():.3f} ms"
import sys as _s
if len(_s.argv) > 1 and _s.argv[1] == "spin":
    t = time.perf_counter()
    while time.perf_counter() - t < 0.2:
        flush.zero_()
    torch.cuda.synchronize()
    print("spun the GPU for 200 ms")
if len(_s.argv) > 1 and _s.argv[1] == "calls":
    for _ in range(60):
        ctx.L.bsg_predict_batch(ctx.h, C.byref(ent), host.n_entries, abi.ptr(host.scenarios), n, C.c_void_p(pout.data_ptr()))
    print("60 warm-up calls without flush")
for i in range(2):
    print(f"round {i} flush  :", run())
    print(f"round {i} noflush:", run(do_flush=False))

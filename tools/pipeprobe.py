"""Timeline of the host-buffer pipeline (bsg_predict_batch with BSG_PIPE_PROFILE=1:
per chunk, when its H2D / kernels / D2H finished on the device and when the host
had enqueued them, microseconds from the call's start). usage: python tools/pipeprobe.py [BSG_PIPE_SPLIT weights, e.g. 4,3,2,1 ...]"""
import ctypes as C
import os
import sys
import time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
from paper_2508_03611_b200 import abi, native

ctx = native.Context(0)
dev = torch.device("cuda", 0)
cfg, ss = bench.capture(ctx, "cfg2")
ctx.set_configs(cfg)
n = len(ss)
pinned = [torch.from_numpy(c).pin_memory() for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
pscen = torch.from_numpy(ss.scenarios.view(np.uint8)).pin_memory()
host = abi.ScenarioSet(*[p.numpy() for p in pinned], pscen.numpy().view(abi.scenario_dtype))
pout = torch.empty(n * abi.result_dtype.itemsize, dtype=torch.uint8).pin_memory()
ent = host.entries()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for chunk in sys.argv[1:] or ["4,3,2,1"]:
    os.environ["BSG_PIPE_SPLIT"] = chunk
    ts = []
    for i in range(60):
        if i == 59:
            os.environ["BSG_PIPE_PROFILE"] = "1"
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = ctx.L.bsg_predict_batch(ctx.h, C.byref(ent), host.n_entries, abi.ptr(host.scenarios), n,
                                     C.c_void_p(pout.data_ptr()))
        ts.append(time.perf_counter() - t0)
        assert st == abi.OK
    os.environ.pop("BSG_PIPE_PROFILE")
    print(f"split {chunk}: median {np.median(ts[20:59]) * 1e3:.3f} ms", flush=True)

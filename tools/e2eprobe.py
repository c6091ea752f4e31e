"""e2e (host buffers through bsg_predict_batch) vs pipeline chunk splits (BSG_PIPE_SPLIT), and the
plain pinned H2D / D2H of the same bytes (cfg2 capture, L2 flushed per call).
usage: python tools/e2eprobe.py [split ...]"""
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

# plain copies of the same bytes
blob = torch.empty(sum(p.numel() * 4 for p in pinned) + pscen.numel(), dtype=torch.uint8).pin_memory()
dblob = torch.empty_like(blob, device=dev)
dout = torch.empty(pout.numel(), dtype=torch.uint8, device=dev)
for name, fn in (("h2d", lambda: dblob.copy_(blob, non_blocking=True)),
                 ("d2h", lambda: pout.copy_(dout, non_blocking=True))):
    ts = []
    for i in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    nb = blob.numel() if name == "h2d" else pout.numel()
    print(f"{name}: {nb / 1e6:.1f} MB  median {np.median(ts[5:]) * 1e3:.3f} ms  "
          f"({nb / np.median(ts[5:]) / 1e9:.1f} GB/s)", flush=True)


def call():
    st = ctx.L.bsg_predict_batch(ctx.h, C.byref(ent), host.n_entries, abi.ptr(host.scenarios), n,
                                 C.c_void_p(pout.data_ptr()))
    assert st == abi.OK


splits = sys.argv[1:] or ["1", "1,1,1", "4,3,2,1", "3,3,2,1", "5,4,3,2,1", "6,4,2,1", "8,6,4,2,1", "2,1", "3,2,1"]
for split in splits:
    os.environ["BSG_PIPE_SPLIT"] = split
    ts = []
    for i in range(80):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    print(f"split {split:>10}: median {np.median(ts[40:]) * 1e3:.3f} ms  "
          f"min {min(ts[40:]) * 1e3:.3f} ms", flush=True)

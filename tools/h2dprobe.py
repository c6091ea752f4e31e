"""Pinned H2D bandwidth: one copy vs the same bytes split over 2/4/8 concurrent
streams (copy engines), and the D2H path. usage: python tools/h2dprobe.py"""
import time
import numpy as np
import torch

dev = torch.device("cuda", 0)
nb = 19_819_712
blob = torch.empty(nb, dtype=torch.uint8).pin_memory()
dblob = torch.empty(nb, dtype=torch.uint8, device=dev)
streams = [torch.cuda.Stream(dev) for _ in range(8)]
for ns in (1, 2, 3, 4, 8):
    parts = np.linspace(0, nb, ns + 1).astype(int)
    ts = []
    for it in range(40):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(ns):
            with torch.cuda.stream(streams[i]):
                dblob[parts[i]:parts[i + 1]].copy_(blob[parts[i]:parts[i + 1]], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    m = np.median(ts[10:])
    print(f"H2D {nb/1e6:.1f} MB over {ns} streams: {m*1e3:.3f} ms ({nb/m/1e9:.1f} GB/s)", flush=True)
# H2D and D2H at the same time
dout = torch.empty(2_880_000, dtype=torch.uint8, device=dev)
pout = torch.empty(2_880_000, dtype=torch.uint8).pin_memory()
ts = []
for it in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(streams[0]):
        dblob.copy_(blob, non_blocking=True)
    with torch.cuda.stream(streams[1]):
        pout.copy_(dout, non_blocking=True)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"H2D 19.8 MB + D2H 2.9 MB concurrently: {np.median(ts[10:])*1e3:.3f} ms", flush=True)

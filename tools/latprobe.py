"""cfg4 dispatch latency only (host-packed bsg_dispatch_mc and the fleet mirror)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import bench
from paper_2508_03611_b200 import native
ctx = native.Context(0)
a = bench.mc_latency(ctx)
b = bench.fleet_latency(ctx)
print("dispatch_mc p50/p99 %.1f/%.1f  mirror p50/p99 %.1f/%.1f" % (a["p50_us"], a["p99_us"], b["p50_us"], b["p99_us"]))

"""Side paths only: cfg4 dispatch latency (host-packed bsg_dispatch_mc and the
fleet mirror) and the cfg5 capacity sweep on the GPU (no reference leg).
usage: [BSG_LIB_PATH=<so>] python tools/latprobe.py [lat] [sweep]"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2508_03611_b200 import native, sweep
what = sys.argv[1:] or ["lat", "sweep"]
ctx = native.Context(0)
if "lat" in what:
    a = bench.mc_latency(ctx)
    b = bench.fleet_latency(ctx)
    print("dispatch_mc p50/p99 %.1f/%.1f  mirror p50/p99 %.1f/%.1f" % (a["p50_us"], a["p99_us"], b["p50_us"], b["p99_us"]),
          flush=True)
if "sweep" in what:
    threads = os.cpu_count() or 1
    prof = sweep.load_profiles()
    native.sweep_run(0, sweep.make_cells([4], prof, request_cap=50, qps_max=2)[0][:1], threads=threads)
    for name, (inst, cap, qmax) in {"full": ([4, 8, 16, 32, 64, 128], 400, 64),
                                    "subset": ([4, 16, 64], 300, 24)}.items():
        cells, _ = sweep.make_cells(inst, prof, request_cap=cap, qps_max=qmax)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            o = native.sweep_run(0, cells, threads=threads)
            ts.append(time.perf_counter() - t0)
        print(f"sweep {name}: best {min(ts):.3f} s  whatifs {int(o['whatif_scenarios'].sum())}"
              f"  checksum {hash(o['result'].tobytes()) & 0xffffffff}", flush=True)

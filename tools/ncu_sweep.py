"""One cfg5 full-grid integer phase on device closed loops (for ncu -k regex:closed_loop)."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2508_03611_b200 import native, sweep
cells, _ = sweep.make_cells([4, 8, 16, 32, 64, 128], sweep.load_profiles(), request_cap=400, qps_max=64)
native.sweep_run(0, cells, threads=16)
print("done")

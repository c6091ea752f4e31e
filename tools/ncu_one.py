"""One predict launch over the cfg2 (or cfg3) capture, for ncu:
ncu -k regex:predict_kernel -c 1 python tools/ncu_one.py [cfg2|cfg3]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2508_03611_b200 import abi, native
which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
ctx = native.Context(0)
if which == "cfg3":
    w = abi.make_workload(count=2000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1)
else:
    w = abi.make_workload(count=5000, qps=27.0, arrival_seed=1)
cfg = abi.make_config()
_, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(12))
ctx.set_configs(cfg)
dev = torch.device("cuda", 0)
cols = [torch.from_numpy(c).to(dev) for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
scen = torch.from_numpy(ss.scenarios.view(np.uint8)).to(dev)
out = torch.empty(len(ss) * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
st = torch.cuda.Stream(dev)
ctx.predict_batch_device([c.data_ptr() for c in cols], scen.data_ptr(), len(ss), out.data_ptr(), st.cuda_stream, member_capacity=ss.member_capacity(cfg))
torch.cuda.synchronize()
print("done", len(ss))

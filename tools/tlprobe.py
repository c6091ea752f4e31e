"""Per-scenario timeline of one predict pass (debug build with -DBSG_PROFILE_TIMELINE):
active warps over time, the tail after the last scenario starts, and how well
cand_est predicts a scenario's duration.
usage: tools/mkvariant.sh tl "-DBSG_PROFILE_TIMELINE"; BSG_LIB_PATH=build/var_tl/libblocksim_b200.so python tools/tlprobe.py [cfg2|cfg1|cfg3|cfg3q]"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2508_03611_b200 import abi, native

SETS = {
    "cfg1": (dict(count=1000, estimator_kind=2, estimator_seed=1, qps=10.0, arrival_seed=1), 4),
    "cfg2": (dict(count=5000, qps=27.0, arrival_seed=1), 12),
    "cfg3": (dict(count=5000, prompt_median=600, output_median=600, qps=4.5, arrival_seed=1), 12),
    "cfg3q": (dict(count=2000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1), 12),
}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
ctx = native.Context(0)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
kw, n_inst = SETS[name]
w = abi.make_workload(**kw)
cfg = abi.make_config()
_, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(n_inst))
ctx.set_configs(cfg)
cols = [torch.from_numpy(c).to(dev) for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
scen = torch.from_numpy(ss.scenarios.view(np.uint8)).to(dev)
n = len(ss)
out = torch.empty(n * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
cap = ss.member_capacity(cfg)
for _ in range(5):
    ctx.predict_batch_device([c.data_ptr() for c in cols], scen.data_ptr(), n, out.data_ptr(),
                             st.cuda_stream, member_capacity=cap)
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["BSG_LIB_PATH"])
buf = np.zeros(3 * n, np.uint64)
assert lib.bsg_debug_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(n)) == 0
t = buf.reshape(n, 3).astype(np.int64)
s, e, sm = t[:, 0], t[:, 1], t[:, 2]
ok = s > 0
s0 = s[ok].min()
s, e = (s - s0) / 1e3, (e - s0) / 1e3  # us
d = e - s
span = e[ok].max()
print(f"{name}: {n} scenarios, span {span:.1f} us (start spread {s[ok].max():.1f} us), kernel {ctx.last_launch}")
print(f"durations us: mean {d[ok].mean():.2f} p50 {np.median(d[ok]):.2f} p99 {np.percentile(d[ok], 99):.2f} "
      f"max {d[ok].max():.2f}; sum {d[ok].sum()/1e3:.1f} ms")
grid = np.arange(0, span + 1, 1.0)
act = np.zeros(len(grid))
for a, b in zip(s[ok], e[ok]):
    act[int(a):int(np.ceil(b))] += 1
peak = act.max()
print(f"active warps: peak {peak:.0f}; mean over span {act[:int(span)].mean():.0f} "
      f"({act[:int(span)].mean()/peak*100:.1f} % of peak)")
for frac in (0.95, 0.9, 0.75, 0.5, 0.25):
    below = np.nonzero(act[: int(span)] < frac * peak)[0]
    below = below[below > 5]
    first = below[0] if len(below) else span
    print(f"  first us with < {frac*100:.0f}% of peak active: {first:.0f}  (tail {span-first:.1f} us)")
# the last-finishing scenarios
order = np.argsort(-e)
sc = ss.scenarios
print("last to finish: idx start dur cand_est run_n wait_n")
for i in order[:6]:
    print(f"  {i:6d} {s[i]:7.1f} {d[i]:6.1f} {sc['cand_est'][i]:6d} {sc['run_n'][i]:3d} {sc['wait_n'][i]:4d}")
lng = np.argsort(-d)
print("longest: idx start dur cand_est run_n wait_n")
for i in lng[:6]:
    print(f"  {i:6d} {s[i]:7.1f} {d[i]:6.1f} {sc['cand_est'][i]:6d} {sc['run_n'][i]:3d} {sc['wait_n'][i]:4d}")
ce = sc["cand_est"][ok].astype(float)
print(f"corr(duration, cand_est) = {np.corrcoef(d[ok], ce)[0,1]:.3f}; "
      f"corr(duration, cand_est+wait_n*100) = {np.corrcoef(d[ok], ce + sc['wait_n'][ok]*100)[0,1]:.3f}")
hist, edges = np.histogram(s[ok], bins=20, range=(0, span))
print("starts per span/20:", hist.tolist())
hist, _ = np.histogram(e[ok], bins=20, range=(0, span))
print("ends   per span/20:", hist.tolist())
print("active per span/20:", [int(act[int(a)]) for a in np.linspace(0, span - 1, 20)])

"""Which steps the windows leave to general iterations (debug: the
BSG_PROFILE_T0 build marks window-retired trace records): per-step kinds
from the reference trace, for general-iteration steps only.
usage: BSG_LIB_PATH=build/t0/libblocksim_b200.so python tools/winclass.py [n]"""
import os, sys, collections
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_03611_b200 import abi, native
from oracle.oracle import Reference
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ctx = native.Context(0)
ref = Reference()
w = abi.make_workload(count=2000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1)
cfg = abi.make_config()
_, _, ss = ctx.replay(w, cfg, abi.make_replay_spec(12))
ctx.set_configs(cfg)
os.environ["BSG_TRACE_J"] = "1"
rng = np.random.default_rng(0)
c = collections.Counter(); tot = 0
for i in rng.choice(len(ss), n, replace=False):
    _, tg = ctx.trace(ss, int(i), cap=1 << 16)
    _, tr = ref.trace(cfg, ss, int(i), cap=1 << 16)
    gen = (tg["n_prefill"] >> 20) == 0
    npf, npe, pt, nd = tr["n_prefill"], tr["n_preempted"], tr["prefill_tokens"], tr["n_decode"]
    A = (npf == 1) & (npe == 0) & (pt == 512 - nd)
    B = (npf == 0) & (npe == 1)
    pa = np.zeros(len(tr), bool); pb = np.zeros(len(tr), bool)
    p = A[:-1] & B[1:]; pa[:-1] |= p; pb[1:] |= p
    tot += len(tr)
    for t in np.nonzero(gen)[0]:
        prev = "after_gen" if t > 0 and gen[t - 1] else "after_win"
        if pa[t]: k = "pairA"
        elif pb[t]: k = "pairB"
        elif npf[t] == 0 and npe[t] == 0: k = "decode"
        else: k = f"pf{min(npf[t],3)}_pe{min(npe[t],3)}"
        c[(k, prev)] += 1
print("steps per scenario", tot / n)
for k, v in c.most_common(): print(k, round(v / n, 1))

"""Generates the committed golden fixtures from the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/libblocksim_ref.so from the reference sources
(oracle/Makefile) and records, for each fixture scenario, the reference's
predict() outputs (doubles, as hex-exact repr) and, for the trace fixtures,
the per-step fingerprints of Instance::execute_step. The GPU box has no
/root/reference; tests there compare against these files (and against the
prebuilt .so that travels with the repo snapshot).
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from oracle import oracle  # noqa: E402
from scenarios import fuzz_set, kat_set  # noqa: E402


def dump_set(names, cfgs, ss, ref_res, traces=None):
    rows = []
    for i in range(len(ss)):
        sc = ss.scenarios[i]
        r0, rn, w0, wn = (int(sc[k]) for k in ("run_off", "run_n", "wait_off", "wait_n"))
        ent = lambda a, b: [[int(ss.prompt[k]), int(ss.est[k]), int(ss.prefill[k]),  # noqa: E731
                             int(ss.decoded[k])] for k in range(a, a + b)]
        rr = ref_res[i]
        row = {
            "name": names[i] if names else f"fuzz_{i}",
            "cfg": int(sc["cfg"]),
            "running": ent(r0, rn),
            "waiting": ent(w0, wn),
            "candidate": [int(sc["cand_prompt"]), int(sc["cand_est"])],
            "expect": {
                "status": int(rr["status"]), "detail": int(rr["detail"]),
                "steps": int(rr["steps"]),
                "e2e_s": float(rr["e2e_s"]).hex(), "ttft_s": float(rr["ttft_s"]).hex(),
                "qdelay_s": float(rr["qdelay_s"]).hex(),
            },
        }
        if traces is not None and i in traces:
            row["trace"] = [[int(x) for x in rec.tolist()] for rec in traces[i]]
        rows.append(row)
    return {
        "configs": [{k: (v.item() if hasattr(v, "item") else v) for k, v in zip(cfgs.dtype.names, c)}
                    for c in cfgs],
        "scenarios": rows,
    }


def main():
    oracle.build(ref=True)
    ref = oracle.Reference()
    names, kc, ks = kat_set()
    kr = ref.predict_batch(kc, ks)
    with open(os.path.join(HERE, "reference_kats.json"), "w") as f:
        json.dump(dump_set(names, kc, ks, kr, None), f, indent=0)
    fc, fs = fuzz_set(7, 400)
    fr = ref.predict_batch(fc, fs)
    with open(os.path.join(HERE, "fuzz_400_seed7.json"), "w") as f:
        json.dump(dump_set(None, fc, fs, fr, None), f, indent=0)
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()

"""cfg5 — auto-provisioning capacity sweep on B200s.

Grid: instances {4, 8, 16, 32, 64, 128} x 3 latency profiles
(configs/profiles.json) x capacity_search over QPS [1, 64] (every integer
QPS, then tenths inside the bracket: metrics.cpp:139-178), BlockPredictive
dispatch, P99-TTFT SLO 3 s (config.cpp:247 default), a request cap per run.
Each cell's closed loops run on host threads with GPU what-ifs
(bsg_sweep_run); cells are LPT-assigned across ranks (shard.py) with no
data-path collective; rank 0 gathers the table.

    python -m paper_2508_03611_b200.sweep [--request-cap 400] [--threads 16]
    torchrun --nproc-per-node N -m paper_2508_03611_b200.sweep ...
"""
from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np

from . import abi, native, shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES_JSON = os.path.join(ROOT, "configs", "profiles.json")


def load_profiles(path: str = PROFILES_JSON) -> dict[str, np.ndarray]:
    with open(path) as f:
        prof = json.load(f)["profiles"]
    return {name: abi.make_config(**kw) for name, kw in prof.items()}


def make_cells(instances, profiles: dict, request_cap: int, qps_min: int = 1, qps_max: int = 64,
               slo: float = 3.0, seed: int = 1, count: int | None = None,
               policy: int = abi.POLICY_BLOCK_PREDICTIVE, provision: dict | None = None
               ) -> tuple[np.ndarray, list]:
    """Cells of the grid. provision: ProvisionPolicy overrides for auto-provisioned
    cells, e.g. dict(provision_kind=abi.PROVISION_PREEMPT, extra_instances=4,
    threshold_s=70, cold_start_s=30, cooldown_s=15) (max_instances = n + extra)."""
    provision = dict(provision or {})
    extra = provision.pop("extra_instances", 0)
    cells = np.zeros(len(instances) * len(profiles), abi.sweep_cell_dtype)
    keys = []
    i = 0
    for pname, cfg in profiles.items():
        for n in instances:
            c = cells[i]
            c["workload"] = abi.make_workload(count=count or request_cap, request_cap=request_cap)[0]
            c["cfg"] = cfg[0]
            c["spec"] = abi.make_replay_spec(n, policy=policy, capture=0,
                                             max_instances=(n + extra) if provision else None,
                                             **provision)[0]
            c["seed"], c["qps_min"], c["qps_max"], c["slo_p99_ttft_s"] = seed, qps_min, qps_max, slo
            keys.append((pname, int(n)))
            i += 1
    return cells, keys


def cell_cost(cell) -> float:
    """LPT key: what-ifs per dispatch (instances) x arrivals per run."""
    return float(cell["spec"]["n_instances"]) * float(cell["workload"]["request_cap"])


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--request-cap", type=int, default=400)
    ap.add_argument("--instances", default="4,8,16,32,64,128")
    ap.add_argument("--qps-max", type=int, default=64)
    ap.add_argument("--threads", type=int, default=16)
    ap.add_argument("--slo", type=float, default=3.0)
    ap.add_argument("--provision", choices=["static", "preempt", "relief"], default="static",
                    help="auto-provisioning policy of every cell (autoscaler.cpp:36-52)")
    ap.add_argument("--extra-instances", type=int, default=4,
                    help="max_instances = instances + this, when provisioning")
    args = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("BSG_DIST_ONE_GPU") == "1":  # multi-rank code path on one GPU (tests)
            local = 0
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prov = None if args.provision == "static" else dict(
        provision_kind={"preempt": abi.PROVISION_PREEMPT, "relief": abi.PROVISION_RELIEF}[args.provision],
        extra_instances=args.extra_instances)
    cells, keys = make_cells([int(x) for x in args.instances.split(",")], load_profiles(),
                             args.request_cap, qps_max=args.qps_max, slo=args.slo, provision=prov)
    native.sweep_run(local, cells[:1], threads=args.threads)  # warm-up: context + module load
    assign = shard.assign_cells_lpt([cell_cost(c) for c in cells], world)
    mine = sorted(assign[rank], key=lambda c: -cell_cost(cells[c]))
    t0 = time.perf_counter()
    out = native.sweep_run(local, cells[mine], threads=args.threads)
    wall = time.perf_counter() - t0
    rows = [(keys[c], out[j]) for j, c in enumerate(mine)]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (wall, rows))
        walls = [g[0] for g in gathered]
        rows = [r for g in gathered for r in g[1]]
        wall = max(walls)
        dist.destroy_process_group()
    if rank != 0:
        return None
    total = sum(int(o["whatif_scenarios"]) for _, o in rows)
    table = {f"{k[0]}/{k[1]}": (abi.STATUS_NAMES.get(int(o["status"]), int(o["status"])) if
                                int(o["status"]) != abi.OK else float(o["result"]["capacity_qps"]))
             for k, o in sorted(rows, key=lambda r: (r[0][0], r[0][1]))}
    line = {"metric": "capacity sweep what-if scenarios/sec (cfg5)", "value": total / wall,
            "unit": "scenarios/s", "n_gpus": world, "wall_s": wall, "whatif_scenarios": total,
            "cells": len(rows), "closed_loops": int(sum(int(o["result"]["n_tested"]) for _, o in rows)),
            "config": {"instances": args.instances, "profiles": list(load_profiles()),
                       "qps": f"1..{args.qps_max} + tenths", "request_cap": args.request_cap,
                       "slo_p99_ttft_s": args.slo, "policy": "block_predictive",
                       "provision": args.provision,
                       "threads_per_gpu": args.threads},
            "capacity_qps": table}
    print(json.dumps(line), flush=True)
    return line


if __name__ == "__main__":
    main()

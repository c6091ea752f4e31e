"""bench.py — simulated what-if scenarios/sec (Block predictive dispatch core).

Workload (N=1, BASELINE.json configs[1]): 12-instance cluster, Llama-2-7B
profile (InstanceConfig defaults: 1056 x 16-token blocks, batch 48, chunk
512, c0 0.01 / 1e-4 / 1e-3 / 1e-7), 5,000 synthetic ShareGPT-shaped requests
(make_synthetic_trace defaults, seed 1234) at 27 QPS with Poisson arrivals.
A BlockPredictive closed loop (host live instances, GPU what-ifs) captures
every per-request what-if fanout: 5,000 arrivals x 12 instances = 60,000
(snapshot, candidate) scenarios. One step = predict() over all 60,000.

  value : device-timed (CUDA events on the launching stream) scenarios/s with
          inputs resident in HBM, L2 flushed (256 MiB write) between steps.
  e2e   : the same metric through the public C-ABI with HOST (pinned) buffers:
          bsg_predict_batch = H2D of the step's inputs + kernel + D2H results.
  parity: every timed set's GPU results against the reference's own predict()
          (oracle/_ref, all host cores) on the same scenarios — mismatch counts.
  --impl reference : the reference's own CPU predict() (oracle/_ref, compiled
          from /root/reference) on all host cores over the same workload,
          captured by the reference's own driver loop.

Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun spawns
the N ranks itself). --scaling weak (default): each rank captures its own
5,000-request replay (arrival seed 1 + rank). --scaling strong: every rank
captures the same replay and simulates a contiguous 1/N of its arrival groups
(all 12 what-ifs of an arrival stay on one GPU, so each argmin is local). No
data-path collective either way; NCCL carries the barrier and the
max-over-ranks timing / count reductions, and in the cfg4 latency leg one
MIN all-reduce of the packed (score, id) key per dispatch, straight from
device memory.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E2E_WARMUP_CALLS = 50
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")

# BASELINE.json configs as bench.py measures them (tests/test_gpu_configs.py
# pins parity on exactly these sets).
CONFIGS = {
    "cfg1": dict(kw=dict(count=1000, estimator_kind=2, estimator_seed=1, qps=10.0, arrival_seed=1),
                 n_inst=4, desc="4 instances, 1000 requests @ 10 QPS, Noisy(0.244) predicted lengths"),
    "cfg2": dict(kw=dict(count=5000, qps=27.0, arrival_seed=1), n_inst=12,
                 desc="12-instance cluster, Llama-2-7B profile (1056x16 blocks, batch 48, chunk 512), "
                      "5000 synthetic ShareGPT-shaped requests @ 27 QPS; per-request what-if fanout "
                      "over all 12 instances captured from a BlockPredictive closed loop"),
    "cfg3": dict(kw=dict(count=5000, prompt_median=600, output_median=600, qps=4.5, arrival_seed=1),
                 n_inst=12, desc="12 instances, long-response shape (prompt/output medians 600), "
                                 "5000 requests @ 4.5 QPS, KV-pressure preemption + chunked prefill"),
    "cfg3_quick": dict(kw=dict(count=2000, prompt_median=600, output_median=600, qps=5.0,
                               arrival_seed=1),
                       n_inst=12, desc="cfg3's quick variant: 2000 requests @ 5 QPS"),
}
N_INST, N_REQ, QPS = 12, CONFIGS["cfg2"]["kw"]["count"], CONFIGS["cfg2"]["kw"]["qps"]


def workload(name: str = "cfg2", arrival_seed: int | None = None):
    from paper_2508_03611_b200 import abi
    c = CONFIGS[name]
    kw = dict(c["kw"])
    if arrival_seed is not None:
        kw["arrival_seed"] = arrival_seed
    return abi.make_workload(**kw), abi.make_config(), abi.make_replay_spec(c["n_inst"])


def capture(ctx, name: str = "cfg2", arrival_seed: int | None = None):
    """The scenario set a BlockPredictive closed loop evaluates on `name` (host
    live instances, GPU what-ifs; tick-identical to the reference's driver)."""
    w, cfg, spec = workload(name, arrival_seed)
    _, _, ss = ctx.replay(w, cfg, spec)
    return cfg, ss


def workload_desc(scaling: str = "weak", world: int = 1):
    return {
        "workload": "cfg2: " + CONFIGS["cfg2"]["desc"] + " = 60000 scenarios per step" + (
            f" per GPU (weak scaling: arrival seed 1 + rank)" if scaling == "weak" and world > 1 else
            f", split by arrival group over {world} GPUs (strong scaling)" if world > 1 else ""),
        "instances": N_INST, "requests": N_REQ, "qps": QPS,
        "l2": "flushed between timed steps (256 MiB write); inputs < L2",
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_cmd(argv: list[str], n: int, port: int | None = None) -> list[str]:
    """The torchrun command that runs this script as n ranks (one per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={port or _free_port()}",
            os.path.abspath(__file__), *argv]


def spawn(args, argv: list[str]) -> int:
    """`--gpus N` outside torchrun: launch the N ranks ourselves (rank 0 prints
    the JSON line). NCCL's init log stays on (NCCL_DEBUG=INFO unless set) so
    the communicator's rank count can be checked."""
    one_gpu = os.environ.get("BSG_DIST_ONE_GPU") == "1"
    if not one_gpu and not args.dist_probe and args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"--gpus {args.gpus}: only {have} CUDA device(s) visible")
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(spawn_cmd(argv, args.gpus), env=env)


def dist_probe():
    """--dist-probe: the rank plumbing alone (gloo, no GPU): every rank joins,
    the ranks' indices are summed; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    world, rank, _ = dist_setup()
    dist.init_process_group("gloo")
    t = torch.tensor([rank, 1], dtype=torch.int64)
    dist.all_reduce(t)
    line = {"probe": "dist", "world": world, "rank_sum": int(t[0]), "ranks": int(t[1])} if rank == 0 else None
    dist.barrier()
    dist.destroy_process_group()
    return line


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2508_03611_b200 import abi, native, shard

    world, rank, local = dist_setup()
    # BSG_DIST_ONE_GPU=1: every rank on cuda:0 with gloo collectives — only for
    # exercising the multi-rank code path on a one-GPU box (timings meaningless)
    one_gpu = os.environ.get("BSG_DIST_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    coll_dev = None if one_gpu else dev  # gloo reduces host tensors
    ctx = native.Context(local)

    # ---- setup (untimed): capture this rank's scenario set --------------------
    strong = args.scaling == "strong"
    t0 = time.perf_counter()
    cfg, ss_all = capture(ctx, "cfg2", arrival_seed=1 if strong else shard.weak_seed(rank))
    capture_s = time.perf_counter() - t0
    ctx.set_configs(cfg)
    if strong:  # contiguous arrival groups (N_INST what-ifs each) per rank
        g0, g1 = shard.group_range(len(ss_all) // N_INST, world, rank)
        rows = slice(g0 * N_INST, g1 * N_INST)
    else:
        rows = slice(0, len(ss_all))
    scen_rows = np.ascontiguousarray(ss_all.scenarios[rows])
    ss = abi.ScenarioSet(ss_all.prompt, ss_all.est, ss_all.prefill, ss_all.decoded, scen_rows)
    n = len(ss)

    # device-resident inputs
    cols = [torch.from_numpy(c).to(dev) for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
    scen = torch.from_numpy(ss.scenarios.view(np.uint8)).to(dev)
    out = torch.empty(max(n, 1) * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # A dedicated stream: the kernel, the L2 flush and the CUDA events all live on it.
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    cap = ss.member_capacity(cfg)

    def step():
        ctx.predict_batch_device([c.data_ptr() for c in cols], scen.data_ptr(), n, out.data_ptr(),
                                 stream.cuda_stream, member_capacity=cap)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    kernel = ctx.last_launch
    res = np.frombuffer(out.cpu().numpy().tobytes(), dtype=abi.result_dtype)[:n].copy()
    assert (res["status"] == abi.OK).all(), "benchmark scenarios must all succeed"
    member_steps = int(res["member_steps"].sum())
    sim_steps = int(res["steps"].sum())

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ctx.launches
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            flush.zero_()  # L2 flush on the same stream, outside the event bracket
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        launches = ctx.launches - launches0
        per_step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        total_ms = sum(per_step_ms)

        # ---- e2e: public C-ABI with pinned HOST buffers ------------------------
        pinned = [torch.from_numpy(c).pin_memory() for c in (ss.prompt, ss.est, ss.prefill,
                                                              ss.decoded)]
        pscen = torch.from_numpy(ss.scenarios.view(np.uint8)).pin_memory()
        host = abi.ScenarioSet(*[p.numpy() for p in pinned],
                               pscen.numpy().view(abi.scenario_dtype))
        pout = torch.empty(max(n, 1) * abi.result_dtype.itemsize, dtype=torch.uint8).pin_memory()
        e2e_times = []
        import ctypes as C
        ent = host.entries()
        # The host-buffer path needs ~40 calls to reach steady state (pinned-page
        # DMA mappings, the stream-ordered scratch pool, clocks): measured 0.99 ms
        # per call over the first 40, 0.72 ms after (tools/e2e_sampler_probe.py).
        e2e_warm = max(args.warmup, E2E_WARMUP_CALLS)
        for i in range(e2e_warm + args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            ta = time.perf_counter()
            st = ctx.L.bsg_predict_batch(ctx.h, C.byref(ent), host.n_entries,
                                         abi.ptr(host.scenarios), n, C.c_void_p(pout.data_ptr()))
            tb = time.perf_counter()
            assert st == abi.OK
            if i >= e2e_warm:
                e2e_times.append(tb - ta)
        e2e_res = np.frombuffer(pout.numpy().tobytes(), dtype=abi.result_dtype)[:n]
    e2e_total = sum(e2e_times)
    e2e_same = bool(e2e_res.tobytes() == res.tobytes())

    # ---- max over ranks (NCCL only here: timings and counts) -------------------
    if world > 1:
        (total_ms, e2e_total), (n_all, ms_all, launches_all, e2e_bad) = shard.reduce_max_sum(
            [total_ms, e2e_total], [n, member_steps, launches, 0 if e2e_same else 1], device=coll_dev)
        e2e_same = e2e_bad == 0
    else:
        n_all, ms_all, launches_all = n, member_steps, launches

    value = n_all * args.steps / (total_ms / 1e3)
    e2e_value = n_all * args.steps / e2e_total

    line = None
    if rank == 0:
        avg_launch_s = (total_ms / args.steps) / 1e3
        line = {
            "metric": "simulated what-if scenarios/sec (predict() fanout, cfg2 12 instances)",
            "value": value, "unit": "scenarios/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "int32+f64", "data": "synthetic (reference generators, seeded)",
            "config": {**workload_desc(args.scaling, world), "scenarios_per_step": n_all,
                       "entries": ss.n_entries,
                       "parallelism": (f"replicas{world} (scenario shards, no collective)" if world > 1
                                       else "1 GPU")},
            "e2e": {"value": e2e_value, "unit": "scenarios/s",
                    "h2d_bytes_per_step": h2d_bytes(ss),
                    "d2h_bytes_per_step": int(n * abi.result_dtype.itemsize),
                    "ms_per_step": e2e_total / args.steps * 1e3,
                    "warmup_calls": e2e_warm, "results_identical_to_device_path": e2e_same,
                    "l2": "flushed before every call"},
            "gpu_launches": launches_all,
            "roofline": roofline(torch, dev, ss, n, member_steps, avg_launch_s, kernel),
            "clocks": clocks.summary(),
            "work": {"simulated_steps_per_step": sim_steps, "member_steps_per_step": ms_all,
                     "capture_s": capture_s},
        }
        if args.cpu_baseline and world == 1:
            line["cpu_baseline"], exp = cpu_baseline(ss, cfg)
            line["parity"] = {"cfg2": parity(res, exp)}
    if args.latency:
        lat = mc_latency(ctx, world, rank, coll_dev)
        if rank == 0:
            line["dispatch_latency"] = lat
            line["dispatch_latency_mirror"] = fleet_latency(ctx)
            if world == 1 and args.cpu_baseline:
                line["dispatch_latency"]["cpu_baseline"] = reference_latency()
    if args.extra and rank == 0 and world == 1:
        line["other_configs"] = other_configs(ctx, dev)
        for k, v in line["other_configs"].items():
            line.setdefault("parity", {})[k] = v["parity"]
        line["capacity_sweep"] = capacity_sweep(local)
        line["capacity_table"] = capacity_table(local)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return line


def h2d_bytes(ss) -> int:
    """Bytes bsg_predict_batch copies host->device for this set: the entry
    range the scenarios reference (4 int32 columns) + the scenario rows."""
    sc = ss.scenarios
    lo = min(int(sc["run_off"].min()), int(sc["wait_off"].min())) if len(sc) else 0
    hi = max(int((sc["run_off"] + sc["run_n"]).max()), int((sc["wait_off"] + sc["wait_n"]).max())) if len(sc) else 0
    return 16 * max(hi - lo, 0) + sc.nbytes


def parity(got, exp_ref) -> dict:
    """Mismatch count of GPU results vs the reference's on the same scenarios:
    status + detail, and ticks / steps of successes, bit-exact."""
    from oracle.oracle import compare_to_ref
    bad = compare_to_ref(got, exp_ref)
    return {"scenarios": int(len(got)), "mismatches": int(bad.sum()),
            "checked_against": "reference predict() (oracle/_ref) on the same scenarios, bit-exact"}


def roofline(torch, dev, ss, n, member_steps, avg_launch_s, kernel):
    """Roofs of the timed step. Primary: SM issue — the path is a
    dependent integer state machine (work unit = member-step, 24 int32 lane-ops
    each) against 148 SMs x 128 int32 lanes x the max SM clock. Secondary: HBM
    (algorithmic bytes vs the measured copy bandwidth). ncu figures come from
    the committed capture named in `ncu.source` (never from a profiled run)."""
    from paper_2508_03611_b200 import abi
    peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    ncu = json.load(open(tpath)) if os.path.exists(tpath) else {}
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    issue_peak = sms * 128 * sm_mhz * 1e6
    achieved_int = member_steps * 24 / avg_launch_s
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # algorithmic bytes per launch: 16 B per snapshot entry + 32 B scenario + 48 B result
    algo_bytes = 16 * ss.n_entries + 32 * n + abi.result_dtype.itemsize * n
    achieved_gbs = algo_bytes / avg_launch_s / 1e9
    return {
        "bound": "issue", "achieved": achieved_int / 1e12, "peak": issue_peak / 1e12,
        "unit": "T int32-lane-ops/s", "frac": achieved_int / issue_peak,
        "traffic": ncu.get("dram_bytes_per_launch"),
        "kernel": kernel,
        "work": {"member_steps_per_launch": member_steps, "ops_per_member_step": 24,
                 "sm_count": sms, "sm_mhz": sm_mhz,
                 "peak_source": "MEASURED_PEAKS.json sm_max_mhz" if "sm_max_mhz" in peaks else
                                "B200_PROFILING.md fallback"},
        "hbm": {"achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak, "algorithmic_bytes_per_launch": algo_bytes},
        "ncu": {k: ncu.get(k) for k in ("issue_active_pct", "achieved_occupancy_pct",
                                         "dram_bytes_per_launch", "source", "kernel")},
        "note": "event skipping retires whole pure-decode windows without executing their "
                "member-steps one by one, so achieved counts algorithmic (reference) work; ncu "
                "issue-active is the executed-instruction gauge",
    }


def mc_latency(ctx, world: int = 1, rank: int = 0, device=None, n_calls: int = 400,
               n_inst: int = 64, n_samples: int = 256):
    """cfg4: p50/p99 wall time of ONE BlockPredictive dispatch call with 256
    Monte-Carlo length samples per candidate over 64 instances (16,384 what-if
    scenarios per call, prefix-shared into 64 simulations), through the public
    C-ABI with host buffers: pack + H2D + on-device sampling (K3) + kernel +
    fused argmin + D2H. Snapshots come from a 64-instance, 3000-request, 130 QPS
    closed loop. With N GPUs, instance i is simulated on rank i % N and the
    per-request argmin is one NCCL MIN all-reduce of the packed key the kernel
    leaves in device memory; one 8-byte read returns the decision."""
    import torch
    from paper_2508_03611_b200 import abi, native, shard
    w = abi.make_workload(count=3000, qps=130.0, arrival_seed=1)
    cfg = abi.make_config()
    _, _, cap = ctx.replay(w, cfg, abi.make_replay_spec(n_inst))
    ctx.set_configs(cfg)
    n_arr = len(cap) // n_inst
    mine = shard.instance_shard(n_inst, world, rank)
    picks = np.linspace(0, n_arr - 1, n_calls).astype(int)
    import ctypes as C
    calls = []
    for g in picks:
        one = cap.compact(g * n_inst + mine)
        calls.append((one, one.entries(), np.array([g], np.uint64), int(g)))
    ids = np.ascontiguousarray(mine, dtype=np.int32)
    chosen = np.zeros(1, np.int32)
    sc_local = np.zeros(len(mine), np.int64)
    key = None
    if world > 1:
        import torch.distributed as dist
        key = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", torch.cuda.current_device()))
    kp = C.c_void_p(key.data_ptr()) if key is not None else None
    lat = []
    for i, (one, ent, rid, g) in enumerate(calls * 2):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        st = ctx.L.bsg_dispatch_mc_sampled(ctx.h, C.byref(ent), one.n_entries, abi.ptr(one.scenarios),
                                           abi.ptr(ids), len(mine), 1, abi.ptr(rid), n_samples, 1,
                                           0.244, 0, abi.ptr(chosen), abi.ptr(sc_local), None, None, kp)
        pick = int(chosen[0]) if world == 1 else shard.reduce_key(key, sc_local, ids, device)
        t1 = time.perf_counter()
        assert st == abi.OK and pick >= 0
        if i >= len(calls):  # first pass is warm-up
            lat.append((t1 - t0) * 1e6)
        elif world > 1 and os.environ.get("BSG_DIST_ONE_GPU") == "1":
            # test mode: the sharded decision must equal the one-GPU decision
            full = cap.compact(g * n_inst + np.arange(n_inst))
            ch1, _, _ = ctx.dispatch_mc_sampled(full, np.arange(n_inst, dtype=np.int32), n_inst,
                                                [g], n_samples, seed=1)
            assert int(ch1[0]) == pick, (g, int(ch1[0]), pick)
    lat = np.array(lat)
    return {"p50_us": float(np.percentile(lat, 50)), "p99_us": float(np.percentile(lat, 99)),
            "max_us": float(lat.max()), "calls": len(lat), "gpus": world,
            "kernel": ctx.last_launch,
            "config": f"cfg4: {n_inst} instances x {n_samples} MC length samples per candidate "
                      "(16384 what-if scenarios per dispatch, 64 prefix-shared simulations), "
                      "snapshots from a 3000-request 130 QPS closed loop; host buffers, samples "
                      "drawn on the device inside the call, wall clock per call"
                      + (f"; instances sharded i % {world}, NCCL MIN of the device-resident key"
                         if world > 1 else "")}


def reference_latency(n_inst: int = 64, n_samples: int = 256, n_calls: int = 400,
                      n_mc_calls: int = 12):
    """The reference's dispatch latency on this host (SURVEY 8(d) "also report"):
    (a) predict_across over the same 64 snapshots per call on ONE thread (the
    reference's own loop, predictor.cpp:139-157), p50/p99 over the same calls;
    (b) the 64 x 256 Monte-Carlo loop (predict per (instance, sample)) on all
    host threads, a bounded sample of calls."""
    from oracle.oracle import Reference
    from paper_2508_03611_b200 import abi, native
    ref = Reference()
    w = abi.make_workload(count=3000, qps=130.0, arrival_seed=1)
    cfg = abi.make_config()
    _, _, cap = ref.replay(w, cfg, abi.make_replay_spec(n_inst))
    n_arr = len(cap) // n_inst
    picks = np.linspace(0, n_arr - 1, n_calls).astype(int)
    one = []
    for g in picks:
        sub = cap.compact(g * n_inst + np.arange(n_inst))
        one.append(ref.time_predict(cfg, sub, threads=1, reps=1) * 1e6)
    threads = os.cpu_count() or 1
    mc = []
    for g in picks[:: max(1, n_calls // n_mc_calls)][:n_mc_calls]:
        sub = cap.compact(g * n_inst + np.arange(n_inst))
        lens = native.mc_lengths(int(sub.scenarios[0]["cand_est"]), int(g), n_samples, seed=1)
        rows = np.repeat(sub.scenarios, n_samples)
        rows["cand_est"] = np.tile(lens, n_inst)
        big = abi.ScenarioSet(sub.prompt, sub.est, sub.prefill, sub.decoded, rows)
        mc.append(ref.time_predict(cfg, big, threads=threads, reps=1) * 1e6)
    one, mc = np.array(one), np.array(mc)
    return {"predict_across_1thread": {"p50_us": float(np.percentile(one, 50)),
                                       "p99_us": float(np.percentile(one, 99)), "calls": len(one),
                                       "cores": 1, "kind": "reference",
                                       "what": "64 predict() per call, no MC samples"},
            "mc_64x256_all_threads": {"p50_us": float(np.percentile(mc, 50)),
                                      "p99_us": float(np.percentile(mc, 99)), "calls": len(mc),
                                      "cores": threads, "kind": "reference",
                                      "what": "16384 predict() per call (each (instance, sample))"}}


def fleet_latency(ctx, n_inst: int = 64, n_samples: int = 256, count: int = 3000,
                  qps: float = 130.0):
    """cfg4 on the device mirror (bsg_fleet_dispatch): the 64-instance cluster's
    live state stays in HBM; every arrival of a 3000-request 130 QPS stream is
    ONE call — advance the instances in place, draw the candidate's 256
    Monte-Carlo lengths on the device (K3), what-ifs on all 64, argmin, admit —
    timed per call (wall clock, host API: only the candidate's scalars go in)."""
    from paper_2508_03611_b200 import abi, native
    cfg = abi.make_config()
    ctx.set_configs(cfg)
    w = abi.make_workload(count=count, qps=qps, arrival_seed=1)
    p, o, e, t = native.make_workload_host(w)
    lat = []
    for rep in range(2):  # first pass warms up (module load, allocations)
        fl = native.Fleet(ctx, n_inst, count)
        for k in range(count):
            t0 = time.perf_counter()
            fl.dispatch_sampled(t[k], p[k], e[k], o[k], request_id=k, n_samples=n_samples, seed=1)
            if rep:
                lat.append((time.perf_counter() - t0) * 1e6)
        fl.finish(count)
        fl.close()
    lat = np.array(lat)
    return {"p50_us": float(np.percentile(lat, 50)), "p99_us": float(np.percentile(lat, 99)),
            "max_us": float(lat.max()), "calls": len(lat),
            "config": f"cfg4 on the device mirror: {n_inst} instances x {n_samples} MC samples, "
                      f"{count} arrivals @ {qps:g} QPS, one bsg_fleet_dispatch per arrival "
                      "(advance + on-device sampling + what-ifs + argmin + admit), wall clock per call"}


def device_time(ctx, ss, cfg, dev, reps: int = 5):
    """Device-timed predict over a resident scenario set (L2 flushed between
    launches); returns (scenarios/s, member_steps, results, kernel)."""
    import torch
    from paper_2508_03611_b200 import abi
    ctx.set_configs(cfg)
    n = len(ss)
    cols = [torch.from_numpy(c).to(dev) for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
    scen = torch.from_numpy(ss.scenarios.view(np.uint8)).to(dev)
    out = torch.empty(n * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    cap = ss.member_capacity(cfg)
    f = lambda: ctx.predict_batch_device([c.data_ptr() for c in cols], scen.data_ptr(), n,
                                         out.data_ptr(), stream.cuda_stream, member_capacity=cap)
    for _ in range(3):
        f()
    ms = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        f()
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms.append(a.elapsed_time(b))
    res = np.frombuffer(out.cpu().numpy().tobytes(), dtype=abi.result_dtype).copy()
    return n / (statistics.median(ms) / 1e3), int(res["member_steps"].sum()), res, ctx.last_launch


def other_configs(ctx, dev):
    """BASELINE configs[0] and [2] (parity cases, reported beside the headline):
    device-timed throughput on their captured what-if sets, the reference's
    predict() on this host's cores over a bounded sample of the same set, and
    the mismatch count of the WHOLE set against the reference."""
    from oracle.oracle import Reference
    ref = Reference()
    threads = os.cpu_count() or 1
    out = {}
    for name, sample in (("cfg1", 4000), ("cfg3", 2400)):
        cfg, ss = capture(ctx, name)
        value, msteps, res, kernel = device_time(ctx, ss, cfg, dev)
        sub = ss.compact(np.unique(np.linspace(0, len(ss) - 1, min(sample, len(ss))).astype(np.int64)))
        secs = ref.time_predict(cfg, sub, threads=threads, reps=1)
        exp = ref.predict_batch(cfg, ss, threads=threads)
        peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
        issue_peak = (torch_sms(dev) * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6)
        achieved = msteps * 24 * value / len(ss)
        out[name] = {"workload": CONFIGS[name]["desc"], "scenarios": len(ss), "value": value,
                     "unit": "scenarios/s", "member_steps": msteps, "kernel": kernel,
                     "roofline": {"bound": "issue", "achieved": achieved / 1e12, "peak": issue_peak / 1e12,
                                  "unit": "T int32-lane-ops/s", "frac": achieved / issue_peak,
                                  "work": "member-steps x 24 int32 lane-ops (SURVEY 8(d)) per launch time"},
                     "parity": parity(res, exp),
                     "cpu_baseline": {"value": len(sub) / secs, "unit": "scenarios/s", "cores": threads,
                                      "kind": "reference",
                                      "sample": f"{len(sub)} scenarios evenly spaced over the same set"}}
    return out


def torch_sms(dev) -> int:
    import torch
    return torch.cuda.get_device_properties(dev).multi_processor_count


def capacity_table(local: int):
    """run_capacity (driver.cpp:392-427) — the paper's capacity-gain table: the
    capacity of BlockPredictive and the heuristics against the Llumnix- baseline
    (8 instances of the P1 profile, 800 requests, QPS 1-40, SLO p99 TTFT < 3 s),
    every capacity search's closed loops on the device (bsg_run_capacity), timed
    against the reference's capacity searches on all host cores (ref_sweep, the
    same (policy, qps) closed loops), rows and gains checked equal."""
    from oracle.oracle import Reference
    from paper_2508_03611_b200 import abi, native, sweep
    threads = os.cpu_count() or 1
    cfg = sweep.load_profiles()["P1_llama2_7b"]
    w = abi.make_workload(count=800)
    spec = abi.make_replay_spec(8, capture=0)
    pols = [abi.POLICY_BLOCK_PREDICTIVE, abi.POLICY_INFAAS_PP, abi.POLICY_MIN_QPM,
            abi.POLICY_ROUND_ROBIN, abi.POLICY_RANDOM]
    base = abi.POLICY_LLUMNIX_MINUS
    native.run_capacity(local, w, cfg, spec, pols[:1], base, 1, 1, 2, 3.0, threads=threads)  # warm-up
    t0 = time.perf_counter()
    rows, bcap = native.run_capacity(local, w, cfg, spec, pols, base, 1, 1, 40, 3.0, threads=threads)
    gpu_s = time.perf_counter() - t0
    cells = np.zeros(len(rows), abi.sweep_cell_dtype)
    for i, p in enumerate(rows["policy"]):
        sp = spec.copy()
        sp["policy"] = p
        cells[i] = (w[0], np.asarray(cfg).reshape(-1)[0], sp[0], 1, 1, 40, 3.0)
    rr, ref_s = Reference().sweep(cells, threads=threads)
    rb = float(rr["result"]["capacity_qps"][list(rows["policy"]).index(base)])
    egain = [("%.1f%%" % ((c - rb) / rb * 100.0)).encode() if p != base else b""
             for p, c in zip(rows["policy"], rr["result"]["capacity_qps"])]
    same = bool(rows["result"].tobytes() == rr["result"].tobytes() and list(rows["gain_text"]) == egain)
    names = {0: "random", 1: "round_robin", 2: "min_qpm", 3: "infaas_pp", 4: "llumnix_minus",
             5: "block_predictive"}
    loops = int(rows["result"]["n_tested"].sum())
    return {"metric": "run_capacity closed loops/s (device-resident, every policy)",
            "value": loops / gpu_s, "unit": "closed loops/s", "wall_s": gpu_s, "closed_loops": loops,
            "baseline": names[base], "baseline_capacity_qps": bcap,
            "rows": [{"policy": names[int(r["policy"])], "capacity_qps": float(r["result"]["capacity_qps"]),
                      "gain": r["gain_text"].decode()} for r in rows],
            "identical_to_reference": same,
            "config": "8 instances x P1 profile, 800 requests, QPS 1-40 (+tenths), SLO p99 TTFT < 3 s, seed 1",
            "cpu_baseline": {"value": loops / ref_s, "unit": "closed loops/s", "wall_s": ref_s,
                             "cores": threads, "kind": "reference",
                             "sample": "the same capacity searches, every (policy, qps) closed loop on "
                                       "a pool of all host threads (ref_sweep)"}}


def capacity_sweep(local: int):
    """BASELINE configs[4]: the auto-provisioning capacity sweep on device-resident
    closed loops (bsg_sweep_run) — the full grid on this GPU, and a 9-cell subset
    timed against the reference's capacity_search on all host cores, scheduled
    at (cell, qps) granularity like the GPU side (ref_sweep)."""
    from oracle.oracle import Reference
    from paper_2508_03611_b200 import native, sweep
    threads = os.cpu_count() or 1
    prof = sweep.load_profiles()
    native.sweep_run(local, sweep.make_cells([4], prof, request_cap=50, qps_max=2)[0][:1], threads=threads)
    full, _ = sweep.make_cells([4, 8, 16, 32, 64, 128], prof, request_cap=400, qps_max=64)
    t0 = time.perf_counter()
    fo = native.sweep_run(local, full, threads=threads)
    full_s = time.perf_counter() - t0
    sub, _ = sweep.make_cells([4, 16, 64], prof, request_cap=300, qps_max=24)
    t0 = time.perf_counter()
    so = native.sweep_run(local, sub, threads=threads)
    sub_s = time.perf_counter() - t0
    rr, ref_s = Reference().sweep(sub, threads=threads)
    same = bool((so["status"] == rr["status"]).all() and so["result"].tobytes() == rr["result"].tobytes())
    scen_sub = int(so["whatif_scenarios"].sum())
    return {"metric": "capacity-sweep what-if scenarios/s (device-resident closed loops)",
            "full_grid": {"value": int(fo["whatif_scenarios"].sum()) / full_s, "wall_s": full_s,
                          "closed_loops": int(fo["result"]["n_tested"].sum()),
                          "cells": "instances 4-128 x 3 profiles x QPS 1-64 (+tenths), 400 requests"},
            "subset": {"value": scen_sub / sub_s, "wall_s": sub_s,
                       "cells": "instances 4,16,64 x 3 profiles x QPS 1-24 (+tenths), 300 requests",
                       "capacities_identical_to_reference": same},
            "cpu_baseline": {"value": scen_sub / ref_s, "unit": "scenarios/s", "wall_s": ref_s,
                             "cores": threads, "kind": "reference",
                             "sample": "the subset's capacity searches, every (cell, qps) closed "
                                       "loop on a pool of all host threads (ref_sweep)"}}


def cpu_baseline(ss, cfg):
    """The reference predict() (oracle/_ref, built from /root/reference) timed on
    this host's cores over the same captured scenario set (bounded sample:
    the whole 60,000-scenario set, best of 3 passes); also returns the
    reference's results on that set for the parity count."""
    from oracle.oracle import Reference
    ref = Reference()
    threads = os.cpu_count() or 1
    secs = ref.time_predict(cfg, ss, threads=threads, reps=3)
    exp = ref.predict_batch(cfg, ss, threads=threads)
    return ({"value": len(ss) / secs, "unit": "scenarios/s", "cores": threads,
             "kind": "reference",
             "sample": f"all {len(ss)} cfg2 scenarios, best of 3 passes, {threads} std::threads, "
                       "predict(req, nullptr) (cache off, bit-identical to exact)"}, exp)


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path on all
    host cores, same workload (captured by the reference's own driver loop)."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return None
    from oracle.oracle import Reference
    ref = Reference()
    w, cfg, spec = workload("cfg2")
    _, _, ss = ref.replay(w, cfg, spec)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        ref.time_predict(cfg, ss, threads=threads, reps=1)
    times = [ref.time_predict(cfg, ss, threads=threads, reps=1) for _ in range(args.steps)]
    total = sum(times)
    value = len(ss) * args.steps / total
    return {
        "impl": "reference",
        "metric": "simulated what-if scenarios/sec (predict() fanout, cfg2 12 instances)",
        "value": value, "unit": "scenarios/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "int32+f64", "data": "synthetic (reference generators, seeded)",
        "config": {**workload_desc(), "scenarios_per_step": len(ss), "entries": ss.n_entries,
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "scenarios/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"all {len(ss)} cfg2 scenarios per step, {threads} std::threads"},
        "e2e": {"value": value, "unit": "scenarios/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-latency", dest="latency", action="store_false")
    ap.add_argument("--no-extra", dest="extra", action="store_false",
                    help="skip the cfg1/cfg3/cfg5 side measurements")
    ap.add_argument("--dist-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args, argv))
    if args.dist_probe:
        line = dist_probe()
    else:
        line = run_reference(args) if args.impl == "reference" else run_gpu(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

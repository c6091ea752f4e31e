"""GPU parity of the sweep-driver row beyond BlockPredictive:
the heuristic dispatch policies (pick_heuristic, scheduler.cpp:68-113) and the
dispatch-overhead mode (driver.cpp:213-231) inside the device-resident closed
loop (K5) and the host-driven one, run_sweep's SweepCell table
(driver.cpp:333-390) and run_capacity's capacity table with its gains
(driver.cpp:392-427) — each against the reference's own functions
(oracle/_ref), bit-exactly."""
import os

import numpy as np
import pytest

from paper_2508_03611_b200 import abi, native

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8
FIELDS = ("instance", "dispatch_ticks", "first_token_ticks", "finish_ticks", "preempt_count")
HEURISTICS = [abi.POLICY_RANDOM, abi.POLICY_ROUND_ROBIN, abi.POLICY_MIN_QPM, abi.POLICY_INFAAS_PP,
              abi.POLICY_LLUMNIX_MINUS]


def check_runs(ctx, ref, cfg, cases, host=True):
    """cases: [(workload, spec)]; device closed loops in one batched launch,
    each also run by the host-driven loop, against run_experiment + aggregate."""
    ctx.set_configs(cfg)
    got = ctx.replay_device([(w, sp, 0) for w, sp in cases])
    reps = ctx.last_reports.copy()
    for (w, sp), (st, out, summ), rep in zip(cases, got, reps):
        exp, esum = ref.run_experiment(w, cfg, sp)
        tag = (int(sp["policy"][0]), float(sp["dispatch_overhead_s"][0]), int(sp["provision_kind"][0]))
        assert st == abi.OK, tag
        for f in FIELDS:
            assert np.array_equal(out[f], exp[f]), (tag, f, np.nonzero(out[f] != exp[f])[0][:5])
        for f in ("total_preemptions", "instances_provisioned", "final_instance_count"):
            assert int(summ[f]) == int(esum[f]), (tag, f)
        erep = ref.run_report(w, cfg, sp)
        assert rep.tobytes() == erep.tobytes(), (tag, rep, erep)
        if host:
            hout, hsum, _ = ctx.replay(w, cfg, sp)
            ctx.set_configs(cfg)
            for f in FIELDS:
                assert np.array_equal(hout[f], exp[f]), ("host", tag, f)
    return got


@pytest.mark.parametrize("policy", HEURISTICS)
def test_device_closed_loop_heuristics_match_reference(ctx, ref, policy):
    """Every heuristic policy on K5 (and the host loop): same decisions and
    timelines as the reference driver, static and preempt provisioning (the
    heuristics then ask predict() for the chosen instance, driver.cpp:202-209)."""
    cfg = abi.make_config()
    cases = []
    for q, s, ni in [(8.0, 1, 4), (24.0, 2, 12), (40.0, 3, 3)]:
        w = abi.make_workload(count=300, qps=q, arrival_seed=s, estimator_kind=2, estimator_seed=s)
        cases.append((w, abi.make_replay_spec(ni, policy=policy, capture=0, policy_seed=s + 10)))
    w = abi.make_workload(count=400, qps=24.0, arrival_seed=5)
    cases.append((w, abi.make_replay_spec(4, policy=policy, capture=0, policy_seed=3,
                                          provision_kind=abi.PROVISION_PREEMPT, max_instances=9,
                                          threshold_s=15.0, cold_start_s=5.0, cooldown_s=3.0)))
    check_runs(ctx, ref, cfg, cases)


@pytest.mark.parametrize("policy", [abi.POLICY_BLOCK_PREDICTIVE, abi.POLICY_LLUMNIX_MINUS,
                                    abi.POLICY_ROUND_ROBIN])
def test_dispatch_overhead_matches_reference(ctx, ref, policy):
    """Overhead mode: the decision at the arrival, the request lands overhead
    seconds later (kDispatch events interleaved with the instance's steps and
    later arrivals). Overheads below, near and above the inter-arrival gap, and
    one that rounds to zero ticks (lands in the same instant, after it)."""
    cfg = abi.make_config()
    cases = []
    for o, q, s, ni in [(0.08, 12.0, 1, 4), (0.5, 20.0, 2, 6), (2.5, 30.0, 3, 12), (1e-10, 40.0, 4, 3)]:
        w = abi.make_workload(count=300, qps=q, arrival_seed=s)
        cases.append((w, abi.make_replay_spec(ni, policy=policy, capture=0, policy_seed=s,
                                              dispatch_overhead_s=o)))
    w = abi.make_workload(count=300, qps=30.0, arrival_seed=6)
    cases.append((w, abi.make_replay_spec(4, policy=policy, capture=0, dispatch_overhead_s=0.3,
                                          provision_kind=2, max_instances=8, threshold_s=10.0,
                                          cold_start_s=2.0, cooldown_s=1.0)))
    got = check_runs(ctx, ref, cfg, cases)
    # test_driver.cpp:90-102: every finished request reports the constant
    rep = ctx.last_reports
    assert abs(rep[0]["mean_overhead_s"] - 0.08) < 1e-9 * 0.08 + 1e-15
    assert rep[0]["mean_overhead_s"] > 0 and got[0][0] == abi.OK


def test_run_sweep_matches_reference(ref):
    """bsg_run_sweep == the reference's run_sweep: every SweepCell field of the
    (policy x qps x seed) table, in the reference's cell order."""
    cfg = abi.make_config()
    w = abi.make_workload(count=250)
    spec = abi.make_replay_spec(6, capture=0)
    pols = [abi.POLICY_ROUND_ROBIN, abi.POLICY_LLUMNIX_MINUS, abi.POLICY_MIN_QPM,
            abi.POLICY_BLOCK_PREDICTIVE]
    qps, seeds = [4.0, 9.5, 30.0], [1, 7]
    got = native.run_sweep(0, w, cfg, spec, pols, qps, seeds, threads=THREADS)
    exp = ref.run_sweep(w, cfg, spec, pols, qps, seeds, jobs=THREADS)
    assert len(got) == len(exp) == len(pols) * len(qps) * len(seeds)
    assert (got["ok"] == 1).all() and (exp["ok"] == 1).all()
    for f in got.dtype.names:
        if f == "status":
            continue
        assert np.array_equal(got[f], exp[f]), (f, got[f], exp[f])


def test_run_capacity_matches_reference(ref):
    """bsg_run_capacity == the reference's run_capacity: the capacity row of
    every policy (baseline appended), its tested count and bracket, and the
    gains table's formatted percentages."""
    cfg = abi.make_config()
    w = abi.make_workload(count=200)
    spec = abi.make_replay_spec(4, capture=0)
    pols = [abi.POLICY_BLOCK_PREDICTIVE, abi.POLICY_INFAAS_PP, abi.POLICY_ROUND_ROBIN]
    base = abi.POLICY_LLUMNIX_MINUS
    st, exp, ebase = ref.run_capacity(w, cfg, spec, pols, base, 3, 1, 16, 3.0)
    assert st == 0
    got, gbase = native.run_capacity(0, w, cfg, spec, pols, base, 3, 1, 16, 3.0, threads=THREADS)
    assert gbase == ebase and len(got) == len(exp) == 4
    assert (got["status"] == abi.OK).all()
    for f in ("policy", "result", "has_gain", "gain_text"):
        assert got[f].tobytes() == exp[f].tobytes(), (f, got[f], exp[f])
    assert any(got["has_gain"])


@pytest.mark.parametrize("cfg_kw", [
    dict(local_policy=1, total_blocks=260, max_batch_size=40, block_size=8,       # prefill priority
         _wl=dict(max_prompt_tokens=1024, max_output_tokens=1024)),              # under KV pressure
    dict(block_size=12, total_blocks=1500, max_batch_size=100, chunk_budget=600),  # K = 4, non-pow2
    dict(cache_mode=2, context_bucket=128, total_blocks=400),                      # bucketed what-ifs
])
def test_policies_and_overhead_across_configs(ctx, ref, cfg_kw):
    """Every policy with and without dispatch overhead, and preempt / relief
    provisioning, on instance configs beyond the default: K5 and the host loop
    against run_experiment + aggregate."""
    cfg_kw = dict(cfg_kw)
    wl = cfg_kw.pop("_wl", {})
    cfg = abi.make_config(**cfg_kw)
    cases = []
    for i, pol in enumerate(HEURISTICS + [abi.POLICY_BLOCK_PREDICTIVE]):
        w = abi.make_workload(count=200, qps=10.0 + 4 * i, arrival_seed=i + 1, **wl)
        cases.append((w, abi.make_replay_spec(3 + i % 3, policy=pol, capture=0, policy_seed=i,
                                              dispatch_overhead_s=(0.0, 0.15, 1.2)[i % 3])))
    w = abi.make_workload(count=250, qps=20.0, arrival_seed=9, **wl)
    cases.append((w, abi.make_replay_spec(2, policy=abi.POLICY_LLUMNIX_MINUS, capture=0, dispatch_overhead_s=0.2,
                                          provision_kind=abi.PROVISION_PREEMPT, max_instances=5,
                                          threshold_s=6.0, cold_start_s=2.0, cooldown_s=1.0)))
    cases.append((w, abi.make_replay_spec(2, policy=abi.POLICY_BLOCK_PREDICTIVE, capture=0,
                                          dispatch_overhead_s=0.05, provision_kind=2, max_instances=5,
                                          threshold_s=6.0, cold_start_s=2.0, cooldown_s=0.0)))
    check_runs(ctx, ref, cfg, cases)


def test_run_sweep_with_overhead_and_provisioning(ref):
    """run_sweep over a base spec with dispatch overhead and preempt
    provisioning (spec_for_cell keeps both), every row equal."""
    cfg = abi.make_config()
    w = abi.make_workload(count=200)
    spec = abi.make_replay_spec(3, capture=0, dispatch_overhead_s=0.1, provision_kind=abi.PROVISION_PREEMPT,
                                max_instances=6, threshold_s=8.0, cold_start_s=3.0, cooldown_s=2.0)
    pols = [abi.POLICY_RANDOM, abi.POLICY_INFAAS_PP, abi.POLICY_BLOCK_PREDICTIVE]
    got = native.run_sweep(0, w, cfg, spec, pols, [6.0, 20.0], [3], threads=THREADS)
    exp = ref.run_sweep(w, cfg, spec, pols, [6.0, 20.0], [3], jobs=THREADS)
    for f in got.dtype.names:
        if f != "status":
            assert np.array_equal(got[f], exp[f]), (f, got[f], exp[f])


def test_sweep_and_capacity_error_semantics(ref):
    """An unservable workload (a request needs more blocks than an instance has):
    run_sweep records every cell as failed (the reference's ok = false), and
    run_capacity fails as a whole (the reference throws out of run_capacity).
    A policy with no capacity at qps_min: its row says NO_CAPACITY (the
    reference's capacity_search throws NoCapacityError for it), the others are
    the reference's capacity_search results."""
    cfg = abi.make_config(total_blocks=40)
    w = abi.make_workload(count=100)
    spec = abi.make_replay_spec(3, capture=0)
    got = native.run_sweep(0, w, cfg, spec, [abi.POLICY_ROUND_ROBIN, abi.POLICY_BLOCK_PREDICTIVE], [5.0], [1])
    exp = ref.run_sweep(w, cfg, spec, [abi.POLICY_ROUND_ROBIN, abi.POLICY_BLOCK_PREDICTIVE], [5.0], [1])
    assert (got["ok"] == 0).all() and (exp["ok"] == 0).all()
    assert (got["status"] == abi.TOO_LARGE_CANDIDATE).all()
    with pytest.raises(native.BsgError):
        native.run_capacity(0, w, cfg, spec, [abi.POLICY_BLOCK_PREDICTIVE], abi.POLICY_LLUMNIX_MINUS, 1, 1, 4, 3.0)
    assert ref.run_capacity(w, cfg, spec, [abi.POLICY_BLOCK_PREDICTIVE], abi.POLICY_LLUMNIX_MINUS, 1, 1, 4, 3.0)[0] < 0
    # no capacity at qps_min for some policies (tight SLO, high qps_min)
    cfg = abi.make_config()
    w = abi.make_workload(count=300)
    pols = [abi.POLICY_BLOCK_PREDICTIVE, abi.POLICY_RANDOM, abi.POLICY_INFAAS_PP]
    rows, _ = native.run_capacity(0, w, cfg, spec, pols, abi.POLICY_LLUMNIX_MINUS, 2, 8, 14, 0.5, threads=THREADS)
    statuses = set()
    for r in rows:
        sp = spec.copy()
        sp["policy"] = r["policy"]
        st, res, _ = ref.capacity_search(w, cfg, sp, 2, 8, 14, 0.5)
        assert int(r["status"]) == st, (int(r["policy"]), int(r["status"]), st)
        if st == abi.OK:
            assert r["result"].tolist() == res.tolist()
        statuses.add(st)
    assert abi.NO_CAPACITY in statuses, statuses


def test_closed_loop_fuzz_matches_reference(ctx, ref):
    """Seeded random closed loops — instance configs (block size, blocks, batch,
    budget, scheduling policy, latency cache), workloads (shape, estimator, load),
    dispatch policies, dispatch overhead and provisioning — on K5 in one batched
    launch per config, against run_experiment + aggregate."""
    rng = np.random.default_rng(20261017)
    for case in range(16):
        bs = int(rng.choice([8, 12, 16, 32]))
        cfg = abi.make_config(block_size=bs, total_blocks=int(rng.integers(3000, 9000)) // bs,
                              max_batch_size=int(rng.choice([8, 24, 48, 64, 100, 160])),
                              chunk_budget=int(rng.choice([256, 512, 1024])),
                              local_policy=int(rng.integers(0, 2)), cache_mode=int(rng.choice([0, 1, 2])),
                              context_bucket=int(rng.choice([64, 256])))
        cases = []
        for _ in range(4):
            w = abi.make_workload(count=int(rng.integers(80, 220)), qps=float(rng.uniform(2, 30)),
                                  arrival_seed=int(rng.integers(1, 1 << 30)),
                                  prompt_median=float(rng.uniform(100, 400)),
                                  output_median=float(rng.uniform(60, 300)),
                                  max_prompt_tokens=1024, max_output_tokens=1024,
                                  estimator_kind=int(rng.choice([0, 2])),
                                  estimator_seed=int(rng.integers(1, 1000)))
            kind = int(rng.choice([0, 0, 1, 2]))
            ni = int(rng.integers(1, 7))
            sp = abi.make_replay_spec(ni, policy=int(rng.integers(0, 6)), objective=int(rng.integers(0, 2)),
                                      capture=0, policy_seed=int(rng.integers(0, 1 << 30)),
                                      provision_kind=kind, max_instances=ni + int(rng.integers(0, 4)),
                                      threshold_s=float(rng.uniform(2, 20)), cold_start_s=float(rng.uniform(0, 5)),
                                      cooldown_s=float(rng.choice([0.0, 1.0, 3.0])),
                                      dispatch_overhead_s=float(rng.choice([0.0, 0.0, 0.05, 0.7])))
            cases.append((w, sp))
        check_runs(ctx, ref, cfg, cases, host=(case % 2 == 0))

"""GPU parity tests proper: the sm_100a kernels, called through the C-ABI,
against the reference (oracle/_ref/libblocksim_ref.so, travels prebuilt) and
the committed golden vectors. Bit-exact on ticks, steps, statuses, per-step
batch composition / allocation / preemption fingerprints, and decisions.
(North star allows 1e-6 relative on latencies; we hold ourselves to equality.)"""
import numpy as np
import pytest

from paper_2508_03611_b200 import abi, native
from oracle.oracle import compare_to_ref
from scenarios import fuzz_set, kat_set
from test_oracle import load_golden

pytestmark = pytest.mark.gpu


def run(ctx, cfgs, ss):
    ctx.set_configs(cfgs)
    return ctx.predict_batch(ss)


@pytest.mark.parametrize("fixture", ["reference_kats.json", "fuzz_400_seed7.json"])
def test_gpu_matches_golden(ctx, fixture):
    names, cfgs, ss, exp = load_golden(fixture)
    got = run(ctx, cfgs, ss)
    bad = compare_to_ref(got, exp)
    assert not bad.any(), [(names[i], got[i], exp[i]) for i in np.nonzero(bad)[0][:5]]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_gpu_matches_reference_fuzz(ctx, ref, seed):
    cfgs, ss = fuzz_set(seed, 20000)
    got = run(ctx, cfgs, ss)
    exp = ref.predict_batch(cfgs, ss, threads=8)
    bad = compare_to_ref(got, exp)
    assert bad.sum() == 0, [(i, got[i], exp[i]) for i in np.nonzero(bad)[0][:5]]


@pytest.mark.parametrize("win_j,cyc", [("1", "1"), ("4", "1"), ("4", "0"), ("1", "0"), ("8", "0")])
def test_gpu_trace_matches_reference(ctx, ref, monkeypatch, win_j, cyc):
    """Per-step batch composition, allocations, preemption victims, first
    tokens, completions and durations (bsg_step_record) for every step — with
    the event-skipping window at both widths the kernels use (32 and 128 steps
    per iteration), so every window-retired step is checked too."""
    monkeypatch.setenv("BSG_TRACE_J", win_j)
    monkeypatch.setenv("BSG_TRACE_CYC", cyc)
    cfgs, ss = fuzz_set(12, 400)
    ctx.set_configs(cfgs)
    names, kc, ks = kat_set()
    for cf, s in ((cfgs, ss), (kc, ks)):
        ctx.set_configs(cf)
        for i in range(len(s)):
            a, ta = ctx.trace(s, i, cap=8192)
            b, tb = ref.trace(cf, s, i, cap=8192)
            assert a["status"] == b["status"], (i, a, b)
            assert len(ta) == len(tb), (i, len(ta), len(tb))
            assert np.array_equal(ta, tb), (i, np.nonzero(ta != tb)[0][:3])


@pytest.mark.parametrize("win_j", ["1", "4"])
def test_gpu_trace_kv_pressure_cycles(ctx, ref, monkeypatch, win_j):
    """cfg3-shaped scenarios (KV pressure, chunked prefill, deep queues) spend
    most general steps in admit / self-preempt cycles, which the windows
    absorb: every step record (plan, preemption victim, free blocks, duration)
    must equal the reference's, and the scenarios must actually contain cycles."""
    monkeypatch.setenv("BSG_TRACE_J", win_j)
    cfg = abi.make_config()
    w = abi.make_workload(count=1000, prompt_median=600, output_median=600, qps=5.0, arrival_seed=1)
    _, _, ss = ref.replay(w, cfg, abi.make_replay_spec(12))
    ctx.set_configs(cfg)
    cycles = 0
    for i in range(len(ss) - 1, len(ss) - 1 - 48 * 12, -12):  # late arrivals queue deepest
        a, ta = ctx.trace(ss, i, cap=1 << 15)
        b, tb = ref.trace(cfg, ss, i, cap=1 << 15)
        assert a["status"] == b["status"] and len(ta) == len(tb), (i, a, b)
        assert np.array_equal(ta, tb), (i, np.nonzero(ta != tb)[0][:3])
        A = (tb["n_prefill"] == 1) & (tb["n_preempted"] == 0)
        B = (tb["n_prefill"] == 0) & (tb["n_preempted"] == 1)
        cycles += int((A[:-1] & B[1:]).sum())
    assert cycles > 5000, cycles


def test_gpu_kats(ctx):
    names, cfgs, ss = kat_set()
    r = run(ctx, cfgs, ss)
    i = names.index("predictor_empty_instance")
    prefill = round((0.01 + 512 * 1e-4) * 1e9)
    total = prefill + sum(round((0.01 + 1e-3 + c * 1e-7) * 1e9) for c in range(513, 522))
    assert r[i]["e2e_ticks"] == total and r[i]["ttft_ticks"] == prefill  # test_driver.cpp:16-36
    assert r[names.index("predictor_impossible")]["status"] == abi.TOO_LARGE_CANDIDATE
    assert r[names.index("predictor_across_0")]["e2e_ticks"] < r[names.index("predictor_across_2")]["e2e_ticks"]


@pytest.mark.parametrize("cfgname,kw,n_inst", [
    ("cfg1", dict(count=1000, estimator_kind=2, estimator_seed=1, qps=10, arrival_seed=1), 4),
    ("cfg2", dict(count=5000, estimator_kind=0, qps=27, arrival_seed=1), 12),
    ("cfg3", dict(count=600, prompt_median=600, output_median=600, qps=4.5, arrival_seed=1), 12),
])
def test_gpu_matches_reference_on_replay_captures(ctx, ref, cfgname, kw, n_inst):
    """Scenario sets a BlockPredictive closed loop evaluates (captured by the
    reference's own driver loop): identical per-scenario results."""
    cfg = abi.make_config()
    w = abi.make_workload(**kw)
    _, _, ss = ref.replay(w, cfg, abi.make_replay_spec(n_inst))
    got = run(ctx, cfg, ss)
    exp = ref.predict_batch(cfg, ss, threads=8)
    assert compare_to_ref(got, exp).sum() == 0


def test_pinned_host_buffers_match_reference(ctx, ref):
    """The e2e path as bench.py drives it: bsg_predict_batch over pinned host
    buffers (pipelined pieces, 3:2:1 chunks, one stream per chunk) equals the
    reference and the pageable-buffer call on the cfg2 capture."""
    import torch
    cfg = abi.make_config()
    w = abi.make_workload(count=5000, estimator_kind=0, qps=27, arrival_seed=1)
    _, _, ss = ref.replay(w, cfg, abi.make_replay_spec(12))
    ctx.set_configs(cfg)
    pinned = [torch.from_numpy(c).pin_memory() for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
    pscen = torch.from_numpy(ss.scenarios.view(np.uint8)).pin_memory()
    host = abi.ScenarioSet(*[p.numpy() for p in pinned], pscen.numpy().view(abi.scenario_dtype))
    pout = torch.full((len(ss) * abi.result_dtype.itemsize,), 0xAB, dtype=torch.uint8).pin_memory()
    out = pout.numpy().view(abi.result_dtype)
    ctx.predict_batch(host, out=out)
    exp = ref.predict_batch(cfg, ss, threads=8)
    assert compare_to_ref(out, exp).sum() == 0
    assert np.array_equal(out, ctx.predict_batch(ss))


@pytest.mark.parametrize("kw,n_inst,policy", [
    (dict(count=1000, estimator_kind=2, estimator_seed=1, qps=10, arrival_seed=1), 4,
     abi.POLICY_BLOCK_PREDICTIVE),
    (dict(count=1500, qps=27, arrival_seed=2), 12, abi.POLICY_BLOCK_PREDICTIVE),
    (dict(count=800, qps=9, arrival_seed=5), 4, abi.POLICY_LLUMNIX_MINUS),
    (dict(count=800, qps=9, arrival_seed=5), 4, abi.POLICY_INFAAS_PP),
    (dict(count=500, qps=9, arrival_seed=5), 3, abi.POLICY_RANDOM),
])
def test_closed_loop_decisions_match_reference(ctx, ref, kw, n_inst, policy):
    """Per-arrival decisions, dispatch/first-token/finish ticks and preemption
    counts of the GPU-driven closed loop equal the reference's run_experiment."""
    cfg = abi.make_config()
    w = abi.make_workload(**kw)
    spec = abi.make_replay_spec(n_inst, policy=policy, capture=1, policy_seed=3)
    got, gp, gss = ctx.replay(w, cfg, spec)
    exp, ep = ref.run_experiment(w, cfg, spec)
    assert np.array_equal(got["instance"], exp["instance"])
    assert np.array_equal(got, exp) and gp.tolist() == ep.tolist()


def test_dispatch_argmin_ties_lowest_id(ctx):
    # test_scheduler.cpp:178-203: identical snapshots tie -> lowest id wins,
    # whatever order the ids arrive in.
    cfg = abi.make_config()
    snap = ([(64, 100, 64, 3)] * 5, [])
    ss = abi.ScenarioSet.from_snapshots([snap] * 4, [(256, 32)] * 4)
    ctx.set_configs(cfg)
    chosen, per = ctx.dispatch(ss, np.array([9, 4, 7, 11], np.int32), 4)
    assert chosen[0] == 4 and len(set(per["e2e_ticks"].tolist())) == 1


@pytest.mark.parametrize("n_inst,n_samples,qps", [(8, 64, 14.0), (64, 256, 130.0)])
def test_mc_dispatch_matches_reference_loop(ctx, ref, n_inst, n_samples, qps):
    """cfg4 semantics: per-instance score = sum over MC length samples of the
    e2e ticks the reference predict() returns with that sample as the
    candidate's length; prefix-shared GPU simulation must give identical
    per-sample e2e, scores and decisions."""
    from paper_2508_03611_b200 import native
    from oracle.oracle import mc_reference_dispatch
    cfg = abi.make_config()
    w = abi.make_workload(count=400, qps=qps, arrival_seed=4)
    _, _, cap = ref.replay(w, cfg, abi.make_replay_spec(n_inst))
    groups = [50, 200, 399] if n_inst == 64 else list(range(100, 400, 25))
    rows = np.concatenate([cap.scenarios[g * n_inst:(g + 1) * n_inst] for g in groups])
    ss = abi.ScenarioSet(cap.prompt, cap.est, cap.prefill, cap.decoded, rows)
    lengths = np.stack([native.mc_lengths(int(rows[i * n_inst]["cand_est"]), g, n_samples)
                        for i, g in enumerate(groups)])
    ctx.set_configs(cfg)
    ids = np.tile(np.arange(n_inst, dtype=np.int32), len(groups))
    chosen, scores, samples, _ = ctx.dispatch_mc(ss, ids, n_inst, lengths, want_samples=True)
    e_chosen, e_scores, e_samples = mc_reference_dispatch(ref, cfg, ss, n_inst, lengths)
    assert np.array_equal(samples, e_samples)
    assert np.array_equal(scores, e_scores)
    assert np.array_equal(chosen, e_chosen)


@pytest.mark.parametrize("kind,policy", [
    (abi.PROVISION_PREEMPT, abi.POLICY_BLOCK_PREDICTIVE),
    (abi.PROVISION_PREEMPT, abi.POLICY_ROUND_ROBIN),
    (abi.PROVISION_RELIEF, abi.POLICY_BLOCK_PREDICTIVE),
])
def test_autoscaler_closed_loop_matches_reference(ctx, ref, kind, policy):
    """Auto-provisioning (autoscaler.cpp:36-52, driver.cpp:197-269): instances
    added mid-run on predicted (preempt) or realized (relief) latency; every
    decision, timeline and the provisioning totals equal run_experiment."""
    cfg = abi.make_config()
    w = abi.make_workload(count=1200, qps=30.0, arrival_seed=3)
    spec = abi.make_replay_spec(3, policy=policy, capture=0, provision_kind=kind, max_instances=8,
                                threshold_s=8.0, cold_start_s=5.0, cooldown_s=2.0)
    got, gs, _ = ctx.replay(w, cfg, spec)
    exp, es = ref.run_experiment(w, cfg, spec)
    assert es["instances_provisioned"] > 0  # the scenario actually provisions
    assert np.array_equal(got, exp) and gs.tolist() == es.tolist()
    from paper_2508_03611_b200 import native
    host_fields = [f for f in abi.report_dtype.names if not f.startswith("free_blocks")]
    rep, exp_rep = native.aggregate(got, gs), ref.run_report(w, cfg, spec)
    assert [rep[f] for f in host_fields] == [exp_rep[f] for f in host_fields]


def test_capacity_search_matches_reference(ctx, ref):
    """capacity_search (metrics.cpp:139-178) over BlockPredictive closed loops
    (GPU what-ifs) equals the reference's run_capacity runner: same tested
    (qps, pass) sequence, bracket and capacity."""
    cfg = abi.make_config()
    w = abi.make_workload(count=600, request_cap=400)
    spec = abi.make_replay_spec(2, capture=0)
    st, got, tested = ctx.capacity_search(w, cfg, spec, seed=7, qps_min=1, qps_max=16, slo=1.0)
    est, exp, etested = ref.capacity_search(w, cfg, spec, seed=7, qps_min=1, qps_max=16, slo=1.0)
    assert st == est == abi.OK
    assert tested == etested
    assert got.tolist() == exp.tolist()
    assert 1 < got["capacity_qps"] < 16  # a real bracket, with tenths tested


@pytest.mark.parametrize("path,provision", [
    ("device", None),
    ("device", dict(provision_kind=abi.PROVISION_PREEMPT, extra_instances=2, threshold_s=4.0,
                    cold_start_s=2.0, cooldown_s=1.0)),
    ("device", dict(provision_kind=abi.PROVISION_RELIEF, extra_instances=2, threshold_s=6.0,
                    cold_start_s=2.0, cooldown_s=1.0)),
    ("host", None),
])
def test_sweep_cells_match_reference_capacity_search(ref, monkeypatch, path, provision):
    """bsg_sweep_run — device-resident closed loops (batched launches), or the
    host-driven loops (BSG_SWEEP_HOST) — gives, per cell, exactly the
    reference's capacity_search result for that cell's profile, instance count
    and auto-provisioning policy."""
    from paper_2508_03611_b200 import native, sweep
    if path == "host":
        monkeypatch.setenv("BSG_SWEEP_HOST", "1")
    profiles = sweep.load_profiles()
    cells, keys = sweep.make_cells([1, 2], profiles, request_cap=150, qps_max=12, slo=1.0,
                                   provision=provision)
    out = native.sweep_run(0, cells, threads=4)
    for c, o in zip(cells, out):
        w = np.array([c["workload"]], abi.workload_dtype)
        cfg = np.array([c["cfg"]], abi.cfg_dtype)
        spec = np.array([c["spec"]], abi.replay_spec_dtype)
        st, exp, _ = ref.capacity_search(w, cfg, spec, int(c["seed"]), int(c["qps_min"]),
                                         int(c["qps_max"]), float(c["slo_p99_ttft_s"]))
        assert int(o["status"]) == st
        assert o["result"].tolist() == exp.tolist()
        assert o["whatif_scenarios"] > 0


@pytest.mark.parametrize("policy_cfg", [
    dict(),                                                      # chunked prefill, P1
    dict(local_policy=1),                                        # prefill priority
    dict(total_blocks=300, max_batch_size=24),                   # KV pressure: preemptions
    dict(block_size=10, total_blocks=1500, chunk_budget=256),    # non-power-of-two blocks
    dict(cache_mode=2, context_bucket=256, max_batch_size=64),   # bucketed latency cache, K=2
    dict(max_batch_size=160, total_blocks=2000, chunk_budget=1024),  # K=8 member slots
    dict(local_policy=1, total_blocks=260, max_batch_size=40, block_size=8,  # prefill priority
         _wl=dict(max_prompt_tokens=1024, max_output_tokens=1024)),          # under KV pressure
])
def test_device_closed_loop_matches_reference(ctx, ref, policy_cfg):
    """bsg_replay_device (whole closed loop on the GPU) == the reference's own
    run_experiment replay: every request's dispatch instance and tick-exact
    dispatch / first-token / finish times and preemption counts."""
    policy_cfg = dict(policy_cfg)
    wl = policy_cfg.pop("_wl", {})  # keep the workload servable (config.cpp:197-205)
    cfg = abi.make_config(**policy_cfg)
    ctx.set_configs(cfg)
    cases = [(abi.make_workload(count=300, qps=q, arrival_seed=s, estimator_kind=2, estimator_seed=s, **wl),
              ni, obj) for q, s, ni, obj in [(6.0, 1, 4, 0), (14.0, 2, 12, 0), (30.0, 3, 7, 1),
                                              (3.0, 4, 1, 0)]]
    got = ctx.replay_device([(w, abi.make_replay_spec(ni, objective=obj, capture=0), 0)
                             for w, ni, obj in cases])
    for (w, ni, obj), (st, out, summ) in zip(cases, got):
        spec = abi.make_replay_spec(ni, objective=obj, capture=0)
        exp, esum, _ = ref.replay(w, cfg, spec, capture=False)
        host, hsum, _ = ctx.replay(w, cfg, spec)  # the host-driven closed loop, same contract
        ctx.set_configs(cfg)
        assert st == abi.OK
        for f in ("instance", "dispatch_ticks", "first_token_ticks", "finish_ticks", "preempt_count"):
            assert np.array_equal(out[f], exp[f]), (policy_cfg, ni, f, np.nonzero(out[f] != exp[f])[0][:5])
            assert np.array_equal(host[f], exp[f]), ("host", policy_cfg, ni, f)
        assert int(summ["total_preemptions"]) == int(esum["total_preemptions"])
        assert int(hsum["total_preemptions"]) == int(esum["total_preemptions"])
    # the device metric pipeline: aggregate() of every run, bit-identical
    for (w, ni, obj), rep in zip(cases, ctx.last_reports):
        exp = ref.run_report(w, cfg, abi.make_replay_spec(ni, objective=obj, capture=0))
        assert rep.tobytes() == exp.tobytes(), (policy_cfg, ni, rep, exp)


@pytest.mark.parametrize("kind,kw", [
    (abi.PROVISION_PREEMPT, dict(threshold_s=20.0, cold_start_s=5.0, cooldown_s=3.0)),
    (abi.PROVISION_PREEMPT, dict(threshold_s=8.0, cold_start_s=0.0, cooldown_s=0.0)),
    (2, dict(threshold_s=20.0, cold_start_s=5.0, cooldown_s=3.0)),
    (2, dict(threshold_s=10.0, cold_start_s=0.0, cooldown_s=0.0)),
])
def test_device_closed_loop_autoscaler_matches_reference(ctx, ref, kind, kw):
    """Auto-provisioning (preempt: predicted e2e at dispatch; relief: realized
    e2e at completion) inside the device-resident closed loop: same instances
    provisioned, same per-request timeline as the reference driver."""
    cfg = abi.make_config()
    ctx.set_configs(cfg)
    cases = [(abi.make_workload(count=400, qps=q, arrival_seed=s), ni, mx)
             for q, s, ni, mx in [(24.0, 1, 6, 10), (40.0, 2, 3, 9), (12.0, 3, 1, 4)]]
    specs = [abi.make_replay_spec(ni, capture=0, provision_kind=kind, max_instances=mx, **kw)
             for _, ni, mx in cases]
    got = ctx.replay_device([(w, sp, 0) for (w, _, _), sp in zip(cases, specs)])
    for (w, ni, mx), sp, (st, out, summ) in zip(cases, specs, got):
        exp, esum = ref.run_experiment(w, cfg, sp)  # the reference's own run_experiment
        assert st == abi.OK
        assert int(summ["instances_provisioned"]) > 0 or kind == 2
        assert int(summ["instances_provisioned"]) == int(esum["instances_provisioned"])
        assert int(summ["final_instance_count"]) == int(esum["final_instance_count"])
        for f in ("instance", "dispatch_ticks", "first_token_ticks", "finish_ticks", "preempt_count"):
            assert np.array_equal(out[f], exp[f]), (kind, ni, f, np.nonzero(out[f] != exp[f])[0][:5])


@pytest.mark.parametrize("policy_cfg,n_inst,obj", [
    (dict(), 12, 0), (dict(local_policy=1), 5, 1), (dict(total_blocks=300, max_batch_size=24), 7, 0),
    (dict(block_size=12, total_blocks=1500, max_batch_size=100, chunk_budget=600), 3, 0),  # K=4, non-pow2
    (dict(cache_mode=2, context_bucket=128), 6, 1),                                       # bucketed what-ifs
])
def test_fleet_matches_reference(ctx, ref, policy_cfg, n_inst, obj):
    """A fleet (device-resident instance mirror, one launch per dispatch) driven
    by a workload's arrivals reproduces the reference's replay exactly."""
    from paper_2508_03611_b200 import native
    cfg = abi.make_config(**policy_cfg)
    ctx.set_configs(cfg)
    w = abi.make_workload(count=300, qps=14.0, arrival_seed=5, estimator_kind=2, estimator_seed=5)
    p, o, e, t = native.make_workload_host(w)
    fl = native.Fleet(ctx, n_inst, len(p))
    picks = [fl.dispatch(t[k], p[k], e[k], o[k], objective=obj) for k in range(len(p))]
    out, summ = fl.finish(len(p))
    exp, esum, _ = ref.replay(w, cfg, abi.make_replay_spec(n_inst, objective=obj, capture=0),
                              capture=False)
    assert picks == exp["instance"].tolist()
    for f in ("instance", "dispatch_ticks", "first_token_ticks", "finish_ticks", "preempt_count"):
        assert np.array_equal(out[f], exp[f]), (f, np.nonzero(out[f] != exp[f])[0][:5])
    assert int(summ["total_preemptions"]) == int(esum["total_preemptions"])


def test_fleet_mc_dispatch_matches_dispatch_mc(ctx):
    """Monte-Carlo fleet dispatches (prefix-shared samples on the mirror, in
    place): per-instance scores and decisions == bsg_dispatch_mc on the same
    snapshots, exported through the mirror's Status API after each dispatch
    (pre-dispatch snapshot = post-dispatch minus the admitted tail entry)."""
    from paper_2508_03611_b200 import native
    cfg = abi.make_config()
    ctx.set_configs(cfg)
    n_inst, S = 8, 64
    w = abi.make_workload(count=150, qps=12.0, arrival_seed=3)
    p, o, e, t = native.make_workload_host(w)
    fl = native.Fleet(ctx, n_inst, len(p))
    ids = np.arange(n_inst, dtype=np.int32)
    for k in range(len(p)):
        lens = native.mc_lengths(int(e[k]), k, S, seed=7)
        sc = np.zeros(n_inst, np.int64)
        pick = fl.dispatch(t[k], p[k], e[k], o[k], lengths=lens, scores=sc)
        if k % 5:
            continue
        cols, scen, off = [[] for _ in range(4)], np.zeros(n_inst, abi.scenario_dtype), 0
        for i in range(n_inst):
            rn, wn, c = fl.snapshot(i)
            if i == pick:
                wn -= 1
            for j in range(4):
                cols[j].append(c[j][:rn + wn])
            scen[i] = (off, rn, off + rn, wn, p[k], e[k], 0, 0)
            off += rn + wn
        ss = abi.ScenarioSet(*[np.concatenate(c).astype(np.int32) for c in cols], scen)
        exp_pick, exp_scores, _, _ = ctx.dispatch_mc(ss, ids, n_inst, lens)
        assert pick == int(exp_pick[0]) and np.array_equal(sc, exp_scores), (k, sc, exp_scores)
    out, _ = fl.finish(len(p))
    assert (out["finish_ticks"] > 0).all()


def test_wire_predict_json_matches_reference_service(ctx, ref):
    """bsg_predict_json (json_io.cpp schema in, GPU predict, schema out) answers
    like the reference predictor role's /predict (service.cpp:229-241):
    byte-identical bodies — PredictionResult JSON for successes (numbers printed
    with nlohmann's Grisu2 digits, which are not always the shortest form) and
    the error bodies (prediction-failure / bad-schema with the reference's
    message, ids and block counts) otherwise — on KATs, fuzz (every failure
    status), malformed bodies and mixed invalid configs."""
    import json
    names, kc, ks = kat_set()
    fc, fs = fuzz_set(77, 600)
    bodies = [ref.request_json(kc, ks, i) for i in range(len(ks))]
    bodies += [ref.request_json(fc, fs, i) for i in range(len(fs))]
    good = json.loads(bodies[0])
    broken = dict(good)
    del broken["candidate"]
    typo = json.loads(bodies[1])
    typo["snapshot"]["running"] = "not-a-list"
    pol = json.loads(bodies[2])
    pol["instance_config"]["local_policy"] = "round_robin"
    # two DIFFERENT invalid configs mixed with good requests: each bad request
    # fails on its own, every good one is still answered
    bad1 = json.loads(bodies[3])
    bad1["instance_config"]["total_blocks"] = 0
    bad2 = json.loads(bodies[4])
    bad2["instance_config"]["cost_model"]["c0_s"] = 0.0
    bodies += ["{not json", json.dumps(broken), json.dumps(typo), json.dumps(pol), "",
               json.dumps(bad1), json.dumps(bad2)]
    bodies.insert(7, json.dumps(bad2))
    got = ctx.predict_json(bodies)
    n_ok = n_err = 0
    for i, (body, (st, text)) in enumerate(zip(bodies, got)):
        code, exp = ref.service_predict(body)
        assert text == exp, (i, code, text, exp)  # byte-identical, successes and errors
        if code == 200:
            assert st == abi.OK
            n_ok += 1
        else:
            assert st != abi.OK, (i, code, exp)
            n_err += 1
    assert n_ok > 400 and n_err >= 8  # mostly successes, with failures of every kind mixed in


def _trace_text(n, seed, offsets, shuffle=False):
    """A JSONL trace built from a synthetic workload (ids sparse, estimates tagged)."""
    import json
    p, o, e, t = native.make_workload_host(abi.make_workload(count=n, qps=9.0, arrival_seed=seed,
                                                             estimator_kind=2, estimator_seed=seed))
    rng = np.random.default_rng(seed)
    ids = rng.permutation(50 * n)[:n] + 1000
    lines = []
    for i in range(n):
        d = {"id": int(ids[i]), "prompt_tokens": int(p[i]), "output_tokens": int(o[i]),
             "estimated_output_tokens": int(e[i])}
        if offsets:
            d["arrival_offset_s"] = float(t[i]) * 1e-9
        lines.append(json.dumps(d))
    if shuffle:  # arrivals out of record order, with exact ties
        rng.shuffle(lines)
        lines[5] = lines[5].replace(lines[5][lines[5].index('"arrival_offset_s"'):],
                                    lines[6][lines[6].index('"arrival_offset_s"'):])
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("offsets,shuffle,est_kind", [
    (False, False, abi.ESTIMATOR_TRACE), (True, False, abi.ESTIMATOR_TRACE),
    (True, False, abi.ESTIMATOR_NOISY), (True, True, abi.ESTIMATOR_ORACLE)])
def test_trace_closed_loop_matches_reference(ctx, ref, offsets, shuffle, est_kind):
    """A JSONL trace through load_trace -> run_experiment (workload.cpp:51-170,
    driver.cpp:137-160): the host closed loop for any arrival order, and the
    device closed loop (K5) for time-ordered arrivals, tick-exact against the
    reference fed the same records."""
    text = _trace_text(400, 3 + est_kind, offsets, shuffle)
    recs = native.load_trace(text)
    want_recs, err = ref.load_trace(text)
    assert err is None and recs.tobytes() == want_recs.tobytes()
    w = abi.make_workload(qps=8.0, arrival_seed=17, estimator_kind=est_kind, estimator_seed=5)
    cfg = abi.make_config(total_blocks=600, max_batch_size=32)
    for ni in (3, 6):
        spec = abi.make_replay_spec(ni, capture=0)
        ref.set_trace(recs)
        try:
            exp, esum = ref.run_experiment(w, cfg, spec)
            erep = ref.run_report(w, cfg, spec)
        finally:
            ref.set_trace(None)
        host, hsum = ctx.replay_trace(recs, w, cfg, spec)
        assert host.tobytes() == exp.tobytes(), (ni, np.nonzero(host != exp)[0][:5])
        assert int(hsum["total_preemptions"]) == int(esum["total_preemptions"])
        cols = native.trace_workload(recs, w)
        if np.all(np.diff(cols[3]) >= 0):
            ctx.set_configs(cfg)
            [(st, out, summ)] = ctx.replay_device([(cols, spec, 0)])
            assert st == abi.OK
            for f in ("instance", "dispatch_ticks", "first_token_ticks", "finish_ticks", "preempt_count"):
                assert np.array_equal(out[f], exp[f]), (ni, f)
            assert ctx.last_reports[0].tobytes() == erep.tobytes()
        else:
            assert shuffle


def test_edge_inputs(ctx, ref):
    """Empty batches, a scenario naming a config that does not exist (every
    per-config pass writes its INVALID_ARGUMENT verdict, the rest are
    unaffected), and a set whose configs are all unused but one."""
    cfgs, ss = fuzz_set(41, 9000)  # >= the queue threshold: cost order (wide sets) + per-config passes
    ctx.set_configs(cfgs)
    empty = abi.ScenarioSet(ss.prompt[:0], ss.est[:0], ss.prefill[:0], ss.decoded[:0], ss.scenarios[:0])
    assert len(ctx.predict_batch(empty)) == 0
    base = ctx.predict_batch(ss)
    bad = ss.scenarios.copy()
    bad["cfg"][[5, 4000, 8999]] = len(cfgs)
    bad["cfg"][77] = -1
    ss2 = abi.ScenarioSet(ss.prompt, ss.est, ss.prefill, ss.decoded, bad)
    got = ctx.predict_batch(ss2)
    hit = np.zeros(len(ss), bool)
    hit[[5, 77, 4000, 8999]] = True
    assert (got["status"][hit] == abi.INVALID_ARGUMENT).all()
    assert got[~hit].tobytes() == base[~hit].tobytes()
    # only config 0 in use: one pass; results equal the reference's
    one = ss.scenarios.copy()
    one["cfg"] = 0
    ss3 = abi.ScenarioSet(ss.prompt, ss.est, ss.prefill, ss.decoded, one)
    got3 = ctx.predict_batch(ss3)
    exp3 = ref.predict_batch(cfgs, ss3, threads=8)
    assert compare_to_ref(got3, exp3).sum() == 0

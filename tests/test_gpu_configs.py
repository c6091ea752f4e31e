"""GPU parity on the configurations exactly as bench.py measures them
(BASELINE.json configs 1-5): the same captured scenario sets, through the
same device-resident entry point (bsg_predict_batch_device: cost-ordered queue,
the optimistic narrow passes with their window-width vote, the wide retry
kernel), checked bit-exactly against the reference's own predict()
(oracle/_ref) on all host cores. Also: both outcomes of the optimistic pass's
vote forced on the same sets, the cfg5 sweep grid as benchmarked against the
reference's capacity_search, the fleet mirror and the device-sampled MC
dispatch at cfg4's 64 x 256 against the reference looping predict()."""
import os

import numpy as np
import pytest

import bench
from oracle.oracle import compare_to_ref, mc_reference_dispatch
from paper_2508_03611_b200 import abi, native
from scenarios import fuzz_set

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8


def device_predict(ctx, cfg, ss):
    """bench.py's timed path: inputs resident in HBM, bsg_predict_batch_device
    on a dedicated stream with the set's member capacity."""
    import torch
    ctx.set_configs(cfg)
    dev = torch.device("cuda", 0)
    cols = [torch.from_numpy(c).to(dev) for c in (ss.prompt, ss.est, ss.prefill, ss.decoded)]
    scen = torch.from_numpy(ss.scenarios.view(np.uint8)).to(dev)
    out = torch.empty(len(ss) * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    ctx.predict_batch_device([c.data_ptr() for c in cols], scen.data_ptr(), len(ss), out.data_ptr(),
                             stream.cuda_stream, member_capacity=ss.member_capacity(cfg))
    stream.synchronize()
    return np.frombuffer(out.cpu().numpy().tobytes(), dtype=abi.result_dtype).copy()


_sets = {}


def captured(ctx, name):
    if name not in _sets:
        _sets[name] = bench.capture(ctx, name)
    return _sets[name]


def deep_share(cfg, ss):
    sc = ss.scenarios
    need = np.maximum(sc["run_n"], np.minimum(cfg["max_batch_size"][0], sc["run_n"] + sc["wait_n"] + 1))
    return float((need > 32).mean()), float((sc["wait_n"] > 8).mean())


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3_quick", "cfg3"])
def test_benchmarked_set_matches_reference(ctx, ref, name):
    """Every scenario of the set bench.py times, bit-exact (ticks, steps,
    status, detail) against the reference predict()."""
    cfg, ss = captured(ctx, name)
    got = device_predict(ctx, cfg, ss)
    exp = ref.predict_batch(cfg, ss, threads=THREADS)
    bad = compare_to_ref(got, exp)
    assert bad.sum() == 0, (name, int(bad.sum()), [(i, got[i], exp[i]) for i in np.nonzero(bad)[0][:3]])
    assert (got["status"] == abi.OK).all()
    if name.startswith("cfg3"):
        wide, deep = deep_share(cfg, ss)
        # the KV-pressure set really runs the optimistic narrow pass + wide retry
        assert len(ss) >= 8192 and wide > 0.2 and deep > 0.2, (len(ss), wide, deep)
        assert "predict_retry_kernel" in ctx.last_launch, ctx.last_launch


@pytest.mark.parametrize("vote", ["0", "1"])
@pytest.mark.parametrize("which", ["cfg3_quick", "fuzz"])
def test_optimistic_pass_both_votes_match_reference(ctx, ref, monkeypatch, vote, which):
    """The optimistic narrow pass has two window widths and a vote picks one
    per launch; force each outcome on the same sets (>= the queue threshold),
    so both passes are pinned whatever the vote would choose."""
    if which == "fuzz":
        cfgs, ss = fuzz_set(5, 12000)
    else:
        cfgs, ss = captured(ctx, which)
    monkeypatch.setenv("BSG_FORCE_VOTE", vote)
    got = device_predict(ctx, cfgs, ss)
    exp = ref.predict_batch(cfgs, ss, threads=THREADS)
    assert compare_to_ref(got, exp).sum() == 0
    if ss.member_capacity(cfgs) > 32:
        assert "(vote)" in ctx.last_launch, ctx.last_launch


def test_cfg5_grid_as_benchmarked_matches_reference():
    """bench.py's full cfg5 grid (instances 4-128 x 3 profiles x QPS 1-64 +
    tenths, 400 requests, incl. 128 instances at QPS 64) on device-resident
    closed loops: every cell's capacity search result equals the reference's
    capacity_search (ref_sweep: the same runner, pinned to capacity_search in
    test_oracle), point for point."""
    from oracle.oracle import Reference
    from paper_2508_03611_b200 import sweep
    cells, keys = sweep.make_cells([4, 8, 16, 32, 64, 128], sweep.load_profiles(), request_cap=400,
                                   qps_max=64)
    got = native.sweep_run(0, cells, threads=THREADS)
    exp, _ = Reference().sweep(cells, threads=THREADS)
    for k, g, e in zip(keys, got, exp):
        assert int(g["status"]) == int(e["status"]), k
        assert g["result"].tolist() == e["result"].tolist(), (k, g["result"], e["result"])
    assert (got["result"]["n_tested"] >= 64).all()


def test_fleet_64x256_matches_reference_loop(ctx, ref):
    """cfg4 as benchmarked on the device mirror (64 instances, 256 MC samples,
    130 QPS): at sampled dispatches the per-instance scores and the decision
    equal the reference predict() looped over every (instance, sample) on the
    mirror's exported pre-dispatch snapshots."""
    cfg = abi.make_config()
    ctx.set_configs(cfg)
    n_inst, S, count = 64, 256, 600
    w = abi.make_workload(count=count, qps=130.0, arrival_seed=1)
    p, o, e, t = native.make_workload_host(w)
    fl = native.Fleet(ctx, n_inst, count)
    checked = 0
    for k in range(count):
        lens = native.mc_lengths(int(e[k]), k, S, seed=1)
        sc = np.zeros(n_inst, np.int64)
        pick = fl.dispatch(t[k], p[k], e[k], o[k], lengths=lens, scores=sc)
        if k % 40 != 39:
            continue
        cols, scen, off = [[] for _ in range(4)], np.zeros(n_inst, abi.scenario_dtype), 0
        for i in range(n_inst):
            rn, wn, c = fl.snapshot(i)
            if i == pick:
                wn -= 1  # pre-dispatch snapshot: without the admitted request
            for j in range(4):
                cols[j].append(c[j][:rn + wn])
            scen[i] = (off, rn, off + rn, wn, p[k], e[k], 0, 0)
            off += rn + wn
        ss = abi.ScenarioSet(*[np.concatenate(c).astype(np.int32) for c in cols], scen)
        e_chosen, e_scores, _ = mc_reference_dispatch(ref, cfg, ss, n_inst, lens[None, :],
                                                      threads=THREADS)
        assert pick == int(e_chosen[0]) and np.array_equal(sc, e_scores), (k, pick, int(e_chosen[0]))
        checked += 1
    fl.close()
    assert checked == count // 40


def test_device_sampled_dispatch_64x256_matches_reference(ctx, ref):
    """bench.py's cfg4 call (bsg_dispatch_mc_sampled: samples drawn on the
    device inside the call): the drawn lengths equal bsg_mc_lengths and the
    reference's Noisy estimator; scores and decisions equal the reference
    predict() looped over every (instance, sample)."""
    cfg = abi.make_config()
    n_inst, S = 64, 256
    w = abi.make_workload(count=3000, qps=130.0, arrival_seed=1)
    _, _, cap = ctx.replay(w, cfg, abi.make_replay_spec(n_inst))
    ctx.set_configs(cfg)
    ids = np.arange(n_inst, dtype=np.int32)
    for g in (100, 1500, 2999):
        one = cap.compact(g * n_inst + np.arange(n_inst))
        chosen, scores, lens = ctx.dispatch_mc_sampled(one, ids, n_inst, [g], S, seed=1, want_lengths=True)
        host = native.mc_lengths(int(one.scenarios[0]["cand_est"]), g, S, seed=1)
        assert np.array_equal(lens[0], host)
        e_chosen, e_scores, _ = mc_reference_dispatch(ref, cfg, one, n_inst, host[None, :], threads=THREADS)
        assert int(chosen[0]) == int(e_chosen[0]) and np.array_equal(scores, e_scores), g


def test_device_sampler_equals_host_sampler_at_scale(ctx):
    """K3 over 768k samples (3000 requests x 256): the device's Box-Muller
    (CUDA log/cos) lands on the same integer length as the host's (glibc)
    for every sample."""
    cfg = abi.make_config()
    ctx.set_configs(cfg)
    snap = ([(64, 100, 64, 3)] * 2, [])
    n_req, S = 3000, 256
    ests = (np.arange(n_req) * 37) % 4000 + 1
    ss = abi.ScenarioSet.from_snapshots([snap] * n_req, [(32, int(x)) for x in ests])
    _, _, lens = ctx.dispatch_mc_sampled(ss, np.zeros(n_req, np.int32), 1, np.arange(n_req), S, seed=9,
                                         want_lengths=True)
    host = np.stack([native.mc_lengths(int(ests[r]), r, S, seed=9) for r in range(n_req)])
    assert np.array_equal(lens, host), int((lens != host).sum())


def test_fleet_device_sampling_equals_host_lengths(ctx):
    """bsg_fleet_dispatch_sampled (samples drawn on the device inside the call)
    == bsg_fleet_dispatch with bsg_mc_lengths' host samples: same decisions,
    scores and final timelines over a 64-instance stream."""
    cfg = abi.make_config()
    ctx.set_configs(cfg)
    n_inst, S, count = 64, 256, 400
    w = abi.make_workload(count=count, qps=130.0, arrival_seed=2)
    p, o, e, t = native.make_workload_host(w)
    fa, fb = native.Fleet(ctx, n_inst, count), native.Fleet(ctx, n_inst, count)
    for k in range(count):
        sa, sb = np.zeros(n_inst, np.int64), np.zeros(n_inst, np.int64)
        a = fa.dispatch(t[k], p[k], e[k], o[k], lengths=native.mc_lengths(int(e[k]), k, S, seed=3), scores=sa)
        b = fb.dispatch_sampled(t[k], p[k], e[k], o[k], request_id=k, n_samples=S, seed=3, scores=sb)
        assert a == b and np.array_equal(sa, sb), k
    oa, _ = fa.finish(count)
    ob, _ = fb.finish(count)
    assert oa.tobytes() == ob.tobytes()
    fa.close()
    fb.close()


def test_multi_device_fanout_equals_one_device(ctx):
    """bsg_multi_* (one context + worker thread per device; here 3 contexts on
    cuda:0, the host-side splitting and merging is what is under test): batch
    results, per-request decisions and the instance-split Monte-Carlo argmin
    equal the single-context calls bit for bit."""
    cfg, ss = captured(ctx, "cfg2")
    ctx.set_configs(cfg)
    one = ctx.predict_batch(ss)
    m = native.MultiContext([0, 0, 0])
    m.set_configs(cfg)
    assert m.predict_batch(ss, group=12).tobytes() == one.tobytes()
    sub = abi.ScenarioSet(ss.prompt, ss.est, ss.prefill, ss.decoded, ss.scenarios[:12 * 500])
    ids = np.tile(np.arange(12, dtype=np.int32), 500)
    c1, p1 = ctx.dispatch(sub, ids, 12)
    c2, p2 = m.dispatch(sub, ids, 12)
    assert np.array_equal(c1, c2) and p1.tobytes() == p2.tobytes()
    w = abi.make_workload(count=600, qps=130.0, arrival_seed=1)
    _, _, cap = ctx.replay(w, cfg, abi.make_replay_spec(64))
    ctx.set_configs(cfg)
    for g in (50, 300, 599):
        one = cap.compact(g * 64 + np.arange(64))
        ch, sc, _ = ctx.dispatch_mc_sampled(one, np.arange(64, dtype=np.int32), 64, [g], 256, seed=1)
        mc, msc = m.dispatch_mc_sampled(one, np.arange(64, dtype=np.int32), g, 256, seed=1)
        assert mc == int(ch[0]) and np.array_equal(msc, sc), g
    assert m.launches > 0
    m.close()

"""CPU tests: pin the oracle (C restatement) against the reference's own
known-answer tests, the committed golden vectors, and the compiled reference.
No GPU needed."""
import json
import math
import os

import numpy as np
import pytest

from paper_2508_03611_b200 import abi
from oracle.oracle import compare_to_ref
from scenarios import fuzz_set, kat_set

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        g = json.load(f)
    cfgs = np.zeros(len(g["configs"]), abi.cfg_dtype)
    for i, c in enumerate(g["configs"]):
        for k, v in c.items():
            cfgs[i][k] = v
    rows = g["scenarios"]
    ss = abi.ScenarioSet.from_snapshots([(r["running"], r["waiting"]) for r in rows],
                                        [tuple(r["candidate"]) for r in rows],
                                        [r["cfg"] for r in rows])
    exp = np.zeros(len(rows), abi.ref_result_dtype)
    for i, r in enumerate(rows):
        e = r["expect"]
        exp[i] = (float.fromhex(e["e2e_s"]), float.fromhex(e["ttft_s"]),
                  float.fromhex(e["qdelay_s"]), e["steps"], e["status"], e["detail"])
    return [r["name"] for r in rows], cfgs, ss, exp


# ---- reference unit-test KATs, restated --------------------------------------

def test_blocks_needed_kats(c_oracle):
    # test_core.cpp:11-17
    bn = c_oracle.lib.oracle_blocks_needed
    assert [bn(0, 16), bn(100, 16), bn(512, 16), bn(1, 16), bn(17, 16)] == [0, 7, 32, 1, 2]
    # test_core.cpp:19-29 (monotone and tight), same seeded sweep shape
    rng = np.random.default_rng(7)
    for _ in range(2000):
        t, b = int(rng.integers(1, 100001)), int(rng.integers(1, 65))
        k = bn(t, b)
        assert k * b >= t and (k - 1) * b < t and bn(t + 1, b) >= k


def test_simtime_kats(c_oracle):
    # test_core.cpp:61-71: from_seconds(0.0612).ticks() == 61,200,000
    assert c_oracle.lib.oracle_llround_1e9(0.0612) == 61_200_000
    assert c_oracle.lib.oracle_llround_1e9(1.5) + c_oracle.lib.oracle_llround_1e9(0.25) == 1_750_000_000


def test_batch_latency_kats(c_oracle):
    # test_backend.cpp:33-50: 0.0612 (512 prefill tokens), 0.05848 (48 decodes, 4800 context)
    cfg = abi.make_config()
    a = c_oracle.lib.oracle_batch_latency(abi.ptr(cfg), 512, 0, 0)
    b = c_oracle.lib.oracle_batch_latency(abi.ptr(cfg), 0, 48, 4800)
    assert math.isclose(a, 0.0612, rel_tol=1e-12) and math.isclose(b, 0.05848, rel_tol=1e-12)
    assert c_oracle.lib.oracle_batch_latency(abi.ptr(cfg), 612, 0, 0) > a


def test_single_request_timeline_kat(c_oracle):
    # test_driver.cpp:16-36 / test_predictor.cpp:55-73: one 512-token prompt, 10 outputs on an
    # idle instance: prefill step emits the first token, then 9 decodes over context 513..521.
    names, cfgs, ss = kat_set()
    i = names.index("predictor_empty_instance")
    res = c_oracle.predict_batch(cfgs, ss)[i]
    prefill = round((0.01 + 512 * 1e-4) * 1e9)
    total = prefill + sum(round((0.01 + 1e-3 + c * 1e-7) * 1e9) for c in range(513, 522))
    assert res["status"] == abi.OK
    assert res["ttft_ticks"] == prefill and res["e2e_ticks"] == total
    assert res["qdelay_ticks"] == 0 and res["steps"] == 10


def test_plan_kats_via_trace(c_oracle):
    names, cfgs, ss = kat_set()
    # test_backend.cpp:82-96: piggyback chunk 472 behind 40 decoders
    _, tr = c_oracle.trace(cfgs, ss, names.index("backend_piggyback_472"))
    assert tr[0]["n_decode"] == 40 and tr[0]["prefill_tokens"] == 472
    # test_backend.cpp:98-112: prefill priority -> pure prefill batch of 300
    _, tr = c_oracle.trace(cfgs, ss, names.index("backend_prefill_priority"))
    assert tr[0]["n_decode"] == 0 and tr[0]["prefill_tokens"] == 300 + 64
    # test_backend.cpp:114-126: prefill priority, nothing waiting but the candidate:
    # the candidate prefill stalls decoders first, then decode context 10 * 72 (+ candidate)
    _, tr = c_oracle.trace(cfgs, ss, names.index("backend_prefill_priority_decode"))
    assert tr[0]["n_decode"] == 0 and tr[1]["n_decode"] == 11
    assert tr[1]["context_tokens"] == 10 * 72 + 65
    # test_backend.cpp:145-166: shortfall preempts the newest member (6 blocks, 3x2 held)
    res, tr = c_oracle.trace(cfgs, ss, names.index("backend_preempt_newest"))
    assert tr[0]["n_preempted"] >= 1 and tr[0]["n_decode"] == 2


def test_correction_kat(c_oracle, ref):
    # test_predictor.cpp:41-53 and acceptance C8: decoded >= est => est = decoded + 10,
    # for running AND waiting entries; parity against the reference proves the rule.
    names, cfgs, ss = kat_set()
    i = names.index("correction_running_waiting")
    a = c_oracle.predict_batch(cfgs, ss)
    b = ref.predict_batch(cfgs, ss)
    assert not compare_to_ref(a, b)[i]


def test_impossible_candidate_kat(c_oracle):
    # test_predictor.cpp:160-171 -> PredictionError (candidate does not fit)
    names, cfgs, ss = kat_set()
    res = c_oracle.predict_batch(cfgs, ss)[names.index("predictor_impossible")]
    assert res["status"] == abi.TOO_LARGE_CANDIDATE and res["detail"] == 64


def test_loaded_vs_idle_kat(c_oracle):
    # test_predictor.cpp:75-85
    names, cfgs, ss = kat_set()
    r = c_oracle.predict_batch(cfgs, ss)
    busy, idle = r[names.index("predictor_loaded_47")], r[names.index("predictor_empty_instance")]
    assert busy["e2e_ticks"] > idle["e2e_ticks"] and busy["ttft_ticks"] > idle["ttft_ticks"]


# ---- committed golden vectors (generated from the reference) -----------------

@pytest.mark.parametrize("fixture", ["reference_kats.json", "fuzz_400_seed7.json"])
def test_oracle_matches_golden(c_oracle, fixture):
    names, cfgs, ss, exp = load_golden(fixture)
    got = c_oracle.predict_batch(cfgs, ss)
    bad = compare_to_ref(got, exp)
    assert not bad.any(), [names[i] for i in np.nonzero(bad)[0][:10]]


# ---- the compiled reference itself -------------------------------------------

def test_oracle_matches_reference_fuzz(c_oracle, ref):
    cfgs, ss = fuzz_set(11, 6000)
    a = c_oracle.predict_batch(cfgs, ss)
    b = ref.predict_batch(cfgs, ss, threads=os.cpu_count() or 4)
    assert compare_to_ref(a, b).sum() == 0
    # the fuzz set exercises the error taxonomy, not just the happy path
    st = set(np.unique(b["status"]).tolist())
    assert {abi.OK, abi.DEADLOCK, abi.TOO_LARGE_CANDIDATE, abi.TOO_LARGE_RUNNING} <= st


def test_oracle_trace_matches_reference(c_oracle, ref):
    cfgs, ss = fuzz_set(12, 300)
    for i in range(len(ss)):
        a, ta = c_oracle.trace(cfgs, ss, i, cap=8192)
        b, tb = ref.trace(cfgs, ss, i, cap=8192)
        assert a["status"] == b["status"]
        assert np.array_equal(ta, tb), i


def test_reference_shim_replay_equals_run_experiment(ref):
    # The shim's hand replay (used to capture scenario sets for --impl reference)
    # is pinned to the reference's own run_experiment (driver.cpp:316-319).
    w = abi.make_workload(count=600, estimator_kind=2, estimator_seed=1, qps=10, arrival_seed=1)
    cfg = abi.make_config()
    spec = abi.make_replay_spec(4)
    a, pa, ss = ref.replay(w, cfg, spec)
    b, pb = ref.run_experiment(w, cfg, spec)
    assert np.array_equal(a, b) and pa["total_preemptions"] == pb["total_preemptions"]
    assert len(ss) == 4 * 600


def test_reference_sweep_equals_capacity_search(ref):
    """ref_sweep (the all-core cfg5 baseline, parallel over (cell, qps) points)
    gives every cell exactly the reference's own capacity_search result
    (metrics.cpp:139-178): same bracket, capacity, monotone flag, tests."""
    import numpy as np
    from paper_2508_03611_b200 import abi, sweep
    cells, _ = sweep.make_cells([1, 3], sweep.load_profiles(), request_cap=120, qps_max=10, slo=1.0)
    cells["qps_min"][0] = 6  # a cell with no capacity at its lowest qps
    got, secs = ref.sweep(cells, threads=8)
    assert secs > 0
    for c, o in zip(cells, got):
        w = np.array([c["workload"]], abi.workload_dtype)
        st, exp, tested = ref.capacity_search(w, np.array([c["cfg"]], abi.cfg_dtype),
                                              np.array([c["spec"]], abi.replay_spec_dtype),
                                              int(c["seed"]), int(c["qps_min"]), int(c["qps_max"]),
                                              float(c["slo_p99_ttft_s"]))
        assert int(o["status"]) == st
        if st == abi.OK:
            assert o["result"].tolist() == exp.tolist()
    assert (got["status"] == abi.NO_CAPACITY).any() and (got["status"] == abi.OK).any()


def test_reference_run_sweep_rows_equal_run_experiment(ref):
    """ref_run_sweep (the reference's own run_sweep, driver.cpp:333-390) —
    pinned cell by cell to spec_for_cell + run_experiment + aggregate through
    the shim, so the GPU table is checked against the real thing."""
    cfg = abi.make_config()
    w = abi.make_workload(count=150)
    spec = abi.make_replay_spec(3, capture=0)
    pols, qps, seeds = [abi.POLICY_ROUND_ROBIN, abi.POLICY_LLUMNIX_MINUS], [5.0, 12.5], [2, 9]
    rows = ref.run_sweep(w, cfg, spec, pols, qps, seeds, jobs=4)
    assert len(rows) == 8
    i = 0
    for p in pols:
        for q in qps:
            for s in seeds:  # the reference's cell order: policy, qps, seed
                cw = w.copy()
                cw["qps"], cw["arrival_seed"], cw["estimator_seed"] = q, s, s
                sp = spec.copy()
                sp["policy"], sp["policy_seed"] = p, s
                rep = ref.run_report(cw, cfg, sp)
                r = rows[i]
                assert (int(r["policy"]), float(r["qps"]), int(r["seed"]), int(r["ok"])) == (p, q, s, 1)
                for f in ("mean_ttft_s", "p99_ttft_s", "mean_e2e_s", "p99_e2e_s", "throughput_rps",
                          "total_preemptions", "finished_requests", "free_blocks_var_avg"):
                    assert r[f] == rep[f], (i, f)
                i += 1


def test_reference_run_capacity_gains_format(ref):
    """ref_run_capacity (run_capacity, driver.cpp:392-427): the baseline is
    appended when absent, rows equal capacity_search per policy, and the gains
    are format_percent of (c - c_base) / c_base."""
    cfg = abi.make_config()
    w = abi.make_workload(count=120)
    spec = abi.make_replay_spec(3, capture=0)
    pols, base = [abi.POLICY_BLOCK_PREDICTIVE, abi.POLICY_ROUND_ROBIN], abi.POLICY_LLUMNIX_MINUS
    st, rows, bcap = ref.run_capacity(w, cfg, spec, pols, base, 2, 1, 10, 3.0)
    assert st == 0 and [int(p) for p in rows["policy"]] == pols + [base]
    for r in rows:
        sp = spec.copy()
        sp["policy"] = r["policy"]
        cst, exp, _ = ref.capacity_search(w, cfg, sp, 2, 1, 10, 3.0)
        assert cst == 0 and r["result"].tolist() == exp.tolist()
    assert bcap == float(rows["result"]["capacity_qps"][-1])
    for r in rows[:-1]:
        g = (float(r["result"]["capacity_qps"]) - bcap) / bcap
        assert r["gain_text"].decode() == "%.1f%%" % (g * 100.0)
    assert rows[-1]["has_gain"] == 0

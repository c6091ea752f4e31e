"""CPU tests of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/blocksim_b200.h declares, and its host-only parts (workload
generators) match the reference. No compute call touches a GPU here."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from paper_2508_03611_b200 import abi, native


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return native.load()


def test_exports_every_header_symbol(lib):
    names = native.exported_symbols_declared_in_header()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_kernels_are_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts(lib):
    assert abi.cfg_dtype.itemsize == 64 and abi.scenario_dtype.itemsize == 32
    assert abi.result_dtype.itemsize == 48 and abi.step_dtype.itemsize == 56
    assert lib.bsg_abi_version() == 1
    assert lib.bsg_ticks_to_seconds(61_200_000) == 61_200_000 * 1e-9


def test_no_cpu_fallback_without_device(lib):
    # In this container there is no GPU: creating a context must fail loudly.
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    h = C.c_void_p()
    assert lib.bsg_ctx_create(0, C.byref(h)) == abi.CUDA_ERROR
    with pytest.raises(native.BsgError):
        native.Context(0)
    with pytest.raises(native.BsgError):
        native.MultiContext([0, 0])


@pytest.mark.parametrize("kw", [
    dict(count=5000, estimator_kind=2, estimator_seed=1, qps=27, arrival_seed=1),
    dict(count=2000, prompt_median=600, output_median=600, qps=4.5, arrival_seed=3),
    dict(count=300, estimator_kind=1, fixed_tokens=100, qps=5, request_cap=100),
])
def test_workload_generators_match_reference(lib, ref, kw):
    # make_synthetic_trace / estimate_length / generate_arrivals (workload.cpp:113-191)
    w = abi.make_workload(**kw)
    a = native.make_workload_host(w)
    b = ref.make_workload(w)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_divisor_magic_matches_integer_division():
    # The kernel divides by block_size with a 32-bit magic multiplier (bsg_capi.cu:
    # to_dev); check the formula exhaustively on small n and randomly on large n.
    rng = np.random.default_rng(0)
    for bs in list(range(1, 70)) + [1000, 4095, 65537, (1 << 20) - 3]:
        if bs & (bs - 1) == 0:
            continue
        l = (bs - 1).bit_length()
        m = (1 << (31 + l)) // bs + 1
        assert m < (1 << 32)
        ns = np.concatenate([np.arange(0, 5000), rng.integers(0, 1 << 31, 20000)]).astype(np.uint64)
        q = ((ns * np.uint64(m)) >> np.uint64(32)) >> np.uint64(l - 1)
        assert np.array_equal(q, ns // np.uint64(bs)), bs


def test_mc_lengths_match_reference_estimator(lib, ref):
    """bsg_mc_lengths == the reference's estimate_length Noisy branch
    (workload.cpp:126-136) applied to the predicted length, sample s drawn from
    the stream of record id request_id * n_samples + s."""
    for est, rid in [(160, 0), (7, 12345), (4000, 2), (1, 99)]:
        got = native.mc_lengths(est, rid, 256, seed=1)
        exp = [ref.lib.ref_estimate_noisy(est, rid * 256 + s, 1, 0.244) for s in range(256)]
        assert got.tolist() == exp


@pytest.mark.parametrize("kw,n_inst", [
    (dict(count=800, qps=9, arrival_seed=5), 4),
    (dict(count=600, prompt_median=600, output_median=600, qps=6, arrival_seed=2), 3),
])
def test_aggregate_matches_reference(lib, ref, kw, n_inst):
    """bsg_aggregate (host) over the reference's own run outcomes equals the
    reference's aggregate() RunReport (metrics.cpp:21-124), double for double."""
    w = abi.make_workload(**kw)
    cfg = abi.make_config()
    spec = abi.make_replay_spec(n_inst, policy=abi.POLICY_LLUMNIX_MINUS)
    out, summ = ref.run_experiment(w, cfg, spec)
    got = native.aggregate(out, summ)
    exp = ref.run_report(w, cfg, spec)
    # the per-dispatch free-block balance needs the run's dispatch points, which
    # only the device metric pipeline (bsg_replay_device) has
    host_fields = [f for f in abi.report_dtype.names if not f.startswith("free_blocks")]
    assert [got[f] for f in host_fields] == [exp[f] for f in host_fields]
    assert got["free_blocks_mean_avg"] == 0 and exp["free_blocks_mean_avg"] > 0


def test_c_struct_layouts_match_numpy(tmp_path):
    """Every struct crossing the C-ABI has the same size and field offsets in
    C (gcc on include/blocksim_b200.h) and in paper_2508_03611_b200/abi.py."""
    pairs = [("bsg_instance_cfg", abi.cfg_dtype), ("bsg_scenario", abi.scenario_dtype),
             ("bsg_result", abi.result_dtype), ("bsg_step_record", abi.step_dtype),
             ("bsg_workload", abi.workload_dtype), ("bsg_replay_spec", abi.replay_spec_dtype),
             ("bsg_replay_summary", abi.summary_dtype), ("bsg_request_outcome", abi.outcome_dtype),
             ("bsg_run_report", abi.report_dtype), ("bsg_capacity_result", abi.capacity_dtype),
             ("bsg_sweep_cell", abi.sweep_cell_dtype), ("bsg_sweep_out", abi.sweep_out_dtype),
             ("bsg_closed_loop_run", abi.closed_loop_run_dtype), ("bsg_sweep_row", abi.sweep_row_dtype),
             ("bsg_capacity_row", abi.capacity_row_dtype)]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "blocksim_b200.h"',
             'int main(void) {']
    for cname, dt in pairs:
        lines.append(f'  printf("%zu\\n", sizeof({cname}));')
        for f in dt.names:
            lines.append(f'  printf("%zu\\n", offsetof({cname}, {f}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    inc = os.path.join(os.path.dirname(native.HEADER))
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(tmp_path / "layout")], check=True)
    got = [int(x) for x in subprocess.run([str(tmp_path / "layout")], capture_output=True,
                                          text=True, check=True).stdout.split()]
    exp = []
    for _, dt in pairs:
        exp.append(dt.itemsize)
        exp.extend(dt.fields[f][1] for f in dt.names)
    assert got == exp


def test_wire_number_text_matches_reference_json(lib, ref):
    """bsg_format_double prints doubles exactly as the reference's JSON layer
    (nlohmann::json::dump, Grisu2 — not always the shortest form), so wire
    responses are byte-identical: tick-derived latencies, random bit patterns,
    and the edge layouts (exponent notation, 15-digit integers, tiny values)."""
    import random
    import struct
    rng = random.Random(2026)
    vals = [199.2876835, 0.0612, 0.05848, 1.0, 0.1, 1e-9, 1e21, 1e-5, 2.5e-7, 1 / 3, 1e15, 1e16,
            123456789012345.0, 9007199254740993.0, 5e-324, 1.7976931348623157e308, 0.5, 2.0 ** -1022]
    vals += [rng.randrange(1, 10 ** 13) * 1e-9 for _ in range(4000)]
    vals += [struct.unpack("<d", struct.pack("<Q", rng.getrandbits(63)))[0] for _ in range(4000)]
    vals += [rng.lognormvariate(0, 25) for _ in range(2000)]
    for v in vals:
        if v != v or v == float("inf"):
            continue
        assert native.format_double(v) == ref.dump_double(v), repr(v)
        assert float(native.format_double(v)) == v  # round trip


def _mutations(base):
    """Request bodies that fail before simulation, one defect each."""
    import copy
    import json
    out = ["{not json", "", "[]", "3", "null", json.dumps({"snapshot": 1})]
    paths = [("snapshot",), ("candidate",), ("instance_config",), ("snapshot", "running"),
             ("snapshot", "qpm"), ("snapshot", "snapshot_time"), ("candidate", "prompt_tokens"),
             ("instance_config", "cost_model"), ("instance_config", "cost_model", "c0_s"),
             ("instance_config", "local_policy"), ("instance_config", "total_blocks")]
    for path in paths:
        for val in (None, "x", True, [1], {"a": 1}, 1.5, -3, "DELETE"):
            d = copy.deepcopy(base)
            o = d
            for k in path[:-1]:
                o = o[k]
            if val == "DELETE":
                del o[path[-1]]
            else:
                o[path[-1]] = val
            out.append(json.dumps(d))
    for field, val in [("total_blocks", 0), ("block_size", 0), ("max_batch_size", 0), ("chunk_budget", 1),
                       ("local_policy", "round_robin")]:
        d = copy.deepcopy(base)
        d["instance_config"][field] = val
        out.append(json.dumps(d))
    for field, val in [("c0_s", 0.0), ("prefill_s_per_token", -1.0), ("decode_s_per_seq", -1e-9),
                       ("context_s_per_token", -2.0)]:
        d = copy.deepcopy(base)
        d["instance_config"]["cost_model"][field] = val
        out.append(json.dumps(d))
    # running given as an object / a string / null: nlohmann's range-for semantics
    entry = base["snapshot"]["running"][0] if base["snapshot"]["running"] else None
    for val in ({"b": entry, "a": entry}, "str", None, [entry, 5]):
        d = copy.deepcopy(base)
        d["snapshot"]["running"] = val
        out.append(json.dumps(d))
    return out


def test_wire_check_error_bodies_match_reference(lib, ref):
    """/predict requests rejected before simulation (schema, types, config
    validation): bsg_wire_check answers the reference role's status class and
    the byte-identical error body (nlohmann's exception text; ConfigError's
    "invalid config: <field>: <rule>"); accepted bodies are accepted by both."""
    import json
    from paper_2508_03611_b200 import native
    from scenarios import kat_set
    names, kc, ks = kat_set()
    base = json.loads(ref.request_json(kc, ks, 1))
    assert base["snapshot"]["running"], "need a running entry to mutate"
    n_err = 0
    for body in _mutations(base):
        code, exp = ref.service_predict(body)
        st, got = native.wire_check(body)
        if code == 400:
            assert st != 0 and got == exp, (body, got, exp)
            n_err += 1
        else:  # simulated by the reference (200 / 422): simulated here too
            assert st == 0, (body, code, exp, got)
    assert n_err > 60


def test_sweep_driver_argument_checks_without_device(lib):
    """run_sweep / run_capacity reject bad policies and arguments before any
    device work (a host check, so it holds on this GPU-less container too)."""
    cfg, w, spec = abi.make_config(), abi.make_workload(count=10), abi.make_replay_spec(2, capture=0)
    with pytest.raises(native.BsgError) as e:
        native.run_sweep(0, w, cfg, spec, [9], [1.0], [1])
    assert e.value.status == abi.BAD_CONFIG
    with pytest.raises(native.BsgError) as e:
        native.run_capacity(0, w, cfg, spec, [abi.POLICY_BLOCK_PREDICTIVE], 7, 1, 1, 2, 3.0)
    assert e.value.status == abi.BAD_CONFIG
    rows = np.zeros(1, abi.sweep_row_dtype)
    assert lib.bsg_run_sweep(0, abi.ptr(w), abi.ptr(cfg), abi.ptr(spec), None, 1, None, 0, None, 0, 1,
                             abi.ptr(rows)) == abi.INVALID_ARGUMENT

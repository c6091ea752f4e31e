"""ctypes binding of the product C-ABI (include/blocksim_b200.h).

Loads paper_2508_03611_b200/_lib/libblocksim_b200.so (built in-tree by
__graft_entry__.build() / `make -C paper_2508_03611_b200/csrc`). There is no
fallback: a missing library or a missing CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi

LIB_PATH = os.environ.get("BSG_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libblocksim_b200.so")
HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "blocksim_b200.h")

_lib = None


class BsgError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {abi.STATUS_NAMES.get(status, status)} {detail}".strip())


def load() -> C.CDLL:
    """Loads the native library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    V, E = C.c_void_p, C.POINTER(abi.Entries)
    sigs = {
        "bsg_abi_version": (C.c_int, []),
        "bsg_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
        "bsg_ctx_destroy": (None, [V]),
        "bsg_last_error": (C.c_char_p, [V]),
        "bsg_launch_count": (C.c_int64, [V]),
        "bsg_set_configs": (C.c_int, [V, V, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "bsg_predict_batch": (C.c_int, [V, E, C.c_int64, V, C.c_int64, V]),
        "bsg_predict_batch_device": (C.c_int, [V, E, V, C.c_int64, C.c_int32, V, V]),
        "bsg_trace": (C.c_int, [V, E, C.c_int64, V, V, C.c_int64, C.POINTER(C.c_int64), V]),
        "bsg_dispatch": (C.c_int, [V, E, C.c_int64, V, V, C.c_int32, C.c_int32, C.c_int32, V, V]),
        "bsg_replay": (C.c_int, [V, V, V, V, V, V, C.POINTER(C.c_void_p)]),
        "bsg_capture_sizes": (None, [V, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "bsg_capture_copy": (None, [V] * 7),
        "bsg_capture_free": (None, [V]),
        "bsg_make_workload": (C.c_int, [V, V, V, V, V]),
        "bsg_ticks_to_seconds": (C.c_double, [C.c_int64]),
        "bsg_dispatch_mc": (C.c_int, [V, E, C.c_int64, V, V, C.c_int32, C.c_int32, V, C.c_int32,
                                      C.c_int32, V, V, V, V]),
        "bsg_aggregate": (C.c_int, [V, C.c_int64, V, V]),
        "bsg_capacity_search": (C.c_int, [V, V, V, V, C.c_uint64, C.c_int32, C.c_int32, C.c_double,
                                          V, V, V, C.c_int32]),
        "bsg_sweep_run": (C.c_int, [C.c_int, V, C.c_int32, C.c_int32, V]),
        "bsg_run_sweep": (C.c_int, [C.c_int, V, V, V, V, C.c_int32, V, C.c_int32, V, C.c_int32,
                                    C.c_int32, V]),
        "bsg_run_capacity": (C.c_int, [C.c_int, V, V, V, V, C.c_int32, C.c_int32, C.c_uint64,
                                       C.c_int32, C.c_int32, C.c_double, C.c_int32, V,
                                       C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
        "bsg_scenario_count": (C.c_int64, [V]),
        "bsg_mc_lengths": (C.c_int, [C.c_int32, C.c_uint64, C.c_int32, C.c_uint64, C.c_double, V]),
        "bsg_replay_device": (C.c_int, [V, V, C.c_int32, V, V, V, V, C.c_int64, V, V, V, V]),
        "bsg_fleet_create": (C.c_int, [V, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
        "bsg_fleet_destroy": (None, [V]),
        "bsg_fleet_dispatch": (C.c_int, [V, C.c_int64, C.c_int32, C.c_int32, C.c_int32, V, C.c_int32,
                                         C.c_int32, V, V]),
        "bsg_fleet_finish": (C.c_int, [V, V, V, V]),
        "bsg_predict_json": (C.c_int, [V, V, C.c_int32, V, C.c_int64, V, V]),
        "bsg_format_double": (C.c_int32, [C.c_double, C.c_char_p, C.c_int32]),
        "bsg_load_trace": (C.c_int, [C.c_char_p, C.c_int64, V, C.c_int64, C.POINTER(C.c_int64),
                                     C.POINTER(abi.TraceError)]),
        "bsg_make_trace": (C.c_int, [V, V]),
        "bsg_write_trace": (C.c_int, [V, C.c_int64, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]),
        "bsg_trace_workload": (C.c_int, [V, C.c_int64, V, V, V, V, V, C.POINTER(C.c_int64),
                                         C.POINTER(abi.TraceError)]),
        "bsg_replay_trace": (C.c_int, [V, V, C.c_int64, V, V, V, V, V, C.POINTER(abi.TraceError)]),
        "bsg_fleet_snapshot": (C.c_int, [V, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                         V, V, V, V, C.c_int32]),
        "bsg_dispatch_mc_sampled": (C.c_int, [V, E, C.c_int64, V, V, C.c_int32, C.c_int32, V,
                                              C.c_int32, C.c_uint64, C.c_double, C.c_int32, V, V, V,
                                              V, V]),
        "bsg_last_launch": (C.c_char_p, [V]),
        "bsg_fleet_dispatch_sampled": (C.c_int, [V, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                                 C.c_uint64, C.c_int32, C.c_uint64, C.c_double,
                                                 C.c_int32, V, V]),
        "bsg_wire_check": (C.c_int32, [C.c_char_p, C.c_char_p, C.c_int64]),
        "bsg_multi_create": (C.c_int, [V, C.c_int32, C.POINTER(C.c_void_p)]),
        "bsg_multi_destroy": (None, [V]),
        "bsg_multi_device_count": (C.c_int32, [V]),
        "bsg_multi_last_error": (C.c_char_p, [V]),
        "bsg_multi_launch_count": (C.c_int64, [V]),
        "bsg_multi_set_configs": (C.c_int, [V, V, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "bsg_multi_predict_batch": (C.c_int, [V, E, C.c_int64, V, C.c_int64, C.c_int32, V]),
        "bsg_multi_dispatch": (C.c_int, [V, E, C.c_int64, V, V, C.c_int32, C.c_int32, C.c_int32, V, V]),
        "bsg_multi_dispatch_mc_sampled": (C.c_int, [V, E, C.c_int64, V, V, C.c_int32, C.c_uint64,
                                                    C.c_int32, C.c_uint64, C.c_double, C.c_int32, V, V]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    if L.bsg_abi_version() != 1:
        raise RuntimeError("ABI version mismatch")
    _lib = L
    return L


def exported_symbols_declared_in_header() -> list[str]:
    """Function names declared in include/blocksim_b200.h (for the export check)."""
    import re
    txt = open(HEADER).read()
    decl = re.compile(r"^\s*(?:bsg_status|void|int|int32_t|int64_t|double|const char\*)\s+(bsg_[a-z_0-9]+)\s*\(",
                      re.M)
    return sorted(set(decl.findall(txt)))


def _p(a):
    return abi.ptr(a)


def aggregate(outcomes: np.ndarray, summary=None) -> np.void:
    """RunReport subset of a replay's outcomes (bsg_aggregate, metrics.cpp:21-124)."""
    out = np.zeros(1, abi.report_dtype)
    summ = None if summary is None else np.array([summary], abi.summary_dtype)
    outcomes = np.ascontiguousarray(outcomes, abi.outcome_dtype)
    st = load().bsg_aggregate(_p(outcomes), len(outcomes), _p(summ), _p(out))
    if st != abi.OK:
        raise BsgError(st, "bsg_aggregate")
    return out[0]


def sweep_run(device: int, cells: np.ndarray, threads: int = 8) -> np.ndarray:
    """bsg_sweep_run: capacity searches for many cells, concurrent on one GPU."""
    cells = np.ascontiguousarray(cells, abi.sweep_cell_dtype)
    out = np.zeros(len(cells), abi.sweep_out_dtype)
    st = load().bsg_sweep_run(device, _p(cells), len(cells), threads, _p(out))
    if st != abi.OK:
        raise BsgError(st, "bsg_sweep_run")
    return out


def run_sweep(device: int, w, cfg, spec, policies, qps_values, seeds, threads: int = 8) -> np.ndarray:
    """bsg_run_sweep (run_sweep, driver.cpp:333-390): one SweepCell row per
    (policy, qps, seed), policies outermost."""
    pol = np.ascontiguousarray(policies, np.int32)
    qps = np.ascontiguousarray(qps_values, np.float64)
    sd = np.ascontiguousarray(seeds, np.uint64)
    rows = np.zeros(len(pol) * len(qps) * len(sd), abi.sweep_row_dtype)
    st = load().bsg_run_sweep(device, _p(w), _p(cfg), _p(spec), _p(pol), len(pol), _p(qps), len(qps),
                              _p(sd), len(sd), threads, _p(rows))
    if st != abi.OK:
        raise BsgError(st, "bsg_run_sweep")
    return rows


def run_capacity(device: int, w, cfg, spec, policies, baseline: int, seed: int, qps_min: int,
                 qps_max: int, slo: float, threads: int = 8):
    """bsg_run_capacity (run_capacity, driver.cpp:392-427): (rows, baseline capacity)."""
    pol = np.ascontiguousarray(policies, np.int32)
    rows = np.zeros(len(pol) + 1, abi.capacity_row_dtype)
    n = C.c_int32(0)
    bc = C.c_double(0)
    st = load().bsg_run_capacity(device, _p(w), _p(cfg), _p(spec), _p(pol), len(pol), baseline, seed,
                                 qps_min, qps_max, slo, threads, _p(rows), C.byref(n), C.byref(bc))
    if st != abi.OK:
        raise BsgError(st, "bsg_run_capacity")
    return rows[:n.value], bc.value


def mc_lengths(est: int, request_id: int, n_samples: int = 256, seed: int = 1,
               mean_abs_rel_error: float = 0.244) -> np.ndarray:
    """Sampled response lengths for one request (bsg_mc_lengths)."""
    out = np.zeros(n_samples, np.int32)
    st = load().bsg_mc_lengths(int(est), int(request_id), n_samples, seed, mean_abs_rel_error,
                               _p(out))
    if st != abi.OK:
        raise BsgError(st, "bsg_mc_lengths")
    return out


def wire_check(body: str) -> tuple[int, str]:
    """bsg_wire_check: (status, the reference role's error body or "")."""
    buf = C.create_string_buffer(1 << 16)
    st = load().bsg_wire_check(body.encode(), buf, len(buf))
    return int(st), buf.value.decode()


def format_double(v: float) -> str:
    """A double as the reference's JSON layer prints it (bsg_format_double)."""
    buf = C.create_string_buffer(64)
    n = load().bsg_format_double(float(v), buf, 64)
    assert n >= 0
    return buf.value.decode()


def make_workload_host(w: np.ndarray):
    """Synthetic trace + estimates + arrival ticks (host C++, no GPU needed)."""
    L = load()
    n = int(w["count"][0]) if w["request_cap"][0] < 0 else min(int(w["count"][0]),
                                                                int(w["request_cap"][0]))
    p, o, e = (np.zeros(n, np.int32) for _ in range(3))
    t = np.zeros(n, np.int64)
    st = L.bsg_make_workload(_p(w), _p(p), _p(o), _p(e), _p(t))
    if st != abi.OK:
        raise BsgError(st, "bsg_make_workload")
    return p, o, e, t


class TraceError(ValueError):
    """load_trace / generate_arrivals rejection: kind 1 TraceParseError (line),
    2 InvalidRecordError (field), 3 ConfigError (field)."""

    def __init__(self, e: abi.TraceError):
        self.kind, self.line = int(e.kind), int(e.line)
        self.field = e.field.decode()
        super().__init__(e.message.decode())


def load_trace(text: str | bytes) -> np.ndarray:
    """load_trace (workload.cpp:51-68) over a JSON Lines text -> trace_record_dtype
    rows; raises TraceError on the first bad line. No GPU needed."""
    L = load()
    b = text.encode() if isinstance(text, str) else bytes(text)
    err, n = abi.TraceError(), C.c_int64(0)
    cap = b.count(b"\n") + 1
    out = np.zeros(cap, abi.trace_record_dtype)
    st = L.bsg_load_trace(b, len(b), _p(out), cap, C.byref(n), C.byref(err))
    if st == abi.BAD_INPUT:
        raise TraceError(err)
    if st != abi.OK:
        raise BsgError(st, "bsg_load_trace")
    return out[:n.value].copy()


def make_trace(w: np.ndarray) -> np.ndarray:
    """make_synthetic_trace (workload.cpp:172-191) as trace records."""
    L = load()
    out = np.zeros(max(int(w["count"][0]), 1), abi.trace_record_dtype)
    st = L.bsg_make_trace(_p(w), _p(out))
    if st != abi.OK:
        raise BsgError(st, "bsg_make_trace")
    return out[:int(w["count"][0])]


def write_trace(recs: np.ndarray) -> bytes:
    """write_trace (workload.cpp:78-89): JSON Lines, byte-identical to the reference."""
    L = load()
    recs = np.ascontiguousarray(recs, dtype=abi.trace_record_dtype)
    need = C.c_int64(0)
    L.bsg_write_trace(_p(recs), len(recs), None, 0, C.byref(need))
    buf = C.create_string_buffer(max(need.value, 1))
    st = L.bsg_write_trace(_p(recs), len(recs), buf, len(buf), C.byref(need))
    if st != abi.OK:
        raise BsgError(st, "bsg_write_trace")
    return buf.raw[:need.value]


def load_trace_file(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        return load_trace(f.read())


def trace_workload(recs: np.ndarray, w: np.ndarray):
    """Request columns (prompt, output, est, arrival_ticks) run_experiment
    builds from trace records: request_cap, generate_arrivals, estimate_length."""
    L = load()
    recs = np.ascontiguousarray(recs, dtype=abi.trace_record_dtype)
    n = len(recs)
    p, o, e = (np.zeros(max(n, 1), np.int32) for _ in range(3))
    t = np.zeros(max(n, 1), np.int64)
    err, m = abi.TraceError(), C.c_int64(0)
    st = L.bsg_trace_workload(_p(recs), n, _p(w), _p(p), _p(o), _p(e), _p(t), C.byref(m), C.byref(err))
    if st == abi.BAD_INPUT:
        raise TraceError(err)
    if st != abi.OK:
        raise BsgError(st, "bsg_trace_workload")
    k = m.value
    return p[:k], o[:k], e[:k], t[:k]


class Fleet:
    """A device-resident mirror of live instances (bsg_fleet_*): one launch per
    dispatch, the snapshots never leave HBM."""

    def __init__(self, ctx: "Context", n_instances: int, max_requests: int, cfg: int = 0):
        self.ctx, self.n = ctx, n_instances
        h = C.c_void_p()
        ctx._check(ctx.L.bsg_fleet_create(ctx.h, cfg, n_instances, max_requests, C.byref(h)),
                   "bsg_fleet_create")
        self.h = h
        self._chosen = C.c_int32(-1)

    def dispatch(self, now_ticks: int, prompt: int, est: int, output: int, lengths=None,
                 objective: int = 0, scores: np.ndarray | None = None) -> int:
        lp, ns = (None, 0) if lengths is None else (_p(lengths), len(lengths))
        st = self.ctx.L.bsg_fleet_dispatch(self.h, int(now_ticks), int(prompt), int(est), int(output),
                                           lp, ns, objective, C.byref(self._chosen),
                                           None if scores is None else _p(scores))
        self.ctx._check(st, "bsg_fleet_dispatch")
        return self._chosen.value

    def dispatch_sampled(self, now_ticks: int, prompt: int, est: int, output: int, request_id: int,
                         n_samples: int = 256, seed: int = 1, mean_abs_rel_error: float = 0.244,
                         objective: int = 0, scores: np.ndarray | None = None) -> int:
        """Monte-Carlo dispatch with the samples drawn on the device (K3)."""
        st = self.ctx.L.bsg_fleet_dispatch_sampled(self.h, int(now_ticks), int(prompt), int(est),
                                                   int(output), int(request_id), n_samples, seed,
                                                   mean_abs_rel_error, objective, C.byref(self._chosen),
                                                   None if scores is None else _p(scores))
        self.ctx._check(st, "bsg_fleet_dispatch_sampled")
        return self._chosen.value

    def snapshot(self, instance: int):
        """(running, waiting) columns (prompt, est, prefill, decoded) of one instance."""
        rn, wn = C.c_int32(0), C.c_int32(0)
        L = self.ctx.L
        self.ctx._check(L.bsg_fleet_snapshot(self.h, instance, C.byref(rn), C.byref(wn), None, None,
                                             None, None, 0), "bsg_fleet_snapshot")
        n = rn.value + wn.value
        cols = [np.zeros(max(n, 1), np.int32) for _ in range(4)]
        self.ctx._check(L.bsg_fleet_snapshot(self.h, instance, C.byref(rn), C.byref(wn),
                                             *[_p(c) for c in cols], max(n, 1)), "bsg_fleet_snapshot")
        return rn.value, wn.value, [c[:n] for c in cols]

    def finish(self, max_requests: int):
        out = np.zeros(max_requests, abi.outcome_dtype)
        n = C.c_int32(0)
        summ = np.zeros(1, abi.summary_dtype)
        self.ctx._check(self.ctx.L.bsg_fleet_finish(self.h, _p(out), C.byref(n), _p(summ)),
                        "bsg_fleet_finish")
        return out[:n.value], summ[0]

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.bsg_fleet_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiContext:
    """Several GPUs in one process (bsg_multi_*): one context + host worker
    thread per device; batches split by arrival group, dispatches by request,
    one Monte-Carlo dispatch by instance (exact host argmin merge)."""

    def __init__(self, devices):
        self.L = load()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        st = self.L.bsg_multi_create(devs, len(devices), C.byref(h))
        if st != abi.OK:
            raise BsgError(st, "bsg_multi_create", "(CUDA devices are required)")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.bsg_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, where):
        if st != abi.OK:
            raise BsgError(st, where, self.L.bsg_multi_last_error(self.h).decode())

    @property
    def launches(self) -> int:
        return int(self.L.bsg_multi_launch_count(self.h))

    def set_configs(self, cfgs: np.ndarray):
        cfgs = np.ascontiguousarray(cfgs, dtype=abi.cfg_dtype)
        bi, fc = C.c_int32(-1), C.c_int32(0)
        self._check(self.L.bsg_multi_set_configs(self.h, _p(cfgs), len(cfgs), C.byref(bi), C.byref(fc)),
                    "bsg_multi_set_configs")

    def predict_batch(self, ss: abi.ScenarioSet, group: int = 1) -> np.ndarray:
        out = np.zeros(len(ss), abi.result_dtype)
        e = ss.entries()
        self._check(self.L.bsg_multi_predict_batch(self.h, C.byref(e), ss.n_entries, _p(ss.scenarios),
                                                   len(ss), group, _p(out)), "bsg_multi_predict_batch")
        return out

    def dispatch(self, ss: abi.ScenarioSet, instance_ids: np.ndarray, n_inst: int, objective: int = 0):
        n_req = len(ss) // n_inst
        ids = np.ascontiguousarray(instance_ids, dtype=np.int32)
        chosen = np.zeros(n_req, np.int32)
        per = np.zeros(len(ss), abi.result_dtype)
        e = ss.entries()
        self._check(self.L.bsg_multi_dispatch(self.h, C.byref(e), ss.n_entries, _p(ss.scenarios), _p(ids),
                                              n_inst, n_req, objective, _p(chosen), _p(per)),
                    "bsg_multi_dispatch")
        return chosen, per

    def dispatch_mc_sampled(self, ss: abi.ScenarioSet, instance_ids: np.ndarray, request_id: int,
                            n_samples: int = 256, seed: int = 1, mean_abs_rel_error: float = 0.244,
                            objective: int = 0):
        ids = np.ascontiguousarray(instance_ids, dtype=np.int32)
        chosen = C.c_int32(-1)
        scores = np.zeros(len(ss), np.int64)
        e = ss.entries()
        self._check(self.L.bsg_multi_dispatch_mc_sampled(
            self.h, C.byref(e), ss.n_entries, _p(ss.scenarios), _p(ids), len(ss), int(request_id),
            n_samples, seed, mean_abs_rel_error, objective, C.byref(chosen), _p(scores)),
            "bsg_multi_dispatch_mc_sampled")
        return chosen.value, scores


class Context:
    """One CUDA device + stream + device buffers (bsg_ctx)."""

    def __init__(self, device: int = 0):
        self.L = load()
        h = C.c_void_p()
        st = self.L.bsg_ctx_create(device, C.byref(h))
        if st != abi.OK:
            raise BsgError(st, "bsg_ctx_create", "(a CUDA device is required)")
        self.h = h
        self.cfgs = None

    def close(self):
        if getattr(self, "h", None):
            self.L.bsg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, where):
        if st != abi.OK:
            raise BsgError(st, where, self.L.bsg_last_error(self.h).decode())

    @property
    def launches(self) -> int:
        return int(self.L.bsg_launch_count(self.h))

    def set_configs(self, cfgs: np.ndarray):
        cfgs = np.ascontiguousarray(cfgs, dtype=abi.cfg_dtype)
        bi, fc = C.c_int32(-1), C.c_int32(0)
        st = self.L.bsg_set_configs(self.h, _p(cfgs), len(cfgs), C.byref(bi), C.byref(fc))
        if st != abi.OK:
            raise BsgError(st, "bsg_set_configs", f"config {bi.value} field {fc.value}")
        self.cfgs = cfgs

    def predict_batch(self, ss: abi.ScenarioSet, out: np.ndarray | None = None) -> np.ndarray:
        """out: optional result array to fill (e.g. a view of pinned host memory:
        32-member chunks then store their results straight into it)."""
        if out is None:
            out = np.zeros(len(ss), abi.result_dtype)
        assert out.dtype == abi.result_dtype and len(out) >= len(ss) and out.flags.c_contiguous
        e = ss.entries()
        self._check(self.L.bsg_predict_batch(self.h, C.byref(e), ss.n_entries, _p(ss.scenarios),
                                             len(ss), _p(out)), "bsg_predict_batch")
        return out

    def predict_batch_device(self, dev_cols, dev_scen_ptr: int, n: int, dev_out_ptr: int,
                             stream_ptr: int | None = None, member_capacity: int = 0):
        """dev_cols: (prompt, est, prefill, decoded) device pointers (ints).
        stream_ptr: a cudaStream_t (not the legacy default stream 0)."""
        e = abi.Entries(None, *[C.c_void_p(x) for x in dev_cols])
        self._check(self.L.bsg_predict_batch_device(self.h, C.byref(e), C.c_void_p(dev_scen_ptr), n,
                                                    member_capacity, C.c_void_p(dev_out_ptr),
                                                    C.c_void_p(stream_ptr) if stream_ptr else None),
                    "bsg_predict_batch_device")

    def trace(self, ss: abi.ScenarioSet, i: int = 0, cap: int = 1 << 20):
        rec = np.zeros(cap, abi.step_dtype)
        out = np.zeros(1, abi.result_dtype)
        n = C.c_int64(0)
        e = ss.entries()
        sc = np.ascontiguousarray(ss.scenarios[i:i + 1])
        self._check(self.L.bsg_trace(self.h, C.byref(e), ss.n_entries, _p(sc), _p(rec), cap,
                                     C.byref(n), _p(out)), "bsg_trace")
        return out[0], rec[:min(n.value, cap)]

    def dispatch(self, ss: abi.ScenarioSet, instance_ids: np.ndarray, n_inst: int,
                 objective: int = 0):
        n_req = len(ss) // n_inst
        ids = np.ascontiguousarray(instance_ids, dtype=np.int32)
        chosen = np.zeros(n_req, np.int32)
        per = np.zeros(len(ss), abi.result_dtype)
        e = ss.entries()
        self._check(self.L.bsg_dispatch(self.h, C.byref(e), ss.n_entries, _p(ss.scenarios), _p(ids),
                                        n_inst, n_req, objective, _p(chosen), _p(per)),
                    "bsg_dispatch")
        return chosen, per

    def dispatch_mc(self, ss: abi.ScenarioSet, instance_ids: np.ndarray, n_inst: int,
                    lengths: np.ndarray, objective: int = 0, want_samples: bool = False,
                    want_results: bool = False):
        """Monte-Carlo BlockPredictive dispatch (bsg_dispatch_mc). lengths: [n_req, S]."""
        n_req = len(ss) // n_inst
        lengths = np.ascontiguousarray(lengths, dtype=np.int32).reshape(n_req, -1)
        S = lengths.shape[1]
        ids = np.ascontiguousarray(instance_ids, dtype=np.int32)
        chosen = np.zeros(n_req, np.int32)
        scores = np.zeros(len(ss), np.int64)
        samples = np.zeros((len(ss), S), np.int64) if want_samples else None
        per = np.zeros(len(ss), abi.result_dtype) if want_results else None
        e = ss.entries()
        self._check(self.L.bsg_dispatch_mc(self.h, C.byref(e), ss.n_entries, _p(ss.scenarios),
                                           _p(ids), n_inst, n_req, _p(lengths), S, objective,
                                           _p(chosen), _p(scores), _p(samples), _p(per)),
                    "bsg_dispatch_mc")
        return chosen, scores, samples, per

    def dispatch_mc_sampled(self, ss: abi.ScenarioSet, instance_ids: np.ndarray, n_inst: int,
                            request_ids, n_samples: int = 256, seed: int = 1,
                            mean_abs_rel_error: float = 0.244, objective: int = 0,
                            want_lengths: bool = False, dev_keys_ptr: int | None = None):
        """bsg_dispatch_mc_sampled: Monte-Carlo dispatch with the length samples
        drawn on the device (K3). Returns (chosen, scores, lengths or None)."""
        n_req = len(ss) // n_inst
        ids = np.ascontiguousarray(instance_ids, dtype=np.int32)
        rid = np.ascontiguousarray(request_ids, dtype=np.uint64).reshape(n_req)
        chosen = np.zeros(n_req, np.int32)
        scores = np.zeros(len(ss), np.int64)
        lens = np.zeros((n_req, n_samples), np.int32) if want_lengths else None
        e = ss.entries()
        self._check(self.L.bsg_dispatch_mc_sampled(
            self.h, C.byref(e), ss.n_entries, _p(ss.scenarios), _p(ids), n_inst, n_req, _p(rid),
            n_samples, seed, mean_abs_rel_error, objective, _p(chosen), _p(scores), _p(lens), None,
            C.c_void_p(dev_keys_ptr) if dev_keys_ptr else None), "bsg_dispatch_mc_sampled")
        return chosen, scores, lens

    @property
    def last_launch(self) -> str:
        return self.L.bsg_last_launch(self.h).decode()

    def capacity_search(self, w, cfg, spec, seed: int, qps_min: int, qps_max: int, slo: float):
        """capacity_search over GPU closed loops. Returns (status, result, [(qps, passed)])."""
        out = np.zeros(1, abi.capacity_dtype)
        tq = np.zeros(256, np.float64)
        tp = np.zeros(256, np.int32)
        st = self.L.bsg_capacity_search(self.h, _p(w), _p(cfg), _p(spec), seed, qps_min, qps_max,
                                        slo, _p(out), _p(tq), _p(tp), 256)
        if st not in (abi.OK, abi.NO_CAPACITY):
            self._check(st, "bsg_capacity_search")
        n = int(out["n_tested"][0])
        return st, out[0], list(zip(tq[:n].tolist(), tp[:n].astype(bool).tolist()))

    def predict_json(self, bodies: list[str]):
        """Wire-format predict (bsg_predict_json): [(status, response text)]."""
        n = len(bodies)
        arr = (C.c_char_p * max(n, 1))(*[b.encode() for b in bodies])
        off = np.zeros(n + 1, np.int64)
        st = np.zeros(max(n, 1), np.int32)
        cap = 256 * n + 64
        for _ in range(2):
            buf = C.create_string_buffer(cap)
            r = self.L.bsg_predict_json(self.h, arr, n, buf, cap, _p(off), _p(st))
            if r == abi.OK:
                raw = buf.raw
                return [(int(st[i]), raw[off[i]:off[i + 1] - 1].decode()) for i in range(n)]
            if r != abi.INVALID_ARGUMENT or off[n] <= cap:
                self._check(r, "bsg_predict_json")
            cap = int(off[n])
        self._check(r, "bsg_predict_json")

    def replay_device(self, runs):
        """Device-resident closed loops (bsg_replay_device). runs: list of
        (workload, replay_spec, cfg_index) with the configs already set (any
        policy, provisioning and dispatch overhead); a workload may also be the
        (prompt, output, est, arrival_ticks) columns, e.g. of trace_workload.
        Returns [(status, outcomes, summary)] per run."""
        cols = [w if isinstance(w, tuple) else make_workload_host(w) for w, *_ in runs]
        desc = np.zeros(len(runs), abi.closed_loop_run_dtype)
        off = 0
        for r, ((w, sp, cf), c) in enumerate(zip(runs, cols)):
            sp = np.asarray(sp).reshape(-1)[0]
            desc[r] = (sp["n_instances"], sp["objective"], cf, len(c[0]), off, sp["provision_kind"],
                       sp["max_instances"], sp["threshold_s"], sp["cold_start_s"], sp["cooldown_s"],
                       sp["policy"], 0, sp["policy_seed"], sp["dispatch_overhead_s"])
            off += len(c[0])
        p, o, e, t = (np.ascontiguousarray(np.concatenate([c[j] for c in cols])) for j in range(4))
        out = np.zeros(off, abi.outcome_dtype)
        summ = np.zeros(len(runs), abi.summary_dtype)
        st = np.zeros(len(runs), np.int32)
        rep = np.zeros(len(runs), abi.report_dtype)
        self._check(self.L.bsg_replay_device(self.h, _p(desc), len(runs), _p(p), _p(o), _p(e), _p(t),
                                             off, _p(out), _p(summ), _p(st), _p(rep)),
                    "bsg_replay_device")
        self.last_reports = rep
        res = []
        for r in range(len(runs)):
            a, n = int(desc[r]["req_off"]), int(desc[r]["n_requests"])
            res.append((int(st[r]), out[a:a + n], summ[r]))
        return res

    def replay_trace(self, recs, w, cfg, spec):
        """Closed-loop replay over trace records (bsg_replay_trace). Returns
        (outcomes, summary)."""
        recs = np.ascontiguousarray(recs, dtype=abi.trace_record_dtype)
        n = len(recs) if w["request_cap"][0] < 0 else min(len(recs), int(w["request_cap"][0]))
        out = np.zeros(max(n, 1), abi.outcome_dtype)
        summ = np.zeros(1, abi.summary_dtype)
        err = abi.TraceError()
        st = self.L.bsg_replay_trace(self.h, _p(recs), len(recs), _p(w), _p(cfg), _p(spec), _p(out),
                                     _p(summ), C.byref(err))
        if st == abi.BAD_INPUT and err.kind:
            raise TraceError(err)
        self._check(st, "bsg_replay_trace")
        return out[:n], summ[0]

    def replay(self, w, cfg, spec):
        """Closed-loop replay (host live instances, GPU what-ifs). Returns
        (outcomes, summary, captured ScenarioSet or None)."""
        n = int(w["count"][0]) if w["request_cap"][0] < 0 else min(int(w["count"][0]),
                                                                    int(w["request_cap"][0]))
        out = np.zeros(n, abi.outcome_dtype)
        summ = np.zeros(1, abi.summary_dtype)
        h = C.c_void_p(None)
        capture = bool(spec["capture"][0])
        self._check(self.L.bsg_replay(self.h, _p(w), _p(cfg), _p(spec), _p(out), _p(summ),
                                      C.byref(h) if capture else None), "bsg_replay")
        ss = None
        if capture:
            ne, ns = C.c_int64(0), C.c_int64(0)
            self.L.bsg_capture_sizes(h, C.byref(ne), C.byref(ns))
            ids = np.zeros(ne.value, np.uint64)
            cols = [np.zeros(ne.value, np.int32) for _ in range(4)]
            sc = np.zeros(ns.value, abi.scenario_dtype)
            self.L.bsg_capture_copy(h, _p(ids), *[_p(c) for c in cols], _p(sc))
            self.L.bsg_capture_free(h)
            ss = abi.ScenarioSet(*cols, sc, ids=ids)
        return out, summ[0], ss

"""ctypes loaders for the two CPU checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) import this module. The product package never does.

  CRestatement  -> oracle/build/liboracle.so       (oracle/blocksim_oracle.c)
  Reference     -> oracle/_ref/libblocksim_ref.so  (the reference compiled from
                   /root/reference by oracle/Makefile + oracle/ref_shim.cpp)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2508_03611_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(HERE, "build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libblocksim_ref.so")
REF_SRC = "/root/reference/proj/core"


def build(ref: bool | None = None) -> None:
    """Compile the C restatement, and the reference shim when its sources exist."""
    targets = ["c"]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, f"-j{os.cpu_count() or 4}", *targets], check=True)


def _vp(a):
    return abi.ptr(a)


class CRestatement:
    def __init__(self, path: str = C_LIB):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = C.CDLL(path)
        L = self.lib
        L.oracle_predict.restype = C.c_int32
        L.oracle_predict.argtypes = [C.c_void_p, C.POINTER(abi.Entries), C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.oracle_predict_batch.restype = None
        L.oracle_predict_batch.argtypes = [C.c_void_p, C.POINTER(abi.Entries), C.c_void_p,
                                           C.c_int64, C.c_void_p]
        L.oracle_blocks_needed.restype = C.c_int64
        L.oracle_blocks_needed.argtypes = [C.c_int64, C.c_int32]
        L.oracle_llround_1e9.restype = C.c_int64
        L.oracle_llround_1e9.argtypes = [C.c_double]
        L.oracle_batch_latency.restype = C.c_double
        L.oracle_batch_latency.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64]
        L.oracle_validate_config.restype = C.c_int32
        L.oracle_validate_config.argtypes = [C.c_void_p]

    def predict_batch(self, cfgs: np.ndarray, ss: abi.ScenarioSet) -> np.ndarray:
        out = np.zeros(len(ss), abi.result_dtype)
        e = ss.entries()
        self.lib.oracle_predict_batch(_vp(cfgs), C.byref(e), _vp(ss.scenarios), len(ss), _vp(out))
        return out

    def trace(self, cfgs: np.ndarray, ss: abi.ScenarioSet, i: int = 0, cap: int = 1 << 20):
        rec = np.zeros(cap, abi.step_dtype)
        out = np.zeros(1, abi.result_dtype)
        n = C.c_int64(0)
        e = ss.entries()
        sc = np.ascontiguousarray(ss.scenarios[i:i + 1])
        cfg = np.ascontiguousarray(cfgs[int(sc["cfg"][0]):int(sc["cfg"][0]) + 1])
        self.lib.oracle_predict(_vp(cfg), C.byref(e), _vp(sc), _vp(out), _vp(rec), cap, C.byref(n))
        return out[0], rec[:min(n.value, cap)]


class Reference:
    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            if not os.path.isdir(REF_SRC):
                raise FileNotFoundError(
                    f"{path} missing and reference sources absent; run oracle.build() where "
                    "/root/reference exists (the built .so travels with the repo snapshot)")
            build(ref=True)
        self.lib = C.CDLL(path)
        L = self.lib
        E = C.POINTER(abi.Entries)
        L.ref_predict_batch.restype = C.c_int
        L.ref_predict_batch.argtypes = [C.c_void_p, E, C.c_void_p, C.c_int64, C.c_void_p, C.c_int]
        L.ref_time_predict.restype = C.c_double
        L.ref_time_predict.argtypes = [C.c_void_p, E, C.c_void_p, C.c_int64, C.c_int, C.c_int]
        L.ref_trace.restype = C.c_int
        L.ref_trace.argtypes = [C.c_void_p, E, C.c_void_p, C.c_void_p, C.c_int64,
                                C.POINTER(C.c_int64), C.c_void_p]
        L.ref_make_workload.restype = C.c_int
        L.ref_make_workload.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        L.ref_run_experiment.restype = C.c_int
        L.ref_run_experiment.argtypes = [C.c_void_p] * 5
        L.ref_replay.restype = C.c_int
        L.ref_replay.argtypes = [C.c_void_p] * 5 + [C.POINTER(C.c_void_p)]
        L.ref_capture_sizes.restype = None
        L.ref_capture_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_capture_copy.restype = None
        L.ref_capture_copy.argtypes = [C.c_void_p] * 7
        L.ref_request_json.restype = C.c_int
        L.ref_request_json.argtypes = [C.c_void_p, E, C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_dump_double.restype = C.c_int
        L.ref_dump_double.argtypes = [C.c_double, C.c_char_p, C.c_int64]
        L.ref_service_predict.restype = C.c_int
        L.ref_service_predict.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_run_report.restype = C.c_int
        L.ref_run_report.argtypes = [C.c_void_p] * 4
        L.ref_capacity_search.restype = C.c_int
        L.ref_capacity_search.argtypes = [C.c_void_p] * 3 + [C.c_uint64, C.c_int32, C.c_int32,
                                                              C.c_double] + [C.c_void_p] * 3 + [C.c_int32]
        L.ref_estimate_noisy.restype = C.c_int32
        L.ref_estimate_noisy.argtypes = [C.c_int32, C.c_uint64, C.c_uint64, C.c_double]
        L.ref_capture_free.restype = None
        L.ref_capture_free.argtypes = [C.c_void_p]
        L.ref_load_trace.argtypes = [C.c_char_p, C.c_int64, C.c_void_p, C.c_int64,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_char_p, C.c_int64]
        L.ref_load_trace.restype = C.c_int64
        L.ref_write_trace.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_int64]
        L.ref_write_trace.restype = C.c_int64
        L.ref_set_trace.argtypes = [C.c_void_p, C.c_int64]
        L.ref_set_trace.restype = None
        L.ref_sweep.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.ref_sweep.restype = C.c_double
        L.ref_run_sweep.argtypes = [C.c_void_p] * 4 + [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                                       C.c_int32, C.c_int32, C.c_void_p]
        L.ref_run_sweep.restype = C.c_int
        L.ref_run_capacity.argtypes = [C.c_void_p] * 4 + [C.c_int32, C.c_int32, C.c_uint64, C.c_int32,
                                                          C.c_int32, C.c_double, C.c_void_p,
                                                          C.POINTER(C.c_double)]
        L.ref_run_capacity.restype = C.c_int

    def predict_batch(self, cfgs, ss: abi.ScenarioSet, threads: int = 1) -> np.ndarray:
        out = np.zeros(len(ss), abi.ref_result_dtype)
        e = ss.entries()
        self.lib.ref_predict_batch(_vp(cfgs), C.byref(e), _vp(ss.scenarios), len(ss), _vp(out),
                                   threads)
        return out

    def time_predict(self, cfgs, ss: abi.ScenarioSet, threads: int, reps: int = 1) -> float:
        e = ss.entries()
        return self.lib.ref_time_predict(_vp(cfgs), C.byref(e), _vp(ss.scenarios), len(ss),
                                         threads, reps)

    def trace(self, cfgs, ss: abi.ScenarioSet, i: int = 0, cap: int = 1 << 20):
        rec = np.zeros(cap, abi.step_dtype)
        out = np.zeros(1, abi.ref_result_dtype)
        n = C.c_int64(0)
        e = ss.entries()
        sc = np.ascontiguousarray(ss.scenarios[i:i + 1])
        cfg = np.ascontiguousarray(cfgs[int(sc["cfg"][0]):int(sc["cfg"][0]) + 1])
        self.lib.ref_trace(_vp(cfg), C.byref(e), _vp(sc), _vp(rec), cap, C.byref(n), _vp(out))
        return out[0], rec[:min(n.value, cap)]

    _trace_n = None

    def _rows(self, w):
        total = int(w["count"][0]) if self._trace_n is None else self._trace_n
        return total if w["request_cap"][0] < 0 else min(total, int(w["request_cap"][0]))

    def load_trace(self, text):
        """load_trace (workload.cpp:51-68): (records, None) or (None, (kind, line, field))."""
        b = text.encode() if isinstance(text, str) else bytes(text)
        cap = b.count(b"\n") + 1
        out = np.zeros(cap, abi.trace_record_dtype)
        kind, line = C.c_int32(0), C.c_int32(0)
        field = C.create_string_buffer(64)
        n = self.lib.ref_load_trace(b, len(b), _vp(out), cap, C.byref(kind), C.byref(line), field, 64)
        if n < 0:
            return None, (kind.value, line.value, field.value.decode())
        return out[:n].copy(), None

    def write_trace(self, recs) -> bytes:
        recs = np.ascontiguousarray(recs, dtype=abi.trace_record_dtype)
        buf = C.create_string_buffer(len(recs) * 160 + 16)
        n = self.lib.ref_write_trace(_vp(recs), len(recs), buf, len(buf))
        assert n >= 0
        return buf.raw[:n]

    def set_trace(self, recs):
        """Replace the synthetic trace of make_workload / run_experiment /
        run_report by these records (None restores it)."""
        if recs is None:
            self.lib.ref_set_trace(None, -1)
            self._trace_n = None
            return
        recs = np.ascontiguousarray(recs, dtype=abi.trace_record_dtype)
        self.lib.ref_set_trace(_vp(recs), len(recs))
        self._trace_n = len(recs)

    def make_workload(self, w):
        n = self._rows(w)
        p, o, e = (np.zeros(max(n, 1), np.int32) for _ in range(3))
        t = np.zeros(max(n, 1), np.int64)
        if self.lib.ref_make_workload(_vp(w), _vp(p), _vp(o), _vp(e), _vp(t)) < 0:
            raise RuntimeError("reference make_workload threw")
        return p[:n], o[:n], e[:n], t[:n]

    def run_experiment(self, w, cfg, spec):
        n = self._rows(w)
        out = np.zeros(n, abi.outcome_dtype)
        summ = np.zeros(1, abi.summary_dtype)
        if self.lib.ref_run_experiment(_vp(w), _vp(cfg), _vp(spec), _vp(out), _vp(summ)) < 0:
            raise RuntimeError("reference run_experiment threw (e.g. an unservable workload)")
        return out, summ[0]

    def request_json(self, cfgs, ss: abi.ScenarioSet, i: int) -> str:
        """prediction_request_to_json (json_io.cpp:125-132) of scenario i."""
        buf = C.create_string_buffer(1 << 22)
        e = ss.entries()
        sc = np.ascontiguousarray(ss.scenarios[i:i + 1])
        cf = np.ascontiguousarray(np.asarray(cfgs)[int(sc["cfg"][0]):int(sc["cfg"][0]) + 1])
        n = self.lib.ref_request_json(_vp(cf), C.byref(e), _vp(sc), buf, len(buf))
        assert n >= 0
        return buf.value.decode()

    def dump_double(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        assert self.lib.ref_dump_double(v, buf, 64) >= 0
        return buf.value.decode()

    def service_predict(self, body: str):
        """The predictor role's /predict (service.cpp:229-241): (HTTP status, body)."""
        buf = C.create_string_buffer(1 << 16)
        code = self.lib.ref_service_predict(body.encode(), buf, len(buf))
        return code, buf.value.decode()

    def run_report(self, w, cfg, spec):
        out = np.zeros(1, abi.report_dtype)
        self.lib.ref_run_report(_vp(w), _vp(cfg), _vp(spec), _vp(out))
        return out[0]

    def capacity_search(self, w, cfg, spec, seed, qps_min, qps_max, slo):
        out = np.zeros(1, abi.capacity_dtype)
        tq = np.zeros(256, np.float64)
        tp = np.zeros(256, np.int32)
        st = self.lib.ref_capacity_search(_vp(w), _vp(cfg), _vp(spec), seed, qps_min, qps_max, slo,
                                          _vp(out), _vp(tq), _vp(tp), 256)
        n = int(out["n_tested"][0])
        return st, out[0], list(zip(tq[:n].tolist(), tp[:n].astype(bool).tolist()))

    def run_sweep(self, w, cfg, spec, policies, qps_values, seeds, jobs: int = 8):
        """The reference's run_sweep (driver.cpp:333-390): SweepCell rows."""
        pol = np.ascontiguousarray(policies, np.int32)
        qps = np.ascontiguousarray(qps_values, np.float64)
        sd = np.ascontiguousarray(seeds, np.uint64)
        rows = np.zeros(len(pol) * len(qps) * len(sd), abi.sweep_row_dtype)
        n = self.lib.ref_run_sweep(_vp(w), _vp(cfg), _vp(spec), _vp(pol), len(pol), _vp(qps), len(qps),
                                   _vp(sd), len(sd), jobs, _vp(rows))
        if n < 0:
            raise RuntimeError("reference run_sweep threw")
        return rows[:n]

    def run_capacity(self, w, cfg, spec, policies, baseline, seed, qps_min, qps_max, slo):
        """The reference's run_capacity (driver.cpp:392-427): (status, rows,
        baseline capacity); status -12 = NoCapacityError."""
        pol = np.ascontiguousarray(policies, np.int32)
        rows = np.zeros(len(pol) + 1, abi.capacity_row_dtype)
        bc = C.c_double(0)
        n = self.lib.ref_run_capacity(_vp(w), _vp(cfg), _vp(spec), _vp(pol), len(pol), baseline, seed,
                                      qps_min, qps_max, slo, _vp(rows), C.byref(bc))
        return (n if n < 0 else 0), rows[:max(n, 0)], bc.value

    def sweep(self, cells, threads: int):
        """capacity_search of every cell, parallel over (cell, qps) points on
        `threads` threads (ref_sweep). Returns (sweep_out rows, wall seconds)."""
        cells = np.ascontiguousarray(cells, abi.sweep_cell_dtype)
        out = np.zeros(len(cells), abi.sweep_out_dtype)
        secs = self.lib.ref_sweep(_vp(cells), len(cells), threads, _vp(out))
        return out, secs

    def replay(self, w, cfg, spec, capture: bool = True):
        n = int(w["count"][0]) if w["request_cap"][0] < 0 else min(int(w["count"][0]),
                                                                    int(w["request_cap"][0]))
        out = np.zeros(n, abi.outcome_dtype)
        summ = np.zeros(1, abi.summary_dtype)
        h = C.c_void_p(None)
        if self.lib.ref_replay(_vp(w), _vp(cfg), _vp(spec), _vp(out), _vp(summ),
                               C.byref(h) if capture else None) < 0:
            raise RuntimeError("reference replay threw (e.g. an unservable workload)")
        ss = None
        if capture:
            ne, ns = C.c_int64(0), C.c_int64(0)
            self.lib.ref_capture_sizes(h, C.byref(ne), C.byref(ns))
            ids = np.zeros(ne.value, np.uint64)
            cols = [np.zeros(ne.value, np.int32) for _ in range(4)]
            sc = np.zeros(ns.value, abi.scenario_dtype)
            self.lib.ref_capture_copy(h, _vp(ids), *[_vp(c) for c in cols], _vp(sc))
            self.lib.ref_capture_free(h)
            ss = abi.ScenarioSet(*cols, sc, ids=ids)
        return out, summ[0], ss


def seconds_to_ticks_exact(sec: np.ndarray) -> np.ndarray:
    """Inverse of SimTime::seconds (ticks * 1e-9, time.h:25), exact for the
    values it produces (the map is injective below ~52 days)."""
    sec = np.asarray(sec, dtype=np.float64)
    t = np.rint(sec * 1e9).astype(np.int64)
    for adj in (0, -1, 1, -2, 2):
        cand = t + adj
        ok = (cand.astype(np.float64) * 1e-9) == sec
        t = np.where(ok, cand, t)
    assert ((t.astype(np.float64) * 1e-9) == sec).all()
    return t


def mc_reference_dispatch(ref, cfg, ss, n_inst, lengths, threads=8):
    """The oracle for cfg4: loop the reference predict() over every (instance,
    sample) with the sample as the candidate's length, sum e2e ticks per
    instance, argmin with lowest-id ties (instance id = index). Returns
    (chosen, scores, sample_e2e)."""
    n_req = len(ss) // n_inst
    S = lengths.shape[1]
    rows = np.repeat(ss.scenarios, S)
    rows["cand_est"] = np.repeat(lengths, n_inst, axis=0).reshape(-1)
    big = abi.ScenarioSet(ss.prompt, ss.est, ss.prefill, ss.decoded, rows)
    rr = ref.predict_batch(cfg, big, threads=threads)
    ok = (rr["status"] == abi.OK).reshape(n_req, n_inst, S)
    e2e = seconds_to_ticks_exact(np.where(rr["status"] == abi.OK, rr["e2e_s"], 0.0))
    e2e = e2e.reshape(n_req, n_inst, S)
    scores = e2e.sum(axis=2)
    chosen = np.where(ok.all(axis=(1, 2)), scores.argmin(axis=1), -1)  # argmin: first (lowest id)
    return chosen, scores.reshape(-1), e2e.reshape(n_req * n_inst, S)


def compare_to_ref(gpu_res: np.ndarray, ref_res: np.ndarray) -> np.ndarray:
    """Boolean mask of scenarios whose product result (ticks) differs from the
    reference's (double seconds): status, steps, and e2e/ttft/qdelay compared
    bit-exactly as ticks * 1e-9 (time.h:25); failures compare status + detail."""
    ok = gpu_res["status"] == ref_res["status"]
    good = ok & (gpu_res["status"] == abi.OK)
    for tk, sk in (("e2e_ticks", "e2e_s"), ("ttft_ticks", "ttft_s"), ("qdelay_ticks", "qdelay_s")):
        sec = abi.ticks_to_seconds(gpu_res[tk])
        ok &= ~good | (sec.view(np.int64) == ref_res[sk].view(np.int64))
    ok &= ~good | (gpu_res["steps"] == ref_res["steps"])
    # failures: the error detail too (deadlocked member's origin, the candidate's
    # block need for TOO_LARGE_CANDIDATE; 0 where the reference message has none)
    ok &= good | (gpu_res["detail"] == ref_res["detail"])
    return ~ok

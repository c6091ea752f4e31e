"""numpy/ctypes mirror of the C-ABI structs in include/blocksim_b200.h.

Layouts are asserted against the header's stated sizes; every array passed
across the boundary is a C-contiguous numpy array of one of these dtypes.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

# bsg_status (include/blocksim_b200.h)
OK = 0
TOO_LARGE_RUNNING = 1
TOO_LARGE_CANDIDATE = 2
DEADLOCK = 3
STEP_LIMIT = 4
VANISHED = 5
EMPTY_PLAN = 6
BAD_INPUT = 7
BAD_CONFIG = 8
CUDA_ERROR = 9
NO_INSTANCES = 10
INVALID_ARGUMENT = 11
STATUS_NAMES = {
    0: "OK", 1: "TOO_LARGE_RUNNING", 2: "TOO_LARGE_CANDIDATE", 3: "DEADLOCK",
    4: "STEP_LIMIT", 5: "VANISHED", 6: "EMPTY_PLAN", 7: "BAD_INPUT", 8: "BAD_CONFIG",
    9: "CUDA_ERROR", 10: "NO_INSTANCES", 11: "INVALID_ARGUMENT",
}

CHUNKED_PREFILL = 0
PREFILL_PRIORITY = 1
CACHE_OFF, CACHE_EXACT, CACHE_BUCKETED = 0, 1, 2
POLICY_RANDOM, POLICY_ROUND_ROBIN, POLICY_MIN_QPM, POLICY_INFAAS_PP, POLICY_LLUMNIX_MINUS, \
    POLICY_BLOCK_PREDICTIVE = range(6)

cfg_dtype = np.dtype([
    ("total_blocks", "<i4"), ("block_size", "<i4"), ("max_batch_size", "<i4"),
    ("chunk_budget", "<i4"), ("local_policy", "<i4"), ("cache_mode", "<i4"),
    ("context_bucket", "<i4"), ("reserved", "<i4"),
    ("c0_s", "<f8"), ("prefill_s_per_token", "<f8"), ("decode_s_per_seq", "<f8"),
    ("context_s_per_token", "<f8"),
])
scenario_dtype = np.dtype([
    ("run_off", "<i4"), ("run_n", "<i4"), ("wait_off", "<i4"), ("wait_n", "<i4"),
    ("cand_prompt", "<i4"), ("cand_est", "<i4"), ("cfg", "<i4"), ("reserved", "<i4"),
])
result_dtype = np.dtype([
    ("e2e_ticks", "<i8"), ("ttft_ticks", "<i8"), ("qdelay_ticks", "<i8"), ("steps", "<i8"),
    ("member_steps", "<i8"), ("status", "<i4"), ("detail", "<i4"),
])
ref_result_dtype = np.dtype([
    ("e2e_s", "<f8"), ("ttft_s", "<f8"), ("qdelay_s", "<f8"), ("steps", "<i8"),
    ("status", "<i4"), ("detail", "<i4"),
])
step_dtype = np.dtype([
    ("duration_ticks", "<i8"), ("context_tokens", "<i8"), ("n_decode", "<i4"),
    ("prefill_tokens", "<i4"), ("n_prefill", "<i4"), ("n_preempted", "<i4"),
    ("n_completed", "<i4"), ("free_blocks_after", "<i4"), ("plan_hash", "<u8"),
    ("event_hash", "<u8"),
])
workload_dtype = np.dtype([
    ("count", "<i4"), ("min_tokens", "<i4"), ("max_prompt_tokens", "<i4"),
    ("max_output_tokens", "<i4"), ("trace_seed", "<u8"), ("prompt_median", "<f8"),
    ("prompt_sigma", "<f8"), ("output_median", "<f8"), ("output_sigma", "<f8"),
    ("estimator_kind", "<i4"), ("fixed_tokens", "<i4"), ("mean_abs_rel_error", "<f8"),
    ("estimator_seed", "<u8"), ("qps", "<f8"), ("arrival_seed", "<u8"),
    ("request_cap", "<i4"), ("reserved", "<i4"),
])
replay_spec_dtype = np.dtype([
    ("n_instances", "<i4"), ("policy", "<i4"), ("objective", "<i4"), ("capture", "<i4"),
    ("policy_seed", "<u8"), ("provision_kind", "<i4"), ("max_instances", "<i4"),
    ("threshold_s", "<f8"), ("cold_start_s", "<f8"), ("cooldown_s", "<f8"),
    ("dispatch_overhead_s", "<f8"),
])
summary_dtype = np.dtype([
    ("total_preemptions", "<i8"), ("end_ticks", "<i8"), ("instances_provisioned", "<i4"),
    ("final_instance_count", "<i4"),
])
report_dtype = np.dtype([
    ("finished_requests", "<i4"), ("censored_requests", "<i4"), ("throughput_rps", "<f8"),
    ("mean_ttft_s", "<f8"), ("p50_ttft_s", "<f8"), ("p99_ttft_s", "<f8"),
    ("mean_e2e_s", "<f8"), ("p50_e2e_s", "<f8"), ("p99_e2e_s", "<f8"),
    ("total_preemptions", "<i8"), ("instances_provisioned", "<i4"),
    ("final_instance_count", "<i4"), ("free_blocks_mean_avg", "<f8"), ("free_blocks_var_avg", "<f8"),
    ("mean_overhead_s", "<f8"),
])
capacity_dtype = np.dtype([
    ("capacity_qps", "<f8"), ("bracket_pass", "<i4"), ("bracket_fail", "<i4"),
    ("monotone", "<i4"), ("n_tested", "<i4"),
])
capacity_row_dtype = np.dtype([
    ("policy", "<i4"), ("status", "<i4"), ("result", capacity_dtype), ("has_gain", "<i4"),
    ("reserved", "<i4"), ("gain", "<f8"), ("gain_text", "S16")])
sweep_cell_dtype = np.dtype([
    ("workload", workload_dtype), ("cfg", cfg_dtype), ("spec", replay_spec_dtype),
    ("seed", "<u8"), ("qps_min", "<i4"), ("qps_max", "<i4"), ("slo_p99_ttft_s", "<f8"),
])
sweep_out_dtype = np.dtype([
    ("status", "<i4"), ("reserved", "<i4"), ("result", capacity_dtype),
    ("whatif_scenarios", "<i8"), ("kernel_launches", "<i8"), ("wall_s", "<f8"),
])
NO_CAPACITY = 12
STATUS_NAMES[12] = "NO_CAPACITY"
PROVISION_STATIC, PROVISION_PREEMPT, PROVISION_RELIEF = 0, 1, 2
closed_loop_run_dtype = np.dtype([
    ("n_instances", "<i4"), ("objective", "<i4"), ("cfg", "<i4"), ("n_requests", "<i4"),
    ("req_off", "<i8"), ("provision_kind", "<i4"), ("max_instances", "<i4"),
    ("threshold_s", "<f8"), ("cold_start_s", "<f8"), ("cooldown_s", "<f8"),
    ("policy", "<i4"), ("reserved", "<i4"), ("policy_seed", "<u8"), ("dispatch_overhead_s", "<f8")])
sweep_row_dtype = np.dtype([
    ("policy", "<i4"), ("ok", "<i4"), ("qps", "<f8"), ("seed", "<u8"), ("status", "<i4"),
    ("finished_requests", "<i4"), ("mean_ttft_s", "<f8"), ("p99_ttft_s", "<f8"),
    ("mean_e2e_s", "<f8"), ("p99_e2e_s", "<f8"), ("throughput_rps", "<f8"),
    ("total_preemptions", "<i8"), ("free_blocks_var_avg", "<f8")])
outcome_dtype = np.dtype([
    ("arrival_ticks", "<i8"), ("dispatch_ticks", "<i8"), ("first_token_ticks", "<i8"),
    ("finish_ticks", "<i8"), ("instance", "<i4"), ("preempt_count", "<i4"),
])

trace_record_dtype = np.dtype([
    ("id", "<u8"), ("prompt_tokens", "<i4"), ("output_tokens", "<i4"),
    ("estimated_output_tokens", "<i4"), ("has_arrival_offset", "<i4"), ("arrival_offset_s", "<f8")])


class TraceError(C.Structure):
    _fields_ = [("kind", C.c_int32), ("line", C.c_int32), ("field", C.c_char * 40),
                ("message", C.c_char * 216)]


ESTIMATOR_ORACLE, ESTIMATOR_FIXED, ESTIMATOR_NOISY, ESTIMATOR_TRACE = 0, 1, 2, 3

assert trace_record_dtype.itemsize == 32
assert C.sizeof(TraceError) == 264
assert cfg_dtype.itemsize == 64
assert scenario_dtype.itemsize == 32
assert result_dtype.itemsize == 48
assert step_dtype.itemsize == 56
assert outcome_dtype.itemsize == 40


class Entries(C.Structure):
    """bsg_entries: SoA column pointers."""
    _fields_ = [("id", C.c_void_p), ("prompt", C.c_void_p), ("est", C.c_void_p),
                ("prefill", C.c_void_p), ("decoded", C.c_void_p)]


def ptr(a: np.ndarray | None) -> C.c_void_p | None:
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C-ABI must be contiguous"
    return C.c_void_p(a.ctypes.data)


def make_config(total_blocks=1056, block_size=16, max_batch_size=48, chunk_budget=512,
                local_policy=CHUNKED_PREFILL, cache_mode=CACHE_OFF, context_bucket=256,
                c0_s=0.01, prefill_s_per_token=1e-4, decode_s_per_seq=1e-3,
                context_s_per_token=1e-7) -> np.ndarray:
    """InstanceConfig defaults (types.h:46-66) — the 'Llama-2-7B profile' of BASELINE.json."""
    c = np.zeros(1, cfg_dtype)
    c["total_blocks"], c["block_size"] = total_blocks, block_size
    c["max_batch_size"], c["chunk_budget"] = max_batch_size, chunk_budget
    c["local_policy"], c["cache_mode"], c["context_bucket"] = local_policy, cache_mode, context_bucket
    c["c0_s"], c["prefill_s_per_token"] = c0_s, prefill_s_per_token
    c["decode_s_per_seq"], c["context_s_per_token"] = decode_s_per_seq, context_s_per_token
    return c


def make_workload(count=1000, trace_seed=1234, prompt_median=230.0, prompt_sigma=0.7,
                  output_median=160.0, output_sigma=1.0, min_tokens=4, max_prompt_tokens=4096,
                  max_output_tokens=8192, estimator_kind=0, fixed_tokens=256,
                  mean_abs_rel_error=0.244, estimator_seed=0, qps=1.0, arrival_seed=0,
                  request_cap=-1) -> np.ndarray:
    """SyntheticTraceSpec (workload.h:63-75) + LengthEstimator + arrivals."""
    w = np.zeros(1, workload_dtype)
    for k, v in dict(count=count, trace_seed=trace_seed, prompt_median=prompt_median,
                     prompt_sigma=prompt_sigma, output_median=output_median,
                     output_sigma=output_sigma, min_tokens=min_tokens,
                     max_prompt_tokens=max_prompt_tokens, max_output_tokens=max_output_tokens,
                     estimator_kind=estimator_kind, fixed_tokens=fixed_tokens,
                     mean_abs_rel_error=mean_abs_rel_error, estimator_seed=estimator_seed,
                     qps=qps, arrival_seed=arrival_seed, request_cap=request_cap).items():
        w[k] = v
    return w


def make_replay_spec(n_instances, policy=POLICY_BLOCK_PREDICTIVE, objective=0, capture=1,
                     policy_seed=0, provision_kind=PROVISION_STATIC, max_instances=None,
                     threshold_s=70.0, cold_start_s=30.0, cooldown_s=15.0,
                     dispatch_overhead_s=0.0) -> np.ndarray:
    """ExperimentSpec subset + ProvisionPolicy (autoscaler.h:10-27) defaults."""
    s = np.zeros(1, replay_spec_dtype)
    s["n_instances"], s["policy"], s["objective"] = n_instances, policy, objective
    s["capture"], s["policy_seed"] = capture, policy_seed
    s["provision_kind"] = provision_kind
    s["max_instances"] = n_instances if max_instances is None else max_instances
    s["threshold_s"], s["cold_start_s"], s["cooldown_s"] = threshold_s, cold_start_s, cooldown_s
    s["dispatch_overhead_s"] = dispatch_overhead_s
    return s


class ScenarioSet:
    """A batch of what-if scenarios: SoA entry columns + scenario rows."""

    def __init__(self, prompt, est, prefill, decoded, scenarios, ids=None):
        self.prompt = np.ascontiguousarray(prompt, dtype=np.int32)
        self.est = np.ascontiguousarray(est, dtype=np.int32)
        self.prefill = np.ascontiguousarray(prefill, dtype=np.int32)
        self.decoded = np.ascontiguousarray(decoded, dtype=np.int32)
        self.ids = None if ids is None else np.ascontiguousarray(ids, dtype=np.uint64)
        self.scenarios = np.ascontiguousarray(scenarios, dtype=scenario_dtype)

    @property
    def n_entries(self) -> int:
        return int(self.prompt.shape[0])

    def __len__(self) -> int:
        return int(self.scenarios.shape[0])

    def entries(self) -> Entries:
        return Entries(ptr(self.ids), ptr(self.prompt), ptr(self.est), ptr(self.prefill),
                       ptr(self.decoded))

    def subset(self, idx) -> "ScenarioSet":
        return ScenarioSet(self.prompt, self.est, self.prefill, self.decoded,
                           self.scenarios[idx], self.ids)

    def compact(self, rows) -> "ScenarioSet":
        """A self-contained copy holding only the entries the selected scenario
        rows reference (what a caller packs for one dispatch call)."""
        sc = np.array(self.scenarios[rows], dtype=scenario_dtype)
        cols = [[], [], [], []]
        src = (self.prompt, self.est, self.prefill, self.decoded)
        off = 0
        for r in sc:
            for start_key, n_key in (("run_off", "run_n"), ("wait_off", "wait_n")):
                a, b = int(r[start_key]), int(r[n_key])
                for c, col in zip(cols, src):
                    c.append(col[a:a + b])
                r[start_key] = off
                off += b
        cat = [np.concatenate(c) if c else np.zeros(0, np.int32) for c in cols]
        return ScenarioSet(*cat, sc)

    def member_capacity(self, cfgs: np.ndarray) -> int:
        """max(run_n, min(max_batch_size, run_n + wait_n + 1)) over the set."""
        sc = self.scenarios
        maxb = cfgs["max_batch_size"][sc["cfg"]]
        need = np.maximum(sc["run_n"], np.minimum(maxb, sc["run_n"] + sc["wait_n"] + 1))
        return int(need.max()) if len(sc) else 1

    def nbytes_in(self) -> int:
        return (self.prompt.nbytes + self.est.nbytes + self.prefill.nbytes + self.decoded.nbytes
                + self.scenarios.nbytes)

    @staticmethod
    def from_snapshots(snapshots, candidates, cfg_index=None) -> "ScenarioSet":
        """snapshots: list of (running, waiting) with entries (prompt, est, prefill, decoded);
        candidates: list of (prompt, est)."""
        cols = [[], [], [], []]
        sc = np.zeros(len(snapshots), scenario_dtype)
        for i, ((running, waiting), (cp, ce)) in enumerate(zip(snapshots, candidates)):
            sc[i]["run_off"] = len(cols[0])
            sc[i]["run_n"] = len(running)
            for r in running:
                for c, v in zip(cols, r):
                    c.append(v)
            sc[i]["wait_off"] = len(cols[0])
            sc[i]["wait_n"] = len(waiting)
            for r in waiting:
                for c, v in zip(cols, r):
                    c.append(v)
            sc[i]["cand_prompt"], sc[i]["cand_est"] = cp, ce
            sc[i]["cfg"] = 0 if cfg_index is None else cfg_index[i]
        return ScenarioSet(*[np.array(c, dtype=np.int32) for c in cols], sc)


def ticks_to_seconds(ticks) -> np.ndarray:
    """SimTime::seconds (time.h:25): ticks * 1e-9 in double."""
    return np.asarray(ticks, dtype=np.int64).astype(np.float64) * 1e-9

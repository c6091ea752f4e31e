/*
 * blocksim_b200.h — C-ABI of the B200-native what-if simulation core.
 *
 * This is the drop-in boundary for Block's predictive-dispatch hot path
 * (arXiv 2508.03611, reference implementation "blocksim"):
 *
 *   reference interface                                   replaced by
 *   ----------------------------------------------------  ------------------------------
 *   predict()            core/src/predictor.cpp:76-137     bsg_predict_batch[_device]
 *   predict_across()     core/src/predictor.cpp:139-157    bsg_predict_batch (1 scenario
 *                                                          per snapshot, same candidate)
 *   PredictorClient::predict_across (scheduler.h:56-61)    bsg_predict_batch via the C++
 *                                                          GpuPredictorClient
 *   Dispatcher::dispatch BlockPredictive argmin
 *                        core/src/scheduler.cpp:115-152    bsg_dispatch / bsg_dispatch_mc
 *   Instance::execute_step loop (per-step StepResult)
 *                        core/src/backend.cpp:338-349      bsg_trace (parity/trace mode)
 *   InstanceConfig + CostModelParams  types.h:46-66         bsg_instance_cfg
 *   LatencyCache modes   core/src/predictor.cpp:26-54      bsg_instance_cfg.cache_mode
 *   SnapshotRequest / InstanceSnapshot types.h:75-94        bsg_entries (SoA) + bsg_scenario
 *   PredictionResult     predictor.h:28-36                 bsg_result (integer ns ticks)
 *
 * Conventions: plain pointers and sizes, no exceptions, no torch types.
 * Every call returns a bsg_status; per-scenario failures are reported in
 * bsg_result.status with the reference's error taxonomy (error.h:31-56).
 * Times are integer nanosecond ticks (SimTime, time.h:14-42); the reference's
 * double seconds are ticks * 1e-9 (time.h:25), reproduced bit-exactly by
 * bsg_ticks_to_seconds().
 */
#ifndef BLOCKSIM_B200_H
#define BLOCKSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSG_ABI_VERSION 1

typedef enum bsg_status {
  BSG_OK = 0,
  /* RequestTooLargeError("snapshot running set exceeds total memory blocks")
   * backend.cpp:42-44 -> PredictionError("candidate does not fit ...") predictor.cpp:134-135 */
  BSG_TOO_LARGE_RUNNING = 1,
  /* RequestTooLargeError from Instance::admit of the candidate, backend.cpp:76-83 */
  BSG_TOO_LARGE_CANDIDATE = 2,
  /* DeadlockError backend.cpp:274-277 -> PredictionError predictor.cpp:132-133;
   * detail = origin index of the deadlocked member */
  BSG_DEADLOCK = 3,
  /* PredictionError("forward simulation exceeded the step limit") predictor.cpp:125-127 */
  BSG_STEP_LIMIT = 4,
  /* PredictionError("candidate vanished from the forward simulation") predictor.cpp:102-104 */
  BSG_VANISHED = 5,
  /* EmptyPlanError backend.cpp:245 (not caught by predict: propagates as EmptyPlanError) */
  BSG_EMPTY_PLAN = 6,
  /* input outside the supported integer domain */
  BSG_BAD_INPUT = 7,
  /* ConfigError from validate_instance_config, types.cpp:47-61; detail = field code */
  BSG_BAD_CONFIG = 8,
  BSG_CUDA_ERROR = 9,
  /* NoInstancesError, predictor.cpp:144 / scheduler.cpp:116 */
  BSG_NO_INSTANCES = 10,
  BSG_INVALID_ARGUMENT = 11,
  /* NoCapacityError: the lowest swept qps already violates the SLO (metrics.cpp:153-155) */
  BSG_NO_CAPACITY = 12
} bsg_status;

typedef enum bsg_local_policy {
  BSG_CHUNKED_PREFILL = 0,  /* LocalPolicy::kChunkedPrefill, backend.cpp:113-149 */
  BSG_PREFILL_PRIORITY = 1  /* LocalPolicy::kPrefillPriority, backend.cpp:151-182 */
} bsg_local_policy;

typedef enum bsg_cache_mode {
  BSG_CACHE_OFF = 0,      /* predict(req, nullptr)                        */
  BSG_CACHE_EXACT = 1,    /* transparent: identical to OFF (predictor.cpp:43-47) */
  BSG_CACHE_BUCKETED = 2  /* context rounded to (C + b/2)/b*b (predictor.cpp:29-32) */
} bsg_cache_mode;

/* InstanceConfig + CostModelParams (types.h:46-66) + predictor cache mode.
 * 64 bytes, naturally aligned. */
typedef struct bsg_instance_cfg {
  int32_t total_blocks;    /* 1056 */
  int32_t block_size;      /* 16   */
  int32_t max_batch_size;  /* 48   */
  int32_t chunk_budget;    /* 512  */
  int32_t local_policy;    /* bsg_local_policy */
  int32_t cache_mode;      /* bsg_cache_mode   */
  int32_t context_bucket;  /* 256; clamped to >= 1 like LatencyCache (predictor.cpp:23-24) */
  int32_t reserved;
  double c0_s;                 /* 0.01 */
  double prefill_s_per_token;  /* 1e-4 */
  double decode_s_per_seq;     /* 1e-3 */
  double context_s_per_token;  /* 1e-7 */
} bsg_instance_cfg;

/* Snapshot entries (SnapshotRequest, types.h:75-81) as SoA columns.
 * `id` is optional (may be NULL); it is only used host-side for messages. */
typedef struct bsg_entries {
  const uint64_t* id;
  const int32_t* prompt;     /* prompt_tokens            */
  const int32_t* est;        /* estimated_output_tokens  */
  const int32_t* prefill;    /* prefill_progress         */
  const int32_t* decoded;    /* decoded_tokens           */
} bsg_entries;

/* One what-if scenario: snapshot (running + waiting slices of the entry
 * columns) + candidate + instance config index. 32 bytes. */
typedef struct bsg_scenario {
  int32_t run_off, run_n;    /* InstanceSnapshot::running, oldest admission first */
  int32_t wait_off, wait_n;  /* InstanceSnapshot::waiting, head first            */
  int32_t cand_prompt;       /* CandidateRequest::prompt_tokens                   */
  int32_t cand_est;          /* CandidateRequest::estimated_output_tokens         */
  int32_t cfg;               /* index into the configs set by bsg_set_configs     */
  int32_t reserved;
} bsg_scenario;

/* PredictionResult (predictor.h:28-36) in integer ticks. 48 bytes.
 * member_steps = sum over simulated steps of (surviving plan items + 1), the
 * algorithmic work unit of SURVEY.md 8(d) (not part of the reference result). */
typedef struct bsg_result {
  int64_t e2e_ticks;     /* predicted_e2e_latency    */
  int64_t ttft_ticks;    /* predicted_ttft           */
  int64_t qdelay_ticks;  /* predicted_queueing_delay */
  int64_t steps;         /* simulated_steps          */
  int64_t member_steps;  /* work counter (roofline numerator) */
  int32_t status;        /* bsg_status               */
  int32_t detail;        /* status-specific (origin index, field code, ...) */
} bsg_result;

/* One simulated step in trace mode (Instance::execute_step's StepResult,
 * backend.h:40-47, reduced to exact integer fingerprints). 56 bytes.
 * Origins: running entry i -> i, waiting entry j -> run_n + j, candidate -> -1. */
typedef struct bsg_step_record {
  int64_t duration_ticks;    /* SimTime::from_seconds(latency(plan))      */
  int64_t context_tokens;    /* BatchPlan::context_tokens                 */
  int32_t n_decode;          /* |BatchPlan::decode_ids|                   */
  int32_t prefill_tokens;    /* BatchPlan::total_prefill_tokens           */
  int32_t n_prefill;         /* |BatchPlan::prefill_segments|             */
  int32_t n_preempted;       /* |StepResult::preempted|                   */
  int32_t n_completed;       /* |StepResult::completed|                   */
  int32_t free_blocks_after; /* Instance::free_blocks() after finish_step */
  uint64_t plan_hash;        /* bsg_hash over (k, origin, chunk) of plan items in order */
  uint64_t event_hash;       /* bsg_hash over preempted (in order), started, first tokens, completed */
} bsg_step_record;

#if defined(__CUDACC__)
#define BSG_HD __host__ __device__
#else
#define BSG_HD
#endif

/* Mixing function shared by the kernel, the oracle and the reference shim
 * (SplitMix64 finaliser, rand.h:16-21). */
static inline BSG_HD uint64_t bsg_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
/* Fingerprint term of item k of list `tag` with origin o and value v; lists
 * hash as the wrapping SUM of their terms (order enters through k). */
static inline BSG_HD uint64_t bsg_hash_term(uint32_t tag, uint32_t k, int32_t origin, int32_t v) {
  return bsg_mix64(((uint64_t)tag << 56) ^ ((uint64_t)k << 32) ^ (uint64_t)(uint32_t)(origin + 1)) +
         bsg_mix64((uint64_t)(uint32_t)v + 0x9e3779b97f4a7c15ULL * (uint64_t)(k + 1));
}
#define BSG_TAG_PLAN 1u
#define BSG_TAG_PREEMPT 2u
#define BSG_TAG_STARTED 3u
#define BSG_TAG_FIRST 4u
#define BSG_TAG_COMPLETED 5u

/* ---- context ------------------------------------------------------------ */
typedef struct bsg_ctx bsg_ctx;

int bsg_abi_version(void);
/* SimTime::seconds (time.h:25): ticks * 1e-9 in double. */
double bsg_ticks_to_seconds(int64_t ticks);
/* Creates a context bound to CUDA device `device`. Fails loudly with
 * BSG_CUDA_ERROR when no device is present: there is no CPU path. */
bsg_status bsg_ctx_create(int device, bsg_ctx** out);
void bsg_ctx_destroy(bsg_ctx* ctx);
const char* bsg_last_error(const bsg_ctx* ctx);
/* Number of kernel launches issued by this context so far. */
int64_t bsg_launch_count(const bsg_ctx* ctx);

/* Validates (validate_instance_config, types.cpp:47-61) and uploads configs.
 * On BSG_BAD_CONFIG, bad_index and field_code identify the first offender
 * (field codes: 1 total_blocks, 2 block_size, 3 max_batch_size, 4 chunk_budget,
 *  5 c0_s, 6 prefill_s_per_token, 7 decode_s_per_seq, 8 context_s_per_token). */
bsg_status bsg_set_configs(bsg_ctx* ctx, const bsg_instance_cfg* cfgs, int32_t n,
                           int32_t* bad_index, int32_t* field_code);

/* predict() over n scenarios, HOST buffers; synchronous. Copies the entry
 * columns and scenarios host->device, runs the scenario kernel, copies the
 * results device->host. */
bsg_status bsg_predict_batch(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                             const bsg_scenario* scenarios, int64_t n, bsg_result* out);

/* Same, with DEVICE pointers (entries columns, scenarios, out), enqueued on
 * `stream` (a cudaStream_t; NULL = the context's own stream); asynchronous.
 * member_capacity: an upper bound the caller guarantees on
 * max(run_n, min(max_batch_size, run_n + wait_n + 1)) over the scenarios
 * (it selects the kernel's per-warp member capacity, 32/64/128/256); <= 0
 * derives it from the configs' max_batch_size. Scenarios exceeding the
 * capacity report BSG_BAD_INPUT. */
bsg_status bsg_predict_batch_device(bsg_ctx* ctx, const bsg_entries* dev_entries,
                                    const bsg_scenario* dev_scenarios, int64_t n,
                                    int32_t member_capacity, bsg_result* dev_out, void* stream);

/* Trace mode: runs ONE scenario (host buffers) and writes one record per
 * simulated step (up to `cap`); *n_steps receives the total step count. */
bsg_status bsg_trace(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                     const bsg_scenario* scenario, bsg_step_record* records, int64_t cap,
                     int64_t* n_steps, bsg_result* out);

/* BlockPredictive dispatch (scheduler.cpp:115-152): for each of n_requests
 * arrivals, scenarios [r*n_inst, (r+1)*n_inst) are the per-instance what-ifs
 * (instance ids given in `instance_ids`, per request block, any order).
 * chosen[r] = argmin over e2e (objective 0) or ttft (objective 1) with the
 * lowest-id tie-break. per_instance may be NULL. HOST buffers. If any
 * scenario of a request fails, chosen[r] = -1 and status reports it. */
bsg_status bsg_dispatch(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                        const bsg_scenario* scenarios, const int32_t* instance_ids,
                        int32_t n_inst, int32_t n_requests, int32_t objective,
                        int32_t* chosen, bsg_result* per_instance);

/* Monte-Carlo BlockPredictive dispatch (BASELINE cfg4; an extension: the
 * reference has no sampling loop). For each of n_requests arrivals,
 * scenarios [r*n_inst, (r+1)*n_inst) are the per-instance what-ifs (the
 * candidate's cand_est is ignored) and lengths[r*n_samples ...] are its sampled
 * response lengths (bsg_mc_lengths). Per instance, score = sum over samples of
 * the e2e ticks predict() would return with that sample as the candidate's
 * length (objective 0), or n_samples * ttft (objective 1); chosen[r] = argmin,
 * lowest instance id on ties, -1 if any (instance, sample) fails. One
 * simulation per (request, instance) serves all samples (prefix sharing).
 * Optional outputs: scores [n_req*n_inst], sample_e2e [n_req*n_inst*n_samples],
 * per_instance [n_req*n_inst]. HOST buffers; 1 <= n_samples <= 1024. */
bsg_status bsg_dispatch_mc(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                           const bsg_scenario* scenarios, const int32_t* instance_ids,
                           int32_t n_inst, int32_t n_requests, const int32_t* lengths,
                           int32_t n_samples, int32_t objective, int32_t* chosen,
                           int64_t* scores, int64_t* sample_e2e, bsg_result* per_instance);

/* Sampled response lengths for one request: estimate_length's Noisy formula
 * (workload.cpp:126-136) applied to the predicted length `est`:
 * L_s = max(1, round(est * (1 + sign * |N(0,1)| * err * sqrt(pi/2)))), with
 * SplitMix64(mix_seed(seed, request_id * n_samples + s)) (rand.h:11-56). */
bsg_status bsg_mc_lengths(int32_t est, uint64_t request_id, int32_t n_samples, uint64_t seed,
                          double mean_abs_rel_error, int32_t* out);

/* bsg_dispatch_mc with the samples drawn ON THE DEVICE inside the call (K3):
 * request r's n_samples lengths are bsg_mc_lengths(cand_est, request_ids[r],
 * n_samples, seed, mean_abs_rel_error) of its scenarios' (common) cand_est,
 * generated and sorted per warp in shared memory, so the sampling cost is
 * part of the dispatch. Optional outputs: scores [n_req*n_inst], lengths_out
 * [n_req*n_samples] (the drawn samples, sample order), per_instance, and
 * dev_keys — a DEVICE buffer [n_req] receiving the packed argmin key
 * (min(score, 2^47-1) << 16 | id, or -1 when the request failed) for a
 * cross-GPU MIN reduction (instance ids must then be < 65535),
 * complete when the call returns. HOST buffers otherwise. */
bsg_status bsg_dispatch_mc_sampled(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                                   const bsg_scenario* scenarios, const int32_t* instance_ids,
                                   int32_t n_inst, int32_t n_requests, const uint64_t* request_ids,
                                   int32_t n_samples, uint64_t seed, double mean_abs_rel_error,
                                   int32_t objective, int32_t* chosen, int64_t* scores,
                                   int32_t* lengths_out, bsg_result* per_instance, int64_t* dev_keys);

/* Name(s) of the simulation kernel(s) this context's last predict / dispatch
 * call launched (template arguments included), for measurement records. */
const char* bsg_last_launch(const bsg_ctx* ctx);

/* ---- several GPUs in one process ---------------------------
 * One context per device, one persistent host worker thread per context: the
 * devices' copies and kernels run concurrently. No data-path collective —
 * scenarios are independent; the only exchange is the per-request argmin,
 * which stays on one device when requests are split and is merged exactly on
 * the host (lowest id on ties, scheduler.cpp:138-150) when one request's
 * instances are split. A device may appear more than once (several contexts
 * on one GPU). This is what a PredictorClient fanning out over a box's GPUs
 * binds (the reference's predictor replicas, service.cpp:218-246, and its
 * concurrent sweep cells, driver.cpp:375-388). HOST buffers throughout. */
typedef struct bsg_multi bsg_multi;
bsg_status bsg_multi_create(const int* devices, int32_t n_devices, bsg_multi** out);
void bsg_multi_destroy(bsg_multi* m);
int32_t bsg_multi_device_count(const bsg_multi* m);
const char* bsg_multi_last_error(const bsg_multi* m);
int64_t bsg_multi_launch_count(const bsg_multi* m);
/* bsg_set_configs on every device. */
bsg_status bsg_multi_set_configs(bsg_multi* m, const bsg_instance_cfg* cfgs, int32_t n,
                                 int32_t* bad_index, int32_t* field_code);
/* bsg_predict_batch with the batch split into contiguous ranges of whole
 * `group`s (e.g. group = instances per arrival) across the devices. */
bsg_status bsg_multi_predict_batch(bsg_multi* m, const bsg_entries* entries, int64_t n_entries,
                                   const bsg_scenario* scenarios, int64_t n, int32_t group,
                                   bsg_result* out);
/* bsg_dispatch with the requests split across the devices. */
bsg_status bsg_multi_dispatch(bsg_multi* m, const bsg_entries* entries, int64_t n_entries,
                              const bsg_scenario* scenarios, const int32_t* instance_ids,
                              int32_t n_inst, int32_t n_requests, int32_t objective,
                              int32_t* chosen, bsg_result* per_instance);
/* ONE Monte-Carlo dispatch (bsg_dispatch_mc_sampled semantics, one request)
 * with its instances split i % n_devices; per-device (score, id) minima
 * merged on the host. scores (optional) in instance order. */
bsg_status bsg_multi_dispatch_mc_sampled(bsg_multi* m, const bsg_entries* entries, int64_t n_entries,
                                         const bsg_scenario* scenarios, const int32_t* instance_ids,
                                         int32_t n_inst, uint64_t request_id, int32_t n_samples,
                                         uint64_t seed, double mean_abs_rel_error, int32_t objective,
                                         int32_t* chosen, int64_t* scores);

/* ---- closed-loop replay (the scenario source; driver.cpp:134-289) -------- */

/* Synthetic ShareGPT-shaped workload: make_synthetic_trace (workload.cpp:172-191,
 * SyntheticTraceSpec workload.h:63-75), estimate_length (workload.cpp:113-139),
 * generate_arrivals (workload.cpp:141-170). */
typedef struct bsg_workload {
  int32_t count;              /* 1000 */
  int32_t min_tokens;         /* 4 */
  int32_t max_prompt_tokens;  /* 4096 */
  int32_t max_output_tokens;  /* 8192 */
  uint64_t trace_seed;        /* SyntheticTraceSpec::seed */
  double prompt_median, prompt_sigma;  /* 230, 0.7 */
  double output_median, output_sigma;  /* 160, 1.0 */
  int32_t estimator_kind;     /* 0 oracle, 1 fixed, 2 noisy, 3 trace (EstimatorKind; 3 only with trace records) */
  int32_t fixed_tokens;       /* 256 */
  double mean_abs_rel_error;  /* 0.244 */
  uint64_t estimator_seed;
  double qps;
  uint64_t arrival_seed;      /* workload.seed */
  int32_t request_cap;        /* < 0: none */
  int32_t reserved;
} bsg_workload;

/* PolicyKind order (scheduler.h:16-23). */
typedef enum bsg_policy {
  BSG_POLICY_RANDOM = 0,
  BSG_POLICY_ROUND_ROBIN = 1,
  BSG_POLICY_MIN_QPM = 2,
  BSG_POLICY_INFAAS_PP = 3,
  BSG_POLICY_LLUMNIX_MINUS = 4,
  BSG_POLICY_BLOCK_PREDICTIVE = 5
} bsg_policy;

/* Probe-free closed loop (ExperimentSpec, config.h:58-70 subset) with the
 * autoscaler (ProvisionPolicy, autoscaler.h:10-27) and the dispatch-overhead
 * mode (overhead.dispatch_s, config.h:65: the decision is taken at the
 * arrival, the request lands at the chosen instance overhead seconds later,
 * driver.cpp:213-218). */
typedef struct bsg_replay_spec {
  int32_t n_instances;     /* cluster.instances */
  int32_t policy;          /* bsg_policy */
  int32_t objective;       /* 0 e2e, 1 ttft */
  int32_t capture;         /* nonzero: record every BlockPredictive what-if scenario */
  uint64_t policy_seed;    /* PolicyConfig::seed (Random's stream) */
  int32_t provision_kind;  /* 0 static, 1 preempt (predicted e2e), 2 relief (realized e2e) */
  int32_t max_instances;   /* provision.max_instances (>= n_instances) */
  double threshold_s;      /* provision.threshold_s (70) */
  double cold_start_s;     /* provision.cold_start_s (30) */
  double cooldown_s;       /* provision.cooldown_s (15) */
  double dispatch_overhead_s; /* overhead.dispatch_s (0: admit at the decision) */
} bsg_replay_spec;

/* RunLog totals (metrics.h:18-54 subset). */
typedef struct bsg_replay_summary {
  int64_t total_preemptions;
  int64_t end_ticks;              /* time of the last processed event */
  int32_t instances_provisioned;  /* Autoscaler::provisioned_total */
  int32_t final_instance_count;
} bsg_replay_summary;

/* Per-request outcome (Request, types.h:30-42). Unset times are -1. */
typedef struct bsg_request_outcome {
  int64_t arrival_ticks, dispatch_ticks, first_token_ticks, finish_ticks;
  int32_t instance;
  int32_t preempt_count;
} bsg_request_outcome;

/* Captured scenario set (opaque, owned by the library). */
typedef struct bsg_capture bsg_capture;

/* Runs the closed loop on host C++ live instances; every BlockPredictive
 * dispatch evaluates its per-instance what-ifs on the GPU (bsg_dispatch).
 * outcomes must hold min(count, request_cap) rows. *capture (optional)
 * receives the what-if scenarios in arrival order (n_instances per arrival). */
bsg_status bsg_replay(bsg_ctx* ctx, const bsg_workload* w, const bsg_instance_cfg* cfg,
                      const bsg_replay_spec* spec, bsg_request_outcome* outcomes,
                      bsg_replay_summary* summary, bsg_capture** capture);
void bsg_capture_sizes(const bsg_capture* c, int64_t* n_entries, int64_t* n_scenarios);
/* Copies the capture into caller buffers (entries columns of n_entries,
 * scenarios of n_scenarios); the `cfg` field of every scenario is 0. */
void bsg_capture_copy(const bsg_capture* c, uint64_t* id, int32_t* prompt, int32_t* est,
                      int32_t* prefill, int32_t* decoded, bsg_scenario* scenarios);
void bsg_capture_free(bsg_capture* c);

/* RunReport subset (metrics.h:80-108) of aggregate (metrics.cpp:21-124):
 * TTFT = first token - dispatch, e2e = finish - arrival over finished
 * requests; nearest-rank percentiles (metrics.cpp:11-19); throughput =
 * finished / (last finish - first arrival). */
typedef struct bsg_run_report {
  int32_t finished_requests, censored_requests;
  double throughput_rps;
  double mean_ttft_s, p50_ttft_s, p99_ttft_s;
  double mean_e2e_s, p50_e2e_s, p99_e2e_s;
  int64_t total_preemptions;
  int32_t instances_provisioned, final_instance_count;
  /* means over dispatch points of the per-dispatch mean / variance of the
   * instances' snapshot free blocks (driver.cpp:142-157, metrics.cpp:79-85);
   * produced by bsg_replay_device's device reports (bsg_aggregate, which has
   * no dispatch points, leaves them 0) */
  double free_blocks_mean_avg, free_blocks_var_avg;
  double mean_overhead_s;  /* mean of dispatch - arrival over finished requests */
} bsg_run_report;
bsg_status bsg_aggregate(const bsg_request_outcome* outcomes, int64_t n,
                         const bsg_replay_summary* summary, bsg_run_report* out);

/* capacity_search (metrics.cpp:139-178) over run_experiment cells built like
 * spec_for_cell (driver.cpp:321-331: policy seed = workload seed = estimator
 * seed = seed, qps swept): every integer qps in [qps_min, qps_max], then
 * tenths inside the bracket; pass iff p99 TTFT < slo. BSG_NO_CAPACITY when
 * qps_min already fails. tested_qps/tested_pass (capacity tested_cap) receive
 * the (qps, passed) sequence in test order. */
typedef struct bsg_capacity_result {
  double capacity_qps;
  int32_t bracket_pass, bracket_fail;
  int32_t monotone;
  int32_t n_tested;
} bsg_capacity_result;
bsg_status bsg_capacity_search(bsg_ctx* ctx, const bsg_workload* base, const bsg_instance_cfg* cfg,
                               const bsg_replay_spec* spec, uint64_t seed, int32_t qps_min,
                               int32_t qps_max, double slo_p99_ttft_s, bsg_capacity_result* out,
                               double* tested_qps, int32_t* tested_pass, int32_t tested_cap);

/* One capacity-sweep cell (BASELINE cfg5): a capacity_search over a closed
 * loop with `spec.n_instances` instances of profile `cfg`. */
typedef struct bsg_sweep_cell {
  bsg_workload workload;     /* base workload (request_cap bounds each run) */
  bsg_instance_cfg cfg;      /* latency profile + memory limits */
  bsg_replay_spec spec;      /* instances, policy, provisioning */
  uint64_t seed;             /* spec_for_cell seed */
  int32_t qps_min, qps_max;
  double slo_p99_ttft_s;
} bsg_sweep_cell;
typedef struct bsg_sweep_out {
  int32_t status;                /* BSG_OK or BSG_NO_CAPACITY or an error */
  int32_t reserved;
  bsg_capacity_result result;
  int64_t whatif_scenarios;      /* predict() scenarios simulated on the GPU for this cell */
  int64_t kernel_launches;
  double wall_s;                 /* host path: summed closed-loop time; device path: the
                                    wall time of the batched launches holding its points */
} bsg_sweep_out;
/* Runs the cells' capacity searches. When every cell is a cluster of <= 256
 * instances (max_instances when provisioning) with max_batch_size <= 256, every
 * (cell, qps) point is a device-resident closed loop (bsg_replay_device, any
 * policy): all integer points in one batched launch, then all tenths in a
 * second one (records generated on `threads` host threads). Otherwise the
 * closed loops run on `threads` host threads, each with its own context on
 * `device` (GPU what-ifs per arrival). BSG_SWEEP_HOST=1 forces the host path. */
bsg_status bsg_sweep_run(int device, const bsg_sweep_cell* cells, int32_t n_cells,
                         int32_t threads, bsg_sweep_out* out);

/* run_sweep (driver.cpp:333-390): one closed loop per (policy, qps, seed) cell,
 * policies outermost, seeds innermost (the reference's cell order), each
 * run_experiment(spec_for_cell(base, policy, qps, seed)) (driver.cpp:321-331)
 * aggregated (metrics.cpp:21-124) into a SweepCell row (driver.h:78-90).
 * A run that fails (e.g. a deadlock or a what-if error) gives ok = 0 and its
 * status instead of the reference's error text. All cells run as device-resident
 * closed loops in one batched launch when they fit (see bsg_sweep_run), else on
 * `threads` host threads. rows: n_policies * n_qps * n_seeds. */
typedef struct bsg_sweep_row {
  int32_t policy;            /* bsg_policy */
  int32_t ok;                /* 1: ran to completion */
  double qps;
  uint64_t seed;
  int32_t status;            /* BSG_OK, or why the run failed */
  int32_t finished_requests;
  double mean_ttft_s, p99_ttft_s, mean_e2e_s, p99_e2e_s;
  double throughput_rps;
  int64_t total_preemptions;
  double free_blocks_var_avg;
} bsg_sweep_row;
bsg_status bsg_run_sweep(int device, const bsg_workload* base, const bsg_instance_cfg* cfg,
                         const bsg_replay_spec* spec, const int32_t* policies, int32_t n_policies,
                         const double* qps_values, int32_t n_qps, const uint64_t* seeds, int32_t n_seeds,
                         int32_t threads, bsg_sweep_row* rows);

/* run_capacity (driver.cpp:392-427): capacity_search per policy of `policies`
 * (the baseline appended when absent), every run spec_for_cell(base, policy,
 * qps, seed); then the gain of every non-baseline policy over the baseline's
 * capacity, (c - c_base) / c_base, also formatted like format_percent ("16.7%",
 * driver.cpp:392-396). rows receive n_policies (+1) entries in that order;
 * *n_rows their count. Rows of policies with no capacity have status
 * BSG_NO_CAPACITY (the reference throws NoCapacityError out of run_capacity). */
typedef struct bsg_capacity_row {
  int32_t policy;
  int32_t status;             /* BSG_OK or BSG_NO_CAPACITY or an error */
  bsg_capacity_result result;
  int32_t has_gain;           /* non-baseline policy with a positive baseline capacity */
  int32_t reserved;
  double gain;                /* (capacity - baseline) / baseline */
  char gain_text[16];         /* format_percent: "%.1f%%" of gain * 100 */
} bsg_capacity_row;
bsg_status bsg_run_capacity(int device, const bsg_workload* base, const bsg_instance_cfg* cfg,
                            const bsg_replay_spec* spec, const int32_t* policies, int32_t n_policies,
                            int32_t baseline, uint64_t seed, int32_t qps_min, int32_t qps_max,
                            double slo_p99_ttft_s, int32_t threads, bsg_capacity_row* rows,
                            int32_t* n_rows, double* baseline_capacity);
/* Scenarios simulated by this context so far (all entry points). */
int64_t bsg_scenario_count(const bsg_ctx* ctx);

/* Device-resident closed loops: each run is one
 * run_experiment (driver.cpp:134-289) — any dispatch policy (BlockPredictive,
 * or the heuristics of pick_heuristic, scheduler.cpp:68-113), static / preempt
 * / relief provisioning (autoscaler.cpp:36-52), optional dispatch overhead
 * (driver.cpp:213-218) — executed entirely on the GPU, one thread block per
 * run: live instances in HBM, every arrival's per-instance what-ifs + argmin
 * (or heuristic scores) on the block's warps, the event loop on the device.
 * Requests of run r are rows [req_off, req_off + n_requests) of the request
 * columns (arrival ticks non-decreasing; request id = row - req_off);
 * outcomes has the same rows. run_status[r] is BSG_OK or the error that ended
 * run r (BSG_DEADLOCK / BSG_EMPTY_PLAN / a what-if failure). HOST buffers. */
typedef struct bsg_closed_loop_run {
  int32_t n_instances;  /* initial instances, 1..256 */
  int32_t objective;    /* 0 e2e, 1 ttft */
  int32_t cfg;          /* index into the configs set by bsg_set_configs */
  int32_t n_requests;
  int64_t req_off;
  /* ProvisionPolicy (autoscaler.h:10-27): 0 static, 1 preempt (predicted e2e at
   * dispatch), 2 relief (realized e2e at completion); max_instances <= 256 */
  int32_t provision_kind;
  int32_t max_instances;
  double threshold_s, cold_start_s, cooldown_s;
  int32_t policy;              /* bsg_policy */
  int32_t reserved;
  uint64_t policy_seed;        /* Random's SplitMix64 stream (PolicyConfig::seed) */
  double dispatch_overhead_s;  /* overhead.dispatch_s */
} bsg_closed_loop_run;
/* outcomes may be NULL (not copied back); reports (optional, one per run) is
 * aggregate (metrics.cpp:21-124) computed on the device:
 * nearest-rank percentiles by radix select over tick keys, means summed in
 * request order as the reference does, so every field is bit-identical. */
bsg_status bsg_replay_device(bsg_ctx* ctx, const bsg_closed_loop_run* runs, int32_t n_runs,
                             const int32_t* prompt, const int32_t* output, const int32_t* est,
                             const int64_t* arrival_ticks, int64_t n_requests_total,
                             bsg_request_outcome* outcomes, bsg_replay_summary* summaries,
                             int32_t* run_status, bsg_run_report* reports);

/* Fleet: a persistent device mirror of n_instances live serving instances
 * (incremental snapshot mirrors). Every instance's running
 * and waiting lists stay resident in HBM (K5's arena); bsg_fleet_dispatch is
 * one launch, one warp per instance: the warp advances its instance to
 * now_ticks (completions strictly before it, after closing the previous
 * dispatch instant — driver.cpp:233-289 semantics), runs predict() on the
 * updated state in place, and the last warp takes the BlockPredictive argmin
 * (scheduler.cpp:138-150) and admits the request; `output` is the request's
 * true length, which drives the simulated instance. lengths/n_samples: the
 * request's Monte-Carlo lengths (bsg_mc_lengths; score = sum of per-sample
 * e2e ticks) or NULL (score = the estimate's e2e / ttft ticks). Arrivals must
 * be non-decreasing in time. Driving a fleet with a workload's arrivals gives
 * exactly bsg_replay_device's outcomes. */
typedef struct bsg_fleet bsg_fleet;
bsg_status bsg_fleet_create(bsg_ctx* ctx, int32_t cfg, int32_t n_instances, int32_t max_requests,
                            bsg_fleet** out);
void bsg_fleet_destroy(bsg_fleet* f);
bsg_status bsg_fleet_dispatch(bsg_fleet* f, int64_t now_ticks, int32_t prompt, int32_t est,
                              int32_t output, const int32_t* lengths, int32_t n_samples,
                              int32_t objective, int32_t* chosen, int64_t* scores);
/* bsg_fleet_dispatch with the candidate's n_samples MC lengths drawn ON THE
 * DEVICE inside the call (K3; bsg_mc_lengths(est, request_id, n_samples, seed,
 * mean_abs_rel_error)): per call only the candidate's scalars go in. */
bsg_status bsg_fleet_dispatch_sampled(bsg_fleet* f, int64_t now_ticks, int32_t prompt, int32_t est,
                                      int32_t output, uint64_t request_id, int32_t n_samples,
                                      uint64_t seed, double mean_abs_rel_error, int32_t objective,
                                      int32_t* chosen, int64_t* scores);
/* The mirror's Status API (Instance::snapshot, backend.cpp:351-373) as of the
 * last dispatch: run_n running entries (admission order) then wait_n waiting
 * entries (head first) into the caller's columns (any may be NULL); when
 * run_n + wait_n > cap only the sizes are written. */
bsg_status bsg_fleet_snapshot(bsg_fleet* f, int32_t instance, int32_t* run_n, int32_t* wait_n,
                              int32_t* prompt, int32_t* est, int32_t* prefill, int32_t* decoded,
                              int32_t cap);
/* Runs every remaining step; copies the outcomes of the admitted requests (in
 * admission order) and the run summary. */
bsg_status bsg_fleet_finish(bsg_fleet* f, bsg_request_outcome* outcomes, int32_t* n_requests,
                            bsg_replay_summary* summary);

/* Wire schema (core/src/json_io.cpp, the codec only — the
 * HTTP roles are out of scope): n PredictionRequest JSON texts in, one GPU
 * batch, n responses out — PredictionResult JSON (as
 * prediction_result_to_json prints it) or the predictor role's error bodies
 * (service.cpp:229-241: "prediction-failure" for PredictionError, "bad-schema"
 * for malformed / invalid requests). status[i] is the request's bsg_status.
 * Responses are NUL-terminated at out + out_off[i]; out_off[n] = bytes needed
 * (BSG_INVALID_ARGUMENT when out_cap is smaller). Sets the context's configs
 * to the requests' distinct instance_configs. */
bsg_status bsg_predict_json(bsg_ctx* ctx, const char* const* requests, int32_t n, char* out,
                            int64_t out_cap, int64_t* out_off, int32_t* status);

/* The /predict role's request checks that precede simulation, on the host
 * (no device needed): parses `body` as prediction_request_from_json
 * (json_io.cpp:136-146) and validates its instance_config
 * (validate_instance_config, types.cpp:47-61). Returns BSG_OK when the request
 * would be simulated; otherwise its status and, in `out`, the exact error body
 * the reference role answers (json_io.cpp:148-152; service.cpp:229-241). */
int32_t bsg_wire_check(const char* body, char* out, int64_t cap);
/* A double as the reference's JSON layer prints it (nlohmann::json::dump:
 * Grisu2 digits, fixed notation for decimal exponents in (-4, 15]); returns the
 * length, or -(bytes needed) when cap is too small. No GPU needed. */
int32_t bsg_format_double(double v, char* out, int32_t cap);

/* ---- trace workloads (workload.cpp:51-170) -------------------------------- */

/* One TraceRecord (workload.h:15-21). estimated_output_tokens 0 = absent
 * (a present estimate is >= 1 after validation); has_arrival_offset 0/1. */
typedef struct bsg_trace_record {
  uint64_t id;
  int32_t prompt_tokens;
  int32_t output_tokens;
  int32_t estimated_output_tokens;
  int32_t has_arrival_offset;
  double arrival_offset_s;
} bsg_trace_record;

/* Why a trace was rejected: kind 0 none, 1 TraceParseError (line = 1-based
 * line number, error.h:64-69), 2 InvalidRecordError (field, error.h:72-76),
 * 3 ConfigError (field, e.g. "workload.qps"). message is the reference's
 * what() text where it is ours to write (NUL-terminated, truncated). */
typedef struct bsg_trace_error {
  int32_t kind;
  int32_t line;
  char field[40];
  char message[216];
} bsg_trace_error;

/* load_trace (workload.cpp:51-68): JSON Lines, one object per line with
 * id, prompt_tokens, output_tokens and optional estimated_output_tokens /
 * arrival_offset_s; blank lines skipped; the first bad line (malformed JSON,
 * missing/mistyped field, invalid value, duplicate id) rejects the trace with
 * BSG_BAD_INPUT and *err filled. *n_records = the number of records; when it
 * exceeds cap nothing past cap is written and BSG_INVALID_ARGUMENT is
 * returned (call again with cap >= *n_records). No GPU needed. */
bsg_status bsg_load_trace(const char* text, int64_t len, bsg_trace_record* out, int64_t cap,
                          int64_t* n_records, bsg_trace_error* err);

/* make_synthetic_trace (workload.cpp:172-191) as records: w->count rows,
 * id = row, no estimates or offsets (only the trace fields of w are read). */
bsg_status bsg_make_trace(const bsg_workload* w, bsg_trace_record* out);

/* write_trace (workload.cpp:78-89): the records as JSON Lines, byte-identical
 * to the reference's (nlohmann object key order, dump() number format).
 * *len = bytes needed; BSG_INVALID_ARGUMENT (nothing written) when > cap. */
bsg_status bsg_write_trace(const bsg_trace_record* recs, int64_t n, char* out, int64_t cap,
                           int64_t* len);

/* The request columns a run_experiment builds from trace records
 * (driver.cpp:137-160): request_cap truncation, generate_arrivals
 * (workload.cpp:141-170: every record's arrival_offset_s, in record order, or
 * Poisson at w->qps with w->arrival_seed when no record has one) and
 * estimate_length (workload.cpp:113-139) with w's estimator; estimator_kind 3
 * is EstimatorKind::kTrace (the records' own estimates). Only the estimator,
 * qps, arrival_seed and request_cap fields of w are read. Rows = *n_out
 * (<= n). Arrival ticks are non-decreasing unless the offsets are not. */
bsg_status bsg_trace_workload(const bsg_trace_record* recs, int64_t n, const bsg_workload* w,
                              int32_t* prompt, int32_t* output, int32_t* est,
                              int64_t* arrival_ticks, int64_t* n_out, bsg_trace_error* err);

/* bsg_replay over trace records instead of the synthetic trace (host event
 * loop; arrivals in any order, ties in record order). */
bsg_status bsg_replay_trace(bsg_ctx* ctx, const bsg_trace_record* recs, int64_t n,
                            const bsg_workload* w, const bsg_instance_cfg* cfg,
                            const bsg_replay_spec* spec, bsg_request_outcome* outcomes,
                            bsg_replay_summary* summary, bsg_trace_error* err);

/* Synthetic trace + estimates + Poisson arrival ticks (no GPU needed). */
bsg_status bsg_make_workload(const bsg_workload* w, int32_t* prompt, int32_t* output,
                             int32_t* est, int64_t* arrival_ticks);

#ifdef __cplusplus
}
#endif

#endif /* BLOCKSIM_B200_H */

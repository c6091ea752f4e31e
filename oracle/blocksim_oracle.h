/*
 * oracle/blocksim_oracle.h — TEST INFRASTRUCTURE ONLY (see blocksim_oracle.c).
 *
 * Two checkers share this header:
 *   oracle_*  — the plain-C restatement (oracle/blocksim_oracle.c), built into
 *               oracle/build/liboracle.so;
 *   ref_*     — a thin shim (oracle/ref_shim.cpp) over the reference itself,
 *               compiled from /root/reference/proj/core/src by oracle/Makefile
 *               with -Dblocksim=blocksim_ref into oracle/_ref/libblocksim_ref.so.
 * Data layouts are the product's C-ABI structs (include/blocksim_b200.h) so
 * checkers and product consume identical buffers.
 */
#ifndef BLOCKSIM_ORACLE_H
#define BLOCKSIM_ORACLE_H

#include "../include/blocksim_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_MAX_STEPS 50000000LL /* kMaxSimulatedSteps, predictor.cpp:11 */

/* ---- C restatement ------------------------------------------------------ */
int32_t oracle_validate_config(const bsg_instance_cfg* c);
int32_t oracle_predict(const bsg_instance_cfg* cfg, const bsg_entries* e, const bsg_scenario* sc,
                       bsg_result* out, bsg_step_record* trace, int64_t trace_cap,
                       int64_t* n_steps);
void oracle_predict_batch(const bsg_instance_cfg* cfgs, const bsg_entries* e,
                          const bsg_scenario* sc, int64_t n, bsg_result* out);
double oracle_ticks_to_seconds(int64_t ticks);
int64_t oracle_llround_1e9(double s);
int64_t oracle_blocks_needed(int64_t tokens, int32_t block_size);
double oracle_batch_latency(const bsg_instance_cfg* c, int64_t prefill_tokens, int64_t n_decode,
                            int64_t context);

/* ---- reference shim ----------------------------------------------------- */
/* PredictionResult as the reference reports it (seconds as doubles). */
typedef struct ref_result {
  double e2e_s, ttft_s, qdelay_s;
  int64_t steps;
  int32_t status; /* bsg_status mapped from the thrown exception type/message */
  int32_t detail;
} ref_result;

/* blocksim_ref::predict(req, cache) per scenario; cache per cfg.cache_mode
 * (nullptr for off, a per-thread LatencyCache otherwise). threads <= 1 runs
 * inline. Returns 0. */
int ref_predict_batch(const bsg_instance_cfg* cfgs, const bsg_entries* e, const bsg_scenario* sc,
                      int64_t n, ref_result* out, int threads);
/* Wall seconds (steady_clock, best of `reps`) to run predict over all n
 * scenarios on `threads` std::threads with dynamic 64-scenario chunks. */
double ref_time_predict(const bsg_instance_cfg* cfgs, const bsg_entries* e,
                        const bsg_scenario* sc, int64_t n, int threads, int reps);
/* Per-step trace through the reference's public Instance::execute_step. */
int ref_trace(const bsg_instance_cfg* cfg, const bsg_entries* e, const bsg_scenario* sc,
              bsg_step_record* rec, int64_t cap, int64_t* n_steps, ref_result* out);
/* estimate_length(Noisy{err, seed}) of a record {id, output_tokens} (workload.cpp:126-136). */
int32_t ref_estimate_noisy(int32_t output_tokens, uint64_t record_id, uint64_t seed,
                           double mean_abs_rel_error);
/* Reference workload generators. */
int ref_make_workload(const bsg_workload* w, int32_t* prompt, int32_t* output, int32_t* est,
                      int64_t* arrival_ticks);
/* blocksim_ref::run_experiment (driver.cpp:316-319), static provisioning. */
int ref_run_experiment(const bsg_workload* w, const bsg_instance_cfg* cfg,
                       const bsg_replay_spec* spec, bsg_request_outcome* out,
                       bsg_replay_summary* summary);
/* aggregate (metrics.cpp:21-124) of run_experiment. */
int ref_run_report(const bsg_workload* w, const bsg_instance_cfg* c, const bsg_replay_spec* s,
                   bsg_run_report* out);
/* capacity_search (metrics.cpp:139-178) with run_capacity's runner (driver.cpp:398-418). */
int ref_capacity_search(const bsg_workload* w, const bsg_instance_cfg* c, const bsg_replay_spec* s,
                        uint64_t seed, int32_t qps_min, int32_t qps_max, double slo,
                        bsg_capacity_result* out, double* tested_qps, int32_t* tested_pass,
                        int32_t tested_cap);
/* Hand replay of SimulationDriver (driver.cpp:134-289) over the reference's
 * public EventLoop / Instance / Dispatcher with a capturing PredictorClient;
 * returns an opaque capture (ref_capture_*). */
typedef struct ref_capture ref_capture;
int ref_replay(const bsg_workload* w, const bsg_instance_cfg* cfg, const bsg_replay_spec* spec,
               bsg_request_outcome* out, bsg_replay_summary* summary, ref_capture** capture);
void ref_capture_sizes(const ref_capture* c, int64_t* n_entries, int64_t* n_scenarios);
void ref_capture_copy(const ref_capture* c, uint64_t* id, int32_t* prompt, int32_t* est,
                      int32_t* prefill, int32_t* decoded, bsg_scenario* scenarios);
void ref_capture_free(ref_capture* c);

#ifdef __cplusplus
}
#endif

#endif /* BLOCKSIM_ORACLE_H */

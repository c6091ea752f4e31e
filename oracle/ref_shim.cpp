// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the REFERENCE implementation itself. It is
// compiled together with the reference's own, unmodified translation units
// (/root/reference/proj/core/src/*.cpp, see oracle/Makefile) with
// -Dblocksim=blocksim_ref, producing oracle/_ref/libblocksim_ref.so. No
// reference source is copied into this repository: this file only calls the
// reference's public API (predictor.h, backend.h, scheduler.h, workload.h,
// driver.h, event_loop.h) and converts between its types and the C-ABI
// buffers of include/blocksim_b200.h.
//
// Users: tests/ (parity checker), bench.py --impl reference and the
// cpu_baseline leg (CPU timing of the reference predict()).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <sstream>
#include <cstdio>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "blocksim/backend.h"
#include "blocksim/driver.h"
#include "blocksim/error.h"
#include "blocksim/event_loop.h"
#include "blocksim/json_io.h"
#include <nlohmann/json.hpp>
#include "blocksim/metrics.h"
#include "blocksim/predictor.h"
#include "blocksim/scheduler.h"
#include "blocksim/workload.h"

#include "blocksim_oracle.h"

namespace {

using namespace blocksim;  // == blocksim_ref under -Dblocksim=blocksim_ref

InstanceConfig to_ref_config(const bsg_instance_cfg& c, InstanceId id = 0) {
  InstanceConfig cfg;
  cfg.instance_id = id;
  cfg.total_blocks = c.total_blocks;
  cfg.block_size = c.block_size;
  cfg.max_batch_size = c.max_batch_size;
  cfg.chunk_budget = c.chunk_budget;
  cfg.local_policy =
      c.local_policy == BSG_PREFILL_PRIORITY ? LocalPolicy::kPrefillPriority : LocalPolicy::kChunkedPrefill;
  cfg.cost_model.c0_s = c.c0_s;
  cfg.cost_model.prefill_s_per_token = c.prefill_s_per_token;
  cfg.cost_model.decode_s_per_seq = c.decode_s_per_seq;
  cfg.cost_model.context_s_per_token = c.context_s_per_token;
  return cfg;
}

CacheMode to_ref_cache(int32_t m) {
  return m == BSG_CACHE_BUCKETED ? CacheMode::kBucketed
                                 : (m == BSG_CACHE_EXACT ? CacheMode::kExact : CacheMode::kOff);
}

// Snapshot with synthetic unique ids: running i -> i+1, waiting j -> run_n+j+1.
InstanceSnapshot make_snapshot(const bsg_entries* e, const bsg_scenario& sc) {
  InstanceSnapshot snap;
  snap.running.reserve(sc.run_n);
  for (int32_t i = 0; i < sc.run_n; ++i) {
    const int32_t k = sc.run_off + i;
    snap.running.push_back({static_cast<RequestId>(i + 1), e->prompt[k], e->est[k], e->prefill[k],
                            e->decoded[k]});
  }
  snap.waiting.reserve(sc.wait_n);
  for (int32_t j = 0; j < sc.wait_n; ++j) {
    const int32_t k = sc.wait_off + j;
    snap.waiting.push_back({static_cast<RequestId>(sc.run_n + j + 1), e->prompt[k], e->est[k],
                            e->prefill[k], e->decoded[k]});
  }
  return snap;
}

int32_t config_field_code(const std::string& field) {
  static const std::map<std::string, int32_t> codes = {
      {"total_blocks", 1},         {"block_size", 2},
      {"max_batch_size", 3},       {"chunk_budget", 4},
      {"cost_model.c0_s", 5},      {"cost_model.prefill_s_per_token", 6},
      {"cost_model.decode_s_per_seq", 7}, {"cost_model.context_s_per_token", 8}};
  auto it = codes.find(field);
  return it == codes.end() ? -1 : it->second;
}

bool starts_with(const std::string& s, const char* p) { return s.rfind(p, 0) == 0; }

// Maps the reference's exception taxonomy onto bsg_status (error.h:31-56,
// predictor.cpp:101-136).
void classify(const std::exception& ex, const bsg_scenario& sc, ref_result* out) {
  const std::string msg = ex.what();
  out->detail = 0;
  if (dynamic_cast<const PredictionError*>(&ex)) {
    if (starts_with(msg, "backend deadlock")) {
      out->status = BSG_DEADLOCK;
      // "…: request <id> cannot proceed with the whole memory free"
      const auto p = msg.find("request ");
      const unsigned long long id = std::stoull(msg.substr(p + 8));
      const unsigned long long cand = static_cast<unsigned long long>(sc.run_n + sc.wait_n + 1);
      out->detail = id == cand ? -1 : static_cast<int32_t>(id - 1);
    } else if (starts_with(msg, "candidate does not fit the instance: snapshot running")) {
      out->status = BSG_TOO_LARGE_RUNNING;
    } else if (starts_with(msg, "candidate does not fit the instance: request")) {
      out->status = BSG_TOO_LARGE_CANDIDATE;
      const auto p = msg.find(" needs ");
      out->detail = static_cast<int32_t>(std::stoll(msg.substr(p + 7)));
    } else if (starts_with(msg, "forward simulation exceeded")) {
      out->status = BSG_STEP_LIMIT;
    } else if (starts_with(msg, "candidate vanished")) {
      out->status = BSG_VANISHED;
    } else {
      out->status = BSG_INVALID_ARGUMENT;
    }
  } else if (dynamic_cast<const EmptyPlanError*>(&ex)) {
    out->status = BSG_EMPTY_PLAN;
  } else if (auto* ce = dynamic_cast<const ConfigError*>(&ex)) {
    out->status = BSG_BAD_CONFIG;
    out->detail = config_field_code(ce->field);
  } else {
    out->status = BSG_INVALID_ARGUMENT;
  }
}

void run_one(const bsg_instance_cfg* cfgs, const bsg_entries* e, const bsg_scenario& sc,
             LatencyCache* exact, LatencyCache* bucketed, ref_result* out) {
  std::memset(out, 0, sizeof(*out));
  const bsg_instance_cfg& c = cfgs[sc.cfg];
  PredictionRequest req;
  req.snapshot = make_snapshot(e, sc);
  req.candidate = {sc.cand_prompt, sc.cand_est};
  req.instance_config = to_ref_config(c);
  LatencyCache* cache = c.cache_mode == BSG_CACHE_EXACT
                            ? exact
                            : (c.cache_mode == BSG_CACHE_BUCKETED ? bucketed : nullptr);
  try {
    const PredictionResult r = predict(req, cache);
    out->e2e_s = r.e2e();
    out->ttft_s = r.ttft();
    out->qdelay_s = r.metrics.at("predicted_queueing_delay");
    out->steps = r.simulated_steps;
    out->status = BSG_OK;
  } catch (const std::exception& ex) {
    classify(ex, sc, out);
  }
}

template <typename F>
void parallel_chunks(int64_t n, int threads, F&& body) {
  if (threads <= 1) {
    body(0, 0, n);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (;;) {
        const int64_t b = next.fetch_add(64);
        if (b >= n) break;
        body(t, b, std::min<int64_t>(n, b + 64));
      }
    });
  }
  for (auto& th : pool) th.join();
}

// Records installed by ref_set_trace replace the synthetic trace (tests only).
std::vector<TraceRecord>* g_trace = nullptr;

std::vector<TraceRecord> make_records(const bsg_workload* w) {
  if (g_trace) {  // request_cap as the driver applies it (driver.cpp:140-144)
    std::vector<TraceRecord> records = *g_trace;
    if (w->request_cap >= 0 && static_cast<std::size_t>(w->request_cap) < records.size())
      records.resize(static_cast<std::size_t>(w->request_cap));
    return records;
  }
  SyntheticTraceSpec t;
  t.count = w->count;
  t.seed = w->trace_seed;
  t.prompt_median = w->prompt_median;
  t.prompt_sigma = w->prompt_sigma;
  t.output_median = w->output_median;
  t.output_sigma = w->output_sigma;
  t.min_tokens = w->min_tokens;
  t.max_prompt_tokens = w->max_prompt_tokens;
  t.max_output_tokens = w->max_output_tokens;
  std::vector<TraceRecord> records = make_synthetic_trace(t);
  if (w->request_cap >= 0 && static_cast<std::size_t>(w->request_cap) < records.size()) {
    records.resize(static_cast<std::size_t>(w->request_cap));
  }
  return records;
}

LengthEstimator make_estimator(const bsg_workload* w) {
  LengthEstimator est;
  est.kind = w->estimator_kind == 1   ? EstimatorKind::kFixed
             : w->estimator_kind == 2 ? EstimatorKind::kNoisy
             : w->estimator_kind == 3 ? EstimatorKind::kTrace
                                      : EstimatorKind::kOracle;
  est.fixed_tokens = w->fixed_tokens;
  est.mean_abs_rel_error = w->mean_abs_rel_error;
  est.seed = w->estimator_seed;
  return est;
}

PolicyKind to_ref_policy(int32_t p) {
  switch (p) {
    case BSG_POLICY_RANDOM: return PolicyKind::kRandom;
    case BSG_POLICY_ROUND_ROBIN: return PolicyKind::kRoundRobin;
    case BSG_POLICY_MIN_QPM: return PolicyKind::kMinQpm;
    case BSG_POLICY_INFAAS_PP: return PolicyKind::kInfaasPlusPlus;
    case BSG_POLICY_LLUMNIX_MINUS: return PolicyKind::kLlumnixMinus;
    default: return PolicyKind::kBlockPredictive;
  }
}

void fill_outcome(const Request& r, InstanceId inst, int preempts, bsg_request_outcome* o) {
  o->arrival_ticks = r.arrival_time.ticks();
  o->dispatch_ticks = r.dispatch_time ? r.dispatch_time->ticks() : -1;
  o->first_token_ticks = r.first_token_time ? r.first_token_time->ticks() : -1;
  o->finish_ticks = r.finish_time ? r.finish_time->ticks() : -1;
  o->instance = inst;
  o->preempt_count = preempts;
}

}  // namespace

struct ref_capture {
  std::vector<uint64_t> id;
  std::vector<int32_t> prompt, est, prefill, decoded;
  std::vector<bsg_scenario> scenarios;
};

namespace {

// Records every snapshot + candidate handed to the predictor, then answers
// exactly like LocalPredictorClient (scheduler.h:63-75).
class CapturingClient : public PredictorClient {
 public:
  CapturingClient(InstanceConfig tmpl, LatencyCache* cache, ref_capture* cap)
      : template_(std::move(tmpl)), cache_(cache), cap_(cap) {}
  std::map<InstanceId, PredictionResult> predict_across(
      const std::vector<InstanceSnapshot>& snapshots, const CandidateRequest& candidate) override {
    if (cap_) {
      for (const InstanceSnapshot& s : snapshots) {
        bsg_scenario sc{};
        sc.run_off = static_cast<int32_t>(cap_->prompt.size());
        sc.run_n = static_cast<int32_t>(s.running.size());
        for (const auto& r : s.running) push(r);
        sc.wait_off = static_cast<int32_t>(cap_->prompt.size());
        sc.wait_n = static_cast<int32_t>(s.waiting.size());
        for (const auto& r : s.waiting) push(r);
        sc.cand_prompt = candidate.prompt_tokens;
        sc.cand_est = candidate.estimated_output_tokens;
        sc.cfg = 0;
        cap_->scenarios.push_back(sc);
      }
    }
    return blocksim::predict_across(snapshots, candidate, template_, cache_);
  }

 private:
  void push(const SnapshotRequest& r) {
    cap_->id.push_back(r.id);
    cap_->prompt.push_back(r.prompt_tokens);
    cap_->est.push_back(r.estimated_output_tokens);
    cap_->prefill.push_back(r.prefill_progress);
    cap_->decoded.push_back(r.decoded_tokens);
  }
  InstanceConfig template_;
  LatencyCache* cache_;
  ref_capture* cap_;
};

// Hand replay of SimulationDriver for static provisioning, zero dispatch
// overhead and no probes: handle_arrival (driver.cpp:134-219),
// admit_to_instance (225-231), handle_batch_complete (233-251),
// end_of_instant (271-289).
class Replay : public EventHandler {
 public:
  Replay(const bsg_workload* w, const bsg_instance_cfg* c, const bsg_replay_spec* s,
         ref_capture* cap)
      : tmpl_(to_ref_config(*c)),
        dispatcher_(PolicyConfig{to_ref_policy(s->policy), s->policy_seed,
                                 s->objective == 1 ? LatencyObjective::kTtft : LatencyObjective::kE2e},
                    tmpl_),
        cache_(to_ref_cache(c->cache_mode) == CacheMode::kOff
                   ? nullptr
                   : std::make_unique<LatencyCache>(to_ref_cache(c->cache_mode), c->context_bucket)),
        client_(tmpl_, cache_.get(), cap) {
    const std::vector<TraceRecord> records = make_records(w);
    const std::vector<Arrival> arrivals = generate_arrivals(records, w->qps, w->arrival_seed);
    const LengthEstimator est = make_estimator(w);
    for (std::size_t i = 0; i < arrivals.size(); ++i) {
      Request r;
      r.id = static_cast<RequestId>(i);
      r.prompt_tokens = arrivals[i].record.prompt_tokens;
      r.true_output_tokens = arrivals[i].record.output_tokens;
      r.estimated_output_tokens = estimate_length(est, arrivals[i].record);
      r.arrival_time = arrivals[i].time;
      requests_.push_back(r);
      engine_.push(EventKind::kArrival, arrivals[i].time, r.id);
    }
    preempts_.assign(requests_.size(), 0);
    dispatched_.assign(requests_.size(), -1);
    for (int i = 0; i < s->n_instances; ++i) {
      InstanceConfig ic = tmpl_;
      ic.instance_id = i;
      instances_.emplace_back(ic);
    }
  }

  void handle(const Event& ev) override {
    if (ev.kind == EventKind::kArrival) {
      arrival(static_cast<RequestId>(ev.a));
    } else if (ev.kind == EventKind::kBatchComplete) {
      complete(static_cast<InstanceId>(ev.a));
    }
  }

  void end_of_instant(SimTime now) override {
    for (Instance& inst : instances_) {
      if (inst.mid_step() || !inst.has_work()) continue;
      const StepBegin begin = inst.begin_step();
      engine_.push(EventKind::kBatchComplete, now + begin.duration,
                   static_cast<std::uint64_t>(inst.config().instance_id));
      for (const RequestId id : begin.preempted) {
        preempts_[id] += 1;
        cum_preemptions_ += 1;
      }
    }
  }

  void run() { engine_.run_until(std::nullopt, *this); }

  void outcomes(bsg_request_outcome* out) const {
    for (std::size_t i = 0; i < requests_.size(); ++i)
      fill_outcome(requests_[i], dispatched_[i], preempts_[i], &out[i]);
  }
  int64_t total_preemptions() const { return cum_preemptions_; }

 private:
  void arrival(RequestId rid) {
    const SimTime now = engine_.now();
    Request& r = requests_[rid];
    std::vector<InstanceSnapshot> snaps;
    for (const Instance& inst : instances_)
      snaps.push_back(inst.snapshot(now, qpm_.qpm(inst.config().instance_id, now)));
    const CandidateRequest cand{r.prompt_tokens, r.estimated_output_tokens};
    const DispatchDecision d = dispatcher_.dispatch(cand, snaps, &client_);
    qpm_.record_dispatch(d.instance_id, now);
    instances_[static_cast<std::size_t>(d.instance_id)].admit(rid, r.prompt_tokens,
                                                              r.true_output_tokens,
                                                              r.estimated_output_tokens);
    r.dispatch_time = now;
    dispatched_[rid] = d.instance_id;
  }

  void complete(InstanceId iid) {
    const SimTime now = engine_.now();
    const StepFinish fin = instances_[static_cast<std::size_t>(iid)].finish_step();
    for (const RequestId id : fin.first_tokens) {
      if (!requests_[id].first_token_time) requests_[id].first_token_time = now;
    }
    for (const RequestId id : fin.completed) {
      requests_[id].finish_time = now;
      requests_[id].state = RequestState::kFinished;
    }
  }

  InstanceConfig tmpl_;
  Dispatcher dispatcher_;
  std::unique_ptr<LatencyCache> cache_;
  CapturingClient client_;
  EventLoop engine_;
  std::vector<Instance> instances_;
  std::vector<Request> requests_;
  std::vector<int> preempts_;
  std::vector<InstanceId> dispatched_;
  QpmTracker qpm_;
  int64_t cum_preemptions_ = 0;
};

}  // namespace

extern "C" {

int ref_predict_batch(const bsg_instance_cfg* cfgs, const bsg_entries* e, const bsg_scenario* sc,
                      int64_t n, ref_result* out, int threads) {
  // One LatencyCache per (thread, config): the cache key (predictor.h:60-65)
  // does not include the cost model or bucket, so a cache must never be
  // shared across configs (the reference shares one per SimulationDriver,
  // i.e. per config).
  const int nt = std::max(1, threads);
  int32_t ncfg = 0;
  for (int64_t i = 0; i < n; ++i) ncfg = std::max(ncfg, sc[i].cfg + 1);
  std::vector<std::vector<std::unique_ptr<LatencyCache>>> caches(nt);
  for (auto& v : caches) v.resize(static_cast<size_t>(ncfg));
  parallel_chunks(n, nt, [&](int t, int64_t b, int64_t end) {
    for (int64_t i = b; i < end; ++i) {
      const int32_t ci = sc[i].cfg;
      const bsg_instance_cfg& c = cfgs[ci];
      auto& slot = caches[t][static_cast<size_t>(ci)];
      if (c.cache_mode != BSG_CACHE_OFF && !slot)
        slot = std::make_unique<LatencyCache>(to_ref_cache(c.cache_mode), c.context_bucket);
      run_one(cfgs, e, sc[i], slot.get(), slot.get(), &out[i]);
    }
  });
  return 0;
}

double ref_time_predict(const bsg_instance_cfg* cfgs, const bsg_entries* e,
                        const bsg_scenario* sc, int64_t n, int threads, int reps) {
  std::vector<ref_result> out(static_cast<std::size_t>(n));
  double best = std::numeric_limits<double>::infinity();
  for (int r = 0; r < std::max(1, reps); ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    ref_predict_batch(cfgs, e, sc, n, out.data(), threads);
    const double dt =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    best = std::min(best, dt);
  }
  return best;
}

int ref_trace(const bsg_instance_cfg* cfg, const bsg_entries* e, const bsg_scenario* sc,
              bsg_step_record* rec, int64_t cap, int64_t* n_steps, ref_result* out) {
  std::memset(out, 0, sizeof(*out));
  *n_steps = 0;
  const InstanceSnapshot snap = make_snapshot(e, *sc);
  const RequestId cand_id = static_cast<RequestId>(sc->run_n + sc->wait_n + 1);
  auto origin = [&](RequestId id) -> int32_t {
    return id == cand_id ? -1 : static_cast<int32_t>(id - 1);
  };
  LatencyCache cache(to_ref_cache(cfg->cache_mode), cfg->context_bucket);
  const CostModelParams params = to_ref_config(*cfg).cost_model;
  int64_t steps = 0;  // steps executed before any exception (trace length)
  try {
    // Mirrors predict() (predictor.cpp:76-137) through the public Instance API.
    const InstanceSnapshot corrected = correct_lengths(snap);
    Instance inst = Instance::from_snapshot(corrected, to_ref_config(*cfg));
    inst.admit(cand_id, sc->cand_prompt, sc->cand_est, sc->cand_est);
    Instance::LatencyFn fn = cfg->cache_mode == BSG_CACHE_OFF
                                 ? Instance::LatencyFn([&](const BatchPlan& p) {
                                     return batch_latency(p, params);
                                   })
                                 : Instance::LatencyFn([&](const BatchPlan& p) {
                                     return cache.lookup_or_compute(p, params);
                                   });
    SimTime elapsed = SimTime::zero();
    bool qd = false, tt = false;
    for (;;) {
      if (!inst.has_work()) throw PredictionError("candidate vanished from the forward simulation");
      const SimTime start = elapsed;
      const StepResult st = inst.execute_step(fn);
      elapsed += st.duration;
      ++steps;
      if (steps <= cap) {
        bsg_step_record& r = rec[steps - 1];
        std::memset(&r, 0, sizeof(r));
        r.duration_ticks = st.duration.ticks();
        r.context_tokens = st.plan.context_tokens;
        r.n_decode = static_cast<int32_t>(st.plan.decode_ids.size());
        r.prefill_tokens = static_cast<int32_t>(st.plan.total_prefill_tokens);
        r.n_prefill = static_cast<int32_t>(st.plan.prefill_segments.size());
        r.n_preempted = static_cast<int32_t>(st.preempted.size());
        r.n_completed = static_cast<int32_t>(st.completed.size());
        r.free_blocks_after = inst.free_blocks();
        uint32_t k = 0;
        for (const RequestId id : st.plan.decode_ids)
          r.plan_hash += bsg_hash_term(BSG_TAG_PLAN, k++, origin(id), 0);
        k = 0;
        for (const auto& [id, chunk] : st.plan.prefill_segments)
          r.plan_hash += bsg_hash_term(BSG_TAG_PLAN + 16u, k++, origin(id), chunk);
        k = 0;
        for (const RequestId id : st.preempted)
          r.event_hash += bsg_hash_term(BSG_TAG_PREEMPT, k++, origin(id), 0);
        k = 0;
        for (const RequestId id : st.started)
          r.event_hash += bsg_hash_term(BSG_TAG_STARTED, k++, origin(id), 0);
        k = 0;
        for (const RequestId id : st.first_tokens)
          r.event_hash += bsg_hash_term(BSG_TAG_FIRST, k++, origin(id), 0);
        k = 0;
        for (const RequestId id : st.completed)
          r.event_hash += bsg_hash_term(BSG_TAG_COMPLETED, k++, origin(id), 0);
      }
      auto has = [&](const std::vector<RequestId>& v) {
        return std::find(v.begin(), v.end(), cand_id) != v.end();
      };
      if (!qd && has(st.started)) {
        out->qdelay_s = start.seconds();
        qd = true;
      }
      if (!tt && has(st.first_tokens)) {
        out->ttft_s = elapsed.seconds();
        tt = true;
      }
      if (has(st.completed)) {
        out->e2e_s = elapsed.seconds();
        if (!tt) out->ttft_s = out->e2e_s;
        break;
      }
      if (steps > ORACLE_MAX_STEPS) throw PredictionError("forward simulation exceeded the step limit");
    }
    out->steps = steps;
    *n_steps = steps;
    out->status = BSG_OK;
  } catch (const DeadlockError& ex) {
    PredictionError wrapped(std::string("backend deadlock during forward simulation: ") + ex.what());
    classify(wrapped, *sc, out);
    *n_steps = steps;
  } catch (const RequestTooLargeError& ex) {
    PredictionError wrapped(std::string("candidate does not fit the instance: ") + ex.what());
    classify(wrapped, *sc, out);
    *n_steps = steps;
  } catch (const std::exception& ex) {
    classify(ex, *sc, out);
    *n_steps = steps;
  }
  return 0;
}

int32_t ref_estimate_noisy(int32_t output_tokens, uint64_t record_id, uint64_t seed,
                           double mean_abs_rel_error) {
  LengthEstimator e;
  e.kind = EstimatorKind::kNoisy;
  e.seed = seed;
  e.mean_abs_rel_error = mean_abs_rel_error;
  TraceRecord r;
  r.id = record_id;
  r.output_tokens = output_tokens;
  return estimate_length(e, r);
}

int ref_make_workload(const bsg_workload* w, int32_t* prompt, int32_t* output, int32_t* est,
                      int64_t* arrival_ticks) {
  try {
    const std::vector<TraceRecord> records = make_records(w);
    const std::vector<Arrival> arrivals = generate_arrivals(records, w->qps, w->arrival_seed);
    const LengthEstimator e = make_estimator(w);
    for (std::size_t i = 0; i < arrivals.size(); ++i) {
      prompt[i] = arrivals[i].record.prompt_tokens;
      output[i] = arrivals[i].record.output_tokens;
      est[i] = estimate_length(e, arrivals[i].record);
      arrival_ticks[i] = arrivals[i].time.ticks();
    }
    return static_cast<int>(arrivals.size());
  } catch (const std::exception&) {
    return -1;
  }
}

static ExperimentSpec make_experiment(const bsg_workload* w, const bsg_instance_cfg* c,
                                     const bsg_replay_spec* s) {
  ExperimentSpec spec;
  spec.initial_instances = s->n_instances;
  spec.instance_template = to_ref_config(*c);
  spec.policy.kind = to_ref_policy(s->policy);
  spec.policy.seed = s->policy_seed;
  spec.policy.objective = s->objective == 1 ? LatencyObjective::kTtft : LatencyObjective::kE2e;
  spec.workload.records = make_records(w);
  spec.workload.qps = w->qps;
  spec.workload.seed = w->arrival_seed;
  spec.workload.estimator = make_estimator(w);
  spec.provision.kind = s->provision_kind == 1 ? ProvisionKind::kPreempt
                        : (s->provision_kind == 2 ? ProvisionKind::kRelief : ProvisionKind::kStatic);
  spec.provision.min_instances = s->n_instances;
  spec.provision.max_instances = std::max(s->n_instances, s->max_instances);
  spec.provision.threshold_s = s->threshold_s;
  spec.provision.cold_start_s = s->cold_start_s;
  spec.provision.cooldown_s = s->cooldown_s;
  spec.cache_mode = to_ref_cache(c->cache_mode);
  spec.cache_bucket = c->context_bucket;
  spec.dispatch_overhead_s = s->dispatch_overhead_s;
  spec.collect_events = false;
  return spec;
}

int ref_run_experiment(const bsg_workload* w, const bsg_instance_cfg* c,
                       const bsg_replay_spec* s, bsg_request_outcome* out,
                       bsg_replay_summary* summary) {
  RunLog log;
  try {
    log = run_experiment(make_experiment(w, c, s));
  } catch (const std::exception&) {
    return -1;
  }
  std::vector<InstanceId> inst(log.requests.size(), -1);
  for (const auto& p : log.dispatch_points) inst[p.request_id] = p.instance_id;
  for (std::size_t i = 0; i < log.requests.size(); ++i)
    fill_outcome(log.requests[i], inst[i], log.preempt_counts[i], &out[i]);
  if (summary) {
    summary->total_preemptions = log.total_preemptions;
    summary->end_ticks = log.end_time.ticks();
    summary->instances_provisioned = log.instances_provisioned;
    summary->final_instance_count = log.final_instance_count;
  }
  return static_cast<int>(log.requests.size());
}

// aggregate (metrics.cpp:21-124) of a reference run.
int ref_run_report(const bsg_workload* w, const bsg_instance_cfg* c, const bsg_replay_spec* s,
                   bsg_run_report* out) {
  const RunLog log = run_experiment(make_experiment(w, c, s));
  const RunReport r = aggregate(log);
  std::memset(out, 0, sizeof(*out));
  out->finished_requests = r.finished_requests;
  out->censored_requests = r.censored_requests;
  out->throughput_rps = r.throughput_rps;
  out->mean_ttft_s = r.mean_ttft_s;
  out->p50_ttft_s = r.p50_ttft_s;
  out->p99_ttft_s = r.p99_ttft_s;
  out->mean_e2e_s = r.mean_e2e_s;
  out->p50_e2e_s = r.p50_e2e_s;
  out->p99_e2e_s = r.p99_e2e_s;
  out->total_preemptions = r.total_preemptions;
  out->instances_provisioned = r.instances_provisioned;
  out->final_instance_count = r.final_instance_count;
  out->free_blocks_mean_avg = r.free_blocks_mean_avg;
  out->free_blocks_var_avg = r.free_blocks_var_avg;
  out->mean_overhead_s = r.mean_overhead_s;
  return 0;
}

// capacity_search (metrics.cpp:139-178) over run_experiment(spec_for_cell(...))
// exactly as run_capacity builds its runner (driver.cpp:398-418). Returns 0,
// or 12 (BSG_NO_CAPACITY) on NoCapacityError.
int ref_capacity_search(const bsg_workload* w, const bsg_instance_cfg* c, const bsg_replay_spec* s,
                        uint64_t seed, int32_t qps_min, int32_t qps_max, double slo,
                        bsg_capacity_result* out, double* tested_qps, int32_t* tested_pass,
                        int32_t tested_cap) {
  const ExperimentSpec base = make_experiment(w, c, s);
  const PolicyKind policy = base.policy.kind;
  auto runner = [&](double qps) {
    ExperimentSpec spec = spec_for_cell(base, policy, qps, seed);
    spec.collect_events = false;
    return aggregate(run_experiment(spec));
  };
  std::memset(out, 0, sizeof(*out));
  try {
    const CapacityResult r = capacity_search(runner, SloSpec{slo}, qps_min, qps_max);
    out->capacity_qps = r.capacity_qps;
    out->bracket_pass = r.bracket_pass;
    out->bracket_fail = r.bracket_fail;
    out->monotone = r.monotone ? 1 : 0;
    out->n_tested = static_cast<int32_t>(r.tested.size());
    for (std::size_t i = 0; i < r.tested.size() && static_cast<int32_t>(i) < tested_cap; ++i) {
      tested_qps[i] = r.tested[i].first;
      tested_pass[i] = r.tested[i].second ? 1 : 0;
    }
    return 0;
  } catch (const NoCapacityError&) {
    return BSG_NO_CAPACITY;
  }
}

// capacity_search (metrics.cpp:139-178) of many cells, scheduled at (cell, qps)
// granularity on `threads` std::threads: every integer point of every cell,
// then every cell's tenths — the same runner as ref_capacity_search
// (spec_for_cell + run_experiment + aggregate, driver.cpp:398-418), so each
// cell's result equals capacity_search's (tested against it). This is the
// all-core CPU baseline of the cfg5 sweep: no core idles while one cell's
// sequential search runs. Returns the wall seconds.
double ref_sweep(const bsg_sweep_cell* cells, int32_t n_cells, int32_t threads, bsg_sweep_out* out) {
  struct Pt {
    int32_t cell;
    double qps;
    int8_t pass;
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<ExperimentSpec> base(static_cast<size_t>(n_cells));
  for (int32_t c = 0; c < n_cells; ++c) base[c] = make_experiment(&cells[c].workload, &cells[c].cfg, &cells[c].spec);
  auto run = [&](std::vector<Pt>& pts) {
    // longest first: more instances and more load per run
    std::vector<size_t> order(pts.size());
    for (size_t i = 0; i < pts.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
      return cells[pts[a].cell].spec.n_instances * pts[a].qps > cells[pts[b].cell].spec.n_instances * pts[b].qps;
    });
    std::atomic<size_t> next{0};
    auto work = [&]() {
      for (size_t k; (k = next.fetch_add(1)) < order.size();) {
        Pt& p = pts[order[k]];
        ExperimentSpec spec = spec_for_cell(base[p.cell], base[p.cell].policy.kind, p.qps, cells[p.cell].seed);
        spec.collect_events = false;
        const RunReport r = aggregate(run_experiment(spec));
        p.pass = r.p99_ttft_s < cells[p.cell].slo_p99_ttft_s ? 1 : 0;
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  };
  std::vector<Pt> ints;
  for (int32_t c = 0; c < n_cells; ++c)
    for (int32_t q = cells[c].qps_min; q <= cells[c].qps_max; ++q) ints.push_back(Pt{c, static_cast<double>(q), 0});
  run(ints);
  std::vector<std::vector<bool>> ip(static_cast<size_t>(n_cells));
  for (const Pt& p : ints) ip[p.cell].push_back(p.pass != 0);
  std::vector<Pt> tenths;
  for (int32_t c = 0; c < n_cells; ++c) {
    std::memset(&out[c], 0, sizeof(out[c]));
    bsg_capacity_result& r = out[c].result;
    if (cells[c].qps_min > cells[c].qps_max) {
      out[c].status = BSG_BAD_CONFIG;
      continue;
    }
    if (!ip[c].front()) {
      out[c].status = BSG_NO_CAPACITY;
      r.n_tested = static_cast<int32_t>(ip[c].size());
      continue;
    }
    int last = 0;
    while (last + 1 < static_cast<int>(ip[c].size()) && ip[c][last + 1]) ++last;
    r.monotone = 1;
    for (int i = last + 1; i < static_cast<int>(ip[c].size()); ++i)
      if (ip[c][i]) r.monotone = 0;
    r.bracket_pass = cells[c].qps_min + last;
    r.bracket_fail = r.bracket_pass + 1;
    r.capacity_qps = r.bracket_pass;
    r.n_tested = static_cast<int32_t>(ip[c].size());
    if (r.bracket_pass < cells[c].qps_max)
      for (int t = 1; t <= 9; ++t) tenths.push_back(Pt{c, static_cast<double>(r.bracket_pass * 10 + t) / 10.0, 0});
  }
  run(tenths);
  for (const Pt& p : tenths) {
    bsg_capacity_result& r = out[p.cell].result;
    ++r.n_tested;
    if (p.pass) r.capacity_qps = std::max(r.capacity_qps, p.qps);
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_replay(const bsg_workload* w, const bsg_instance_cfg* cfg, const bsg_replay_spec* spec,
               bsg_request_outcome* out, bsg_replay_summary* summary, ref_capture** capture) {
  ref_capture* cap = capture ? new ref_capture() : nullptr;
  Replay replay(w, cfg, spec, cap);
  try {
    replay.run();
  } catch (const std::exception&) {  // e.g. an unservable workload: report, don't abort the host
    delete cap;
    if (capture) *capture = nullptr;
    return -1;
  }
  if (out) replay.outcomes(out);
  if (summary) {
    std::memset(summary, 0, sizeof(*summary));
    summary->total_preemptions = replay.total_preemptions();
    summary->final_instance_count = spec->n_instances;
  }
  if (capture) *capture = cap;
  return 0;
}

void ref_capture_sizes(const ref_capture* c, int64_t* n_entries, int64_t* n_scenarios) {
  *n_entries = static_cast<int64_t>(c->prompt.size());
  *n_scenarios = static_cast<int64_t>(c->scenarios.size());
}

void ref_capture_copy(const ref_capture* c, uint64_t* id, int32_t* prompt, int32_t* est,
                      int32_t* prefill, int32_t* decoded, bsg_scenario* scenarios) {
  const std::size_t n = c->prompt.size();
  if (id) std::memcpy(id, c->id.data(), n * sizeof(uint64_t));
  std::memcpy(prompt, c->prompt.data(), n * sizeof(int32_t));
  std::memcpy(est, c->est.data(), n * sizeof(int32_t));
  std::memcpy(prefill, c->prefill.data(), n * sizeof(int32_t));
  std::memcpy(decoded, c->decoded.data(), n * sizeof(int32_t));
  std::memcpy(scenarios, c->scenarios.data(), c->scenarios.size() * sizeof(bsg_scenario));
}

void ref_capture_free(ref_capture* c) { delete c; }


// ---- wire schema (json_io.cpp) and the predictor role's /predict handler ----
static int put_text(const std::string& t, char* out, int64_t cap) {
  if (static_cast<int64_t>(t.size()) + 1 > cap) return -static_cast<int>(t.size() + 1);
  std::memcpy(out, t.c_str(), t.size() + 1);
  return static_cast<int>(t.size());
}

// prediction_request_to_json of scenario sc (synthetic ids as make_snapshot).
int ref_request_json(const bsg_instance_cfg* cfg, const bsg_entries* e, const bsg_scenario* sc,
                     char* out, int64_t cap) {
  PredictionRequest req;
  req.snapshot = make_snapshot(e, *sc);
  req.candidate = CandidateRequest{sc->cand_prompt, sc->cand_est};
  req.instance_config = to_ref_config(*cfg);
  return put_text(prediction_request_to_json(req), out, cap);
}

// PredictorService's /predict route (service.cpp:229-241) without the socket:
// returns the HTTP status (200 / 422 / 400) and writes the response body.
int ref_service_predict(const char* body, char* out, int64_t cap) {
  // predictor.cache default (config.cpp:192). One cache per request: the
  // reference service keeps one cache for its lifetime, keyed by batch shape only
  // (predictor.cpp:26-54), which is transparent only while every request carries
  // the same cost model — the fixtures here mix cost models.
  LatencyCache cache(CacheMode::kExact, 256);
  int code = 200;
  std::string text;
  try {
    const PredictionRequest request = prediction_request_from_json(body);
    const PredictionResult result = predict(request, &cache);
    text = prediction_result_to_json(result);
  } catch (const PredictionError& ex) {
    code = 422;
    text = error_body("prediction-failure", ex.what());
  } catch (const Error& ex) {
    code = 400;
    text = error_body("bad-schema", ex.what());
  }
  const int n = put_text(text, out, cap);
  return n < 0 ? n : code;
}


// How the reference's JSON layer prints a double (nlohmann::json::dump).
int ref_dump_double(double v, char* out, int64_t cap) {
  return put_text(nlohmann::json(v).dump(), out, cap);
}

// load_trace (workload.cpp:51-68) on a text; returns the record count, or -1
// with *kind = 1 (TraceParseError, *line) / 2 (InvalidRecordError, field).
int64_t ref_load_trace(const char* text, int64_t len, bsg_trace_record* out, int64_t cap,
                       int32_t* kind, int32_t* line, char* field, int64_t field_cap) {
  *kind = 0;
  *line = 0;
  if (field_cap > 0) field[0] = 0;
  std::istringstream in(std::string(text, static_cast<size_t>(len)));
  std::vector<TraceRecord> recs;
  try {
    recs = load_trace(in);
  } catch (const TraceParseError& e) {
    *kind = 1;
    *line = e.line;
    return -1;
  } catch (const InvalidRecordError& e) {
    *kind = 2;
    std::snprintf(field, static_cast<size_t>(field_cap), "%s", e.field.c_str());
    return -1;
  }
  for (size_t i = 0; i < recs.size() && static_cast<int64_t>(i) < cap; ++i) {
    bsg_trace_record& r = out[i];
    r.id = recs[i].id;
    r.prompt_tokens = recs[i].prompt_tokens;
    r.output_tokens = recs[i].output_tokens;
    r.estimated_output_tokens = recs[i].estimated_output_tokens.value_or(0);
    r.has_arrival_offset = recs[i].arrival_offset_s.has_value() ? 1 : 0;
    r.arrival_offset_s = recs[i].arrival_offset_s.value_or(0.0);
  }
  return static_cast<int64_t>(recs.size());
}

// Installs trace records for make_workload / run_experiment / run_report
// (n < 0 restores the synthetic trace).
void ref_set_trace(const bsg_trace_record* recs, int64_t n) {
  delete g_trace;
  g_trace = nullptr;
  if (n < 0) return;
  g_trace = new std::vector<TraceRecord>();
  for (int64_t i = 0; i < n; ++i) {
    TraceRecord r;
    r.id = recs[i].id;
    r.prompt_tokens = recs[i].prompt_tokens;
    r.output_tokens = recs[i].output_tokens;
    if (recs[i].estimated_output_tokens > 0) r.estimated_output_tokens = recs[i].estimated_output_tokens;
    if (recs[i].has_arrival_offset) r.arrival_offset_s = recs[i].arrival_offset_s;
    g_trace->push_back(r);
  }
}

// write_trace (workload.cpp:78-89) into out; returns the length (or -needed).
int64_t ref_write_trace(const bsg_trace_record* recs, int64_t n, char* out, int64_t cap) {
  std::vector<TraceRecord> v;
  for (int64_t i = 0; i < n; ++i) {
    TraceRecord r;
    r.id = recs[i].id;
    r.prompt_tokens = recs[i].prompt_tokens;
    r.output_tokens = recs[i].output_tokens;
    if (recs[i].estimated_output_tokens > 0) r.estimated_output_tokens = recs[i].estimated_output_tokens;
    if (recs[i].has_arrival_offset) r.arrival_offset_s = recs[i].arrival_offset_s;
    v.push_back(r);
  }
  std::ostringstream os;
  write_trace(os, v);
  const std::string s = os.str();
  if (static_cast<int64_t>(s.size()) > cap) return -static_cast<int64_t>(s.size());
  std::memcpy(out, s.data(), s.size());
  return static_cast<int64_t>(s.size());
}

}  // extern "C"


// ---- run_sweep / run_capacity (driver.cpp:333-427) through the reference itself
extern "C" {

// run_sweep(base, SweepSpec{policies, qps_values, seeds, jobs}); rows in the
// reference's cell order. Returns the number of rows, -1 if it threw.
int ref_run_sweep(const bsg_workload* w, const bsg_instance_cfg* c, const bsg_replay_spec* s,
                  const int32_t* policies, int32_t n_policies, const double* qps, int32_t n_qps,
                  const uint64_t* seeds, int32_t n_seeds, int32_t jobs, bsg_sweep_row* rows) {
  try {
    const ExperimentSpec base = make_experiment(w, c, s);
    SweepSpec sw;
    for (int32_t i = 0; i < n_policies; ++i) sw.policies.push_back(to_ref_policy(policies[i]));
    sw.qps_values.assign(qps, qps + n_qps);
    sw.seeds.assign(seeds, seeds + n_seeds);
    sw.jobs = jobs;
    const std::vector<SweepCell> cells = run_sweep(base, sw);
    for (std::size_t i = 0; i < cells.size(); ++i) {
      const SweepCell& x = cells[i];
      bsg_sweep_row& r = rows[i];
      std::memset(&r, 0, sizeof(r));
      r.policy = static_cast<int32_t>(x.policy);
      r.ok = x.ok ? 1 : 0;
      r.qps = x.qps;
      r.seed = x.seed;
      r.status = x.ok ? 0 : -1;
      r.finished_requests = x.finished_requests;
      r.mean_ttft_s = x.mean_ttft_s;
      r.p99_ttft_s = x.p99_ttft_s;
      r.mean_e2e_s = x.mean_e2e_s;
      r.p99_e2e_s = x.p99_e2e_s;
      r.throughput_rps = x.throughput_rps;
      r.total_preemptions = x.total_preemptions;
      r.free_blocks_var_avg = x.free_blocks_var_avg;
    }
    return static_cast<int>(cells.size());
  } catch (const std::exception&) {
    return -1;
  }
}

// run_capacity(base, CapacitySpec{...}): rows in table order, gains as the
// reference formats them. Returns the row count; -12 on NoCapacityError, -1 on
// any other exception.
int ref_run_capacity(const bsg_workload* w, const bsg_instance_cfg* c, const bsg_replay_spec* s,
                     const int32_t* policies, int32_t n_policies, int32_t baseline, uint64_t seed,
                     int32_t qps_min, int32_t qps_max, double slo, bsg_capacity_row* rows,
                     double* baseline_capacity) {
  try {
    const ExperimentSpec base = make_experiment(w, c, s);
    CapacitySpec cs;
    for (int32_t i = 0; i < n_policies; ++i) cs.policies.push_back(to_ref_policy(policies[i]));
    cs.baseline = to_ref_policy(baseline);
    cs.qps_min = qps_min;
    cs.qps_max = qps_max;
    cs.slo_p99_ttft_s = slo;
    cs.seed = seed;
    const CapacityTable t = run_capacity(base, cs);
    *baseline_capacity = t.baseline_capacity;
    for (std::size_t i = 0; i < t.rows.size(); ++i) {
      const CapacityTableRow& x = t.rows[i];
      bsg_capacity_row& r = rows[i];
      std::memset(&r, 0, sizeof(r));
      r.policy = static_cast<int32_t>(x.policy);
      r.result.capacity_qps = x.result.capacity_qps;
      r.result.bracket_pass = x.result.bracket_pass;
      r.result.bracket_fail = x.result.bracket_fail;
      r.result.monotone = x.result.monotone ? 1 : 0;
      r.result.n_tested = static_cast<int32_t>(x.result.tested.size());
      for (const auto& [name, text] : t.gains)
        if (name == to_string(x.policy)) {
          r.has_gain = 1;
          std::snprintf(r.gain_text, sizeof(r.gain_text), "%s", text.c_str());
        }
    }
    return static_cast<int>(t.rows.size());
  } catch (const NoCapacityError&) {
    return -12;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"

// bsg_driver.cpp — closed-loop replay: the scenario source and sweep driver.
//
// Replays a synthetic trace through N live serving instances; every arrival
// is dispatched by the configured policy, and BlockPredictive dispatches run
// their per-instance what-if simulations on the GPU (bsg_dispatch). This is
// the behaviour of SimulationDriver (core/src/driver.cpp:134-289) for static
// provisioning, zero dispatch overhead and no probes, over the same
// workload generators (core/src/workload.cpp:113-191) and dispatcher
// heuristics (core/src/scheduler.cpp:33-113).
//
// The live instances here are host C++ (they are the simulated backends the
// snapshots come from, not the prediction path). Their state is kept in the
// same "resident list" form as the GPU kernel (scenario_sim.cuh): running
// members [0,n) in admission order, preemption victims [n,L) = the waiting
// front, then never-scheduled arrivals in FIFO order.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstring>
#include <deque>
#include <limits>
#include <memory>
#include <queue>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "bsg_internal.h"

namespace {

// ---- fully specified RNG (SplitMix64 + helpers, rand.h:11-56) -------------
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double u01_open_low() { return 1.0 - u01(); }
  uint64_t below(uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t r;
    do r = next(); while (r >= limit);
    return r % n;
  }
  double exponential(double rate) { return -std::log(u01_open_low()) / rate; }
  double normal() {
    const double u1 = u01_open_low();
    const double u2 = u01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }
};
uint64_t mix_seed(uint64_t seed, uint64_t id) {
  Rng s(id * 0x9e3779b97f4a7c15ULL + 0x1b873593ULL);
  return seed ^ s.next();
}

int64_t ticks_from_seconds(double s) { return static_cast<int64_t>(std::llround(s * 1e9)); }

struct Record {
  int32_t prompt, output, est;
  int64_t arrival;
};

// estimate_length (workload.cpp:113-139) for the oracle / fixed / noisy kinds.
int32_t estimate(const bsg_workload& w, uint64_t record_id, int32_t output) {
  switch (w.estimator_kind) {
    case 1: return w.fixed_tokens;
    case 2: {
      Rng e(mix_seed(w.estimator_seed, record_id));
      const double half = std::abs(e.normal());
      const double sign = (e.next() & 1) ? 1.0 : -1.0;
      const double scale = w.mean_abs_rel_error * std::sqrt(3.14159265358979323846 / 2.0);
      const double est = std::round(static_cast<double>(output) * (1.0 + sign * half * scale));
      return static_cast<int32_t>(std::max(1.0, est));
    }
    default: return output;
  }
}

void trace_err(bsg_trace_error* err, int32_t kind, const char* field, const std::string& msg) {
  if (!err) return;
  err->kind = kind;
  err->line = 0;
  std::snprintf(err->field, sizeof(err->field), "%s", field);
  std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

// The SimulationDriver constructor's request build (driver.cpp:137-160) over
// trace records: request_cap, generate_arrivals (workload.cpp:141-170), then
// estimate_length per request in arrival-list order.
bsg_status records_from_trace(const bsg_trace_record* tr, int64_t n, const bsg_workload& w,
                              std::vector<Record>* out, bsg_trace_error* err) {
  if (n < 0 || (!tr && n > 0)) return BSG_INVALID_ARGUMENT;
  if (err) std::memset(err, 0, sizeof(*err));
  const int64_t m = (w.request_cap >= 0 && w.request_cap < n) ? w.request_cap : n;
  std::vector<Record> recs(static_cast<size_t>(m));
  if (m > 0) {
    const bool first = tr[0].has_arrival_offset != 0;
    for (int64_t i = 0; i < m; ++i)
      if ((tr[i].has_arrival_offset != 0) != first) {
        trace_err(err, 2, "arrival_offset_s",
                  "invalid trace record: arrival_offset_s: either every record carries an offset or none does");
        return BSG_BAD_INPUT;
      }
    if (first) {
      for (int64_t i = 0; i < m; ++i) recs[i].arrival = ticks_from_seconds(tr[i].arrival_offset_s);
    } else {
      if (!(w.qps > 0)) {
        trace_err(err, 3, "workload.qps", "invalid config: workload.qps: must be > 0");
        return BSG_BAD_INPUT;
      }
      Rng arr(w.arrival_seed);
      int64_t t = 0;
      for (int64_t i = 0; i < m; ++i) {
        t += ticks_from_seconds(arr.exponential(w.qps));
        recs[i].arrival = t;
      }
    }
  }
  for (int64_t i = 0; i < m; ++i) {
    Record& r = recs[i];
    r.prompt = tr[i].prompt_tokens;
    r.output = tr[i].output_tokens;
    if (w.estimator_kind == 3) {  // EstimatorKind::kTrace
      if (tr[i].estimated_output_tokens < 1) {
        trace_err(err, 2, "estimated_output_tokens",
                  "invalid trace record: estimated_output_tokens: trace estimator needs pre-tagged records (record " +
                      std::to_string(tr[i].id) + " has none)");
        return BSG_BAD_INPUT;
      }
      r.est = tr[i].estimated_output_tokens;
    } else {
      r.est = estimate(w, tr[i].id, r.output);
    }
  }
  *out = std::move(recs);
  return BSG_OK;
}

// make_synthetic_trace (workload.cpp:172-191) + estimate_length
// (workload.cpp:113-139) + generate_arrivals (workload.cpp:141-170).
// make_synthetic_trace (workload.cpp:172-191): lognormal prompt / output
// lengths, record i has id i.
std::vector<Record> synthetic_trace(const bsg_workload& w) {
  Rng rng(w.trace_seed);
  std::vector<Record> recs;
  recs.reserve(static_cast<size_t>(std::max(w.count, 0)));
  for (int i = 0; i < w.count; ++i) {
    const double p = w.prompt_median * std::exp(w.prompt_sigma * rng.normal());
    const double o = w.output_median * std::exp(w.output_sigma * rng.normal());
    Record r{};
    r.prompt = static_cast<int32_t>(std::clamp<double>(std::round(p), w.min_tokens, w.max_prompt_tokens));
    r.output = static_cast<int32_t>(std::clamp<double>(std::round(o), w.min_tokens, w.max_output_tokens));
    recs.push_back(r);
  }
  return recs;
}

bsg_status make_records(const bsg_workload& w, std::vector<Record>* out) {
  if (!(w.qps > 0)) return BSG_INVALID_ARGUMENT;
  const int n = w.count;
  std::vector<Record> recs = synthetic_trace(w);
  if (w.request_cap >= 0 && w.request_cap < n) recs.resize(w.request_cap);
  Rng arr(w.arrival_seed);
  int64_t t = 0;
  for (size_t i = 0; i < recs.size(); ++i) {
    Record& r = recs[i];
    r.est = estimate(w, static_cast<uint64_t>(i), r.output);  // synthetic ids are row numbers
    t += ticks_from_seconds(arr.exponential(w.qps));
    r.arrival = t;
  }
  *out = std::move(recs);
  return BSG_OK;
}

int64_t blocks(int64_t t, int32_t bs) { return t <= 0 ? 0 : (t + bs - 1) / bs; }

// ---- live serving instance ------------------------------------------------
struct Member {
  int32_t prompt, target, est, prefill, decoded;
  int32_t rid;
  bool ever;
  int32_t stored() const { return prefill + decoded; }
  bool ready() const { return prefill == prompt; }
};

class LiveInstance {
 public:
  explicit LiveInstance(const bsg_instance_cfg& c) : c_(c), free_(c.total_blocks) {}

  void admit(int32_t rid, int32_t prompt, int32_t target, int32_t est) {
    fifo_.push_back(Member{prompt, target, est, 0, 0, rid, false});
  }
  bool has_work() const { return n_ > 0 || res_.size() > static_cast<size_t>(n_) || !fifo_.empty(); }
  bool mid_step() const { return mid_; }

  // Status snapshot (Instance::snapshot semantics, backend.cpp:351-373): running
  // in admission order, waiting head first, free recomputed from stored tokens.
  void snapshot(std::vector<Member>* running, std::vector<Member>* waiting, int32_t* free_blocks,
                int32_t* batch) const {
    running->assign(res_.begin(), res_.begin() + n_);
    waiting->assign(res_.begin() + n_, res_.end());
    waiting->insert(waiting->end(), fifo_.begin(), fifo_.end());
    int64_t held = 0;
    for (int32_t p = 0; p < n_; ++p) held += blocks(res_[p].stored(), c_.block_size);
    *free_blocks = static_cast<int32_t>(c_.total_blocks - held);
    *batch = n_;
  }

  // Forms the batch, admits, allocates with newest-member preemption and prices
  // the step. Returns the step duration in ticks; appends victim request ids.
  bsg_status begin_step(int64_t* duration, std::vector<int32_t>* preempted) {
    const int32_t bs = c_.block_size;
    const bool chunked = c_.local_policy == BSG_CHUNKED_PREFILL;
    const int32_t L = static_cast<int32_t>(res_.size());
    chunk_.assign(res_.size(), 0);
    decode_.assign(res_.size(), 0);
    std::vector<int32_t> delta(res_.size(), 0);
    int32_t D = 0;
    bool any_nonready = false;
    for (int32_t p = 0; p < n_; ++p) {
      if (res_[p].ready()) ++D;
      else any_nonready = true;
    }
    const bool waiting = L > n_ || !fifo_.empty();
    int64_t budget = 0;
    bool prefill_step = false;
    if (chunked) {
      budget = std::max<int64_t>(0, static_cast<int64_t>(c_.chunk_budget) - D);
      for (int32_t p = 0; p < n_; ++p) decode_[p] = res_[p].ready();
      for (int32_t p = 0; p < n_ && budget > 0; ++p) {
        if (!res_[p].ready()) {
          chunk_[p] = static_cast<int32_t>(std::min<int64_t>(res_[p].prompt - res_[p].prefill, budget));
          budget -= chunk_[p];
        }
      }
    } else {
      prefill_step = waiting || any_nonready;
      for (int32_t p = 0; p < n_; ++p) {
        if (prefill_step && !res_[p].ready()) chunk_[p] = res_[p].prompt - res_[p].prefill;
        decode_[p] = !prefill_step && res_[p].ready();
      }
    }
    auto item_delta = [&](const Member& m, bool dec, int32_t ch) -> int32_t {
      const int32_t s = m.stored();
      int32_t ns = s;
      if (dec) ns = s + 1;
      else if (ch > 0) ns = m.prefill + ch + m.decoded + (m.prefill + ch == m.prompt ? 1 : 0);
      return static_cast<int32_t>(blocks(ns, bs) - blocks(s, bs));
    };
    int64_t pf = free_;
    for (int32_t p = 0; p < n_; ++p) {
      if (decode_[p] || chunk_[p] > 0) {
        delta[p] = item_delta(res_[p], decode_[p], chunk_[p]);
        pf -= delta[p];
      }
    }
    // waiting admissions: victim stack first, then FIFO arrivals
    int32_t a = 0;
    std::vector<int32_t> adm_chunk, adm_delta;
    {
      int32_t members = n_;
      const size_t total_wait = static_cast<size_t>(L - n_) + fifo_.size();
      for (size_t j = 0; j < total_wait; ++j) {
        if ((chunked && budget == 0) || members >= c_.max_batch_size) break;
        const Member& m = j < static_cast<size_t>(L - n_) ? res_[n_ + j] : fifo_[j - (L - n_)];
        int32_t ch = m.prompt - m.prefill;
        if (chunked) ch = static_cast<int32_t>(std::min<int64_t>(ch, budget));
        const int32_t d = item_delta(m, false, ch);
        if (d > pf) break;
        adm_chunk.push_back(ch);
        adm_delta.push_back(d);
        if (chunked) budget -= ch;
        pf -= d;
        ++members;
        ++a;
      }
    }
    if (!chunked && prefill_step && !any_nonready && a == 0) {
      for (int32_t p = 0; p < n_; ++p) {
        decode_[p] = res_[p].ready();
        delta[p] = decode_[p] ? item_delta(res_[p], true, 0) : 0;
      }
    }
    if (n_ == 0 && a == 0) return BSG_EMPTY_PLAN;
    // admissions move waiting heads into the running tail
    const int32_t n_adm = n_ + a;
    for (int32_t j = 0; j < a; ++j) {
      if (n_ + j >= static_cast<int32_t>(res_.size())) {
        res_.push_back(fifo_.front());
        fifo_.pop_front();
        chunk_.push_back(0);
        decode_.push_back(0);
        delta.push_back(0);
      }
      chunk_[n_ + j] = adm_chunk[j];
      delta[n_ + j] = adm_delta[j];
      res_[n_ + j].ever = true;
    }
    // allocation: survivors e* = max{e : F(e) >= 0} (see scenario_sim.cuh)
    int64_t tot = 0;
    for (int32_t p = 0; p < n_adm; ++p) tot += delta[p];
    int32_t e_star = n_adm;
    if (tot > free_) {
      int64_t f = free_;
      for (int32_t p = 0; p < n_; ++p) f += blocks(res_[p].stored(), bs);  // F(0)
      // F(e+1) = F(e) - held_old[e] - delta[e]
      e_star = 0;
      for (int32_t p = 0; p < n_adm; ++p) {
        const int64_t fn = f - (p < n_ ? blocks(res_[p].stored(), bs) : 0) - delta[p];
        if (fn < 0) break;
        f = fn;
        e_star = p + 1;
      }
      if (e_star == 0) return BSG_DEADLOCK;
      free_ = f;
      for (int32_t p = n_adm - 1; p >= e_star; --p) {
        preempted->push_back(res_[p].rid);
        res_[p].prefill = 0;
        res_[p].decoded = 0;
        chunk_[p] = 0;
        decode_[p] = 0;
      }
    } else {
      free_ -= tot;
    }
    n_ = e_star;
    int64_t ctx = 0, pt = 0, nd = 0;
    for (int32_t p = 0; p < n_; ++p) {
      if (decode_[p]) {
        ++nd;
        ctx += res_[p].stored();
      } else if (chunk_[p] > 0) {
        pt += chunk_[p];
      }
    }
    // batch_latency itself (driver.cpp:274: begin_step() without a latency
    // function); the predictor's cache mode does not apply to live instances
    const double x = c_.c0_s + c_.prefill_s_per_token * static_cast<double>(pt) +
                     c_.decode_s_per_seq * static_cast<double>(nd) +
                     c_.context_s_per_token * static_cast<double>(ctx);
    *duration = ticks_from_seconds(x);
    mid_ = true;
    return BSG_OK;
  }

  void finish_step(std::vector<int32_t>* first_tokens, std::vector<int32_t>* completed) {
    std::vector<char> done(res_.size(), 0);
    for (int32_t p = 0; p < n_; ++p) {
      Member& m = res_[p];
      const bool item = decode_[p] || chunk_[p] > 0;
      if (!item) continue;
      const int32_t prev = m.decoded;
      if (decode_[p]) {
        m.decoded += 1;
      } else {
        m.prefill += chunk_[p];
        if (m.prefill == m.prompt) m.decoded += 1;
      }
      if (prev == 0 && m.decoded >= 1) first_tokens->push_back(m.rid);
      if (m.decoded >= m.target) {
        completed->push_back(m.rid);
        done[p] = 1;
      }
    }
    std::vector<Member> keep;
    keep.reserve(res_.size());
    int32_t removed = 0;
    for (size_t p = 0; p < res_.size(); ++p) {
      if (done[p]) {
        free_ += blocks(res_[p].stored(), c_.block_size);
        ++removed;
      } else {
        keep.push_back(res_[p]);
      }
    }
    res_.swap(keep);
    n_ -= removed;
    mid_ = false;
  }

 private:
  bsg_instance_cfg c_;
  std::vector<Member> res_;  // [0,n) running, [n, L) victims (waiting front)
  int32_t n_ = 0;
  std::deque<Member> fifo_;
  int64_t free_;
  bool mid_ = false;
  std::vector<int32_t> chunk_;
  std::vector<char> decode_;
};

// ---- DES kernel (event_loop.cpp:28-57 semantics) --------------------------
struct Ev {
  int64_t t;
  uint64_t seq;
  int32_t kind;  // 0 arrival, 1 batch complete, 2 provision complete, 3 dispatch (landing)
  int32_t a;
  bool operator>(const Ev& o) const { return t != o.t ? t > o.t : seq > o.seq; }
};

struct QpmWindow {  // QpmTracker (scheduler.cpp:48-63)
  std::deque<int64_t> w;
  void record(int64_t now) {
    w.push_back(now);
    const int64_t cutoff = now - ticks_from_seconds(60.0);
    while (!w.empty() && w.front() <= cutoff) w.pop_front();
  }
  int qpm(int64_t now) const {
    const int64_t cutoff = now - ticks_from_seconds(60.0);
    return static_cast<int>(w.end() - std::upper_bound(w.begin(), w.end(), cutoff));
  }
};

}  // namespace

struct bsg_capture {
  std::vector<uint64_t> id;
  std::vector<int32_t> prompt, est, prefill, decoded;
  std::vector<bsg_scenario> scenarios;
};

namespace {

class Replay {
 public:
  Replay(bsg_ctx* ctx, const bsg_instance_cfg& cfg, const bsg_replay_spec& spec,
         std::vector<Record> recs, bsg_capture* cap)
      : ctx_(ctx), cfg_(cfg), spec_(spec), recs_(std::move(recs)), cap_(cap), rng_(spec.policy_seed) {
    for (int i = 0; i < spec.n_instances; ++i) inst_.emplace_back(cfg);
    qpm_.resize(spec.n_instances);
    active_ = spec.n_instances;
    next_instance_id_ = spec.n_instances;
    out_.resize(recs_.size());
    land_inst_.assign(recs_.size(), -1);
    for (size_t i = 0; i < recs_.size(); ++i) {
      out_[i] = bsg_request_outcome{recs_[i].arrival, -1, -1, -1, -1, 0};
      push(recs_[i].arrival, 0, static_cast<int32_t>(i));
    }
  }

  bsg_status run() {
    bool open = false;
    for (;;) {
      if (q_.empty() || (open && q_.top().t > now_)) {
        if (open) {
          open = false;
          const bsg_status st = end_of_instant();
          if (st != BSG_OK) return st;
          continue;
        }
        if (q_.empty()) break;
      }
      const Ev ev = q_.top();
      q_.pop();
      now_ = ev.t;
      const bsg_status st = ev.kind == 0   ? arrival(ev.a)
                            : ev.kind == 1 ? complete(ev.a)
                            : ev.kind == 2 ? provision_complete(ev.a)
                                           : land(ev.a);
      if (st != BSG_OK) return st;
      open = true;
    }
    return BSG_OK;
  }

  const std::vector<bsg_request_outcome>& outcomes() const { return out_; }
  // means over dispatch points of the snapshot free-block mean / variance (metrics.cpp:79-86)
  void balance(double* mean_avg, double* var_avg) const {
    *mean_avg = n_points_ ? fm_sum_ / static_cast<double>(n_points_) : 0.0;
    *var_avg = n_points_ ? fv_sum_ / static_cast<double>(n_points_) : 0.0;
  }
  void summary(bsg_replay_summary* s) const {
    s->total_preemptions = preemptions_;
    s->end_ticks = now_;
    s->instances_provisioned = provisioned_total_;
    s->final_instance_count = static_cast<int32_t>(inst_.size());
  }

 private:
  void push(int64_t t, int32_t kind, int32_t a) { q_.push(Ev{t, seq_++, kind, a}); }

  bsg_status end_of_instant() {  // driver.cpp:271-289
    for (size_t i = 0; i < inst_.size(); ++i) {
      LiveInstance& li = inst_[i];
      if (li.mid_step() || !li.has_work()) continue;
      int64_t dur = 0;
      victims_.clear();
      const bsg_status st = li.begin_step(&dur, &victims_);
      if (st != BSG_OK) return st;
      push(now_ + dur, 1, static_cast<int32_t>(i));
      for (int32_t rid : victims_) {
        out_[rid].preempt_count += 1;
        preemptions_ += 1;
      }
    }
    return BSG_OK;
  }

  bsg_status complete(int32_t iid) {  // driver.cpp:233-251
    firsts_.clear();
    dones_.clear();
    inst_[iid].finish_step(&firsts_, &dones_);
    for (int32_t rid : firsts_)
      if (out_[rid].first_token_ticks < 0) out_[rid].first_token_ticks = now_;
    for (int32_t rid : dones_) {
      out_[rid].finish_ticks = now_;
      if (spec_.provision_kind == 2)
        maybe_provision(2, static_cast<double>(now_ - out_[rid].arrival_ticks) * 1e-9);
    }
    return BSG_OK;
  }

  // Autoscaler::evaluate (autoscaler.cpp:36-52) + maybe_provision (driver.cpp:253-261).
  void maybe_provision(int32_t signal_kind, double latency_s) {
    if (spec_.provision_kind == 0 || signal_kind != spec_.provision_kind) return;
    if (latency_s < spec_.threshold_s) return;
    if (has_last_provision_ && now_ - last_provision_ < ticks_from_seconds(spec_.cooldown_s)) return;
    if (active_ + pending_ >= spec_.max_instances) return;
    last_provision_ = now_;
    has_last_provision_ = true;
    ++pending_;
    ++provisioned_total_;
    push(now_ + ticks_from_seconds(spec_.cold_start_s), 2, next_instance_id_++);
  }

  bsg_status provision_complete(int32_t iid) {  // driver.cpp:263-269
    if (iid < static_cast<int32_t>(inst_.size())) return BSG_INVALID_ARGUMENT;
    inst_.emplace_back(cfg_);
    qpm_.resize(inst_.size());
    --pending_;
    ++active_;
    return BSG_OK;
  }

  bsg_status arrival(int32_t rid) {  // driver.cpp:134-219 (static, no probes)
    const int n = static_cast<int>(inst_.size());
    snaps_run_.resize(n);
    snaps_wait_.resize(n);
    free_.resize(n);
    batch_.resize(n);
    for (int i = 0; i < n; ++i)
      inst_[i].snapshot(&snaps_run_[i], &snaps_wait_[i], &free_[i], &batch_[i]);
    {  // memory-balance sample before this dispatch lands (driver.cpp:142-157)
      double mean = 0;
      for (int i = 0; i < n; ++i) mean += free_[i];
      mean /= static_cast<double>(n);
      double var = 0;
      for (int i = 0; i < n; ++i) {
        const double d = free_[i] - mean;
        var += d * d;
      }
      var /= static_cast<double>(n);
      fm_sum_ += mean;
      fv_sum_ += var;
      n_points_ += 1;
    }
    int32_t chosen = 0;
    bool have_prediction = false;
    const bsg_status st = decide(rid, &chosen, &have_prediction);
    if (st != BSG_OK) return st;
    qpm_[chosen].record(now_);
    if (spec_.provision_kind == 1) {  // driver.cpp:197-211
      int64_t e2e = 0;
      if (have_prediction) {
        e2e = per_[chosen].e2e_ticks;
      } else {
        const bsg_status ps = predict_one(rid, chosen, &e2e);
        if (ps != BSG_OK) return ps;
      }
      maybe_provision(1, static_cast<double>(e2e) * 1e-9);
    }
    out_[rid].instance = chosen;
    if (spec_.dispatch_overhead_s == 0) {  // driver.cpp:213-218
      admit_to_instance(rid, chosen);
    } else {
      land_inst_[rid] = chosen;
      push(now_ + ticks_from_seconds(spec_.dispatch_overhead_s), 3, rid);
    }
    return BSG_OK;
  }

  // kDispatch: the request lands at its instance after the overhead (handle_dispatch)
  bsg_status land(int32_t rid) {
    admit_to_instance(rid, land_inst_[rid]);
    return BSG_OK;
  }

  void admit_to_instance(int32_t rid, int32_t iid) {  // driver.cpp:224-231
    const Record& r = recs_[rid];
    inst_[iid].admit(rid, r.prompt, r.output, r.est);
    out_[rid].dispatch_ticks = now_;
  }

  // Dispatcher::dispatch (scheduler.cpp:115-152) with the heuristics of
  // pick_heuristic (scheduler.cpp:68-113).
  // predict() for one instance's snapshot (heuristic policies under preempt
  // provisioning ask for the chosen instance's prediction, driver.cpp:202-209).
  bsg_status predict_one(int32_t rid, int32_t iid, int64_t* e2e) {
    prompt_.clear();
    est_.clear();
    prefill_.clear();
    decoded_.clear();
    ids_.clear();
    bsg_scenario sc{};
    sc.run_n = static_cast<int32_t>(snaps_run_[iid].size());
    for (const Member& m : snaps_run_[iid]) add(m);
    sc.wait_off = static_cast<int32_t>(prompt_.size());
    sc.wait_n = static_cast<int32_t>(snaps_wait_[iid].size());
    for (const Member& m : snaps_wait_[iid]) add(m);
    sc.cand_prompt = recs_[rid].prompt;
    sc.cand_est = recs_[rid].est;
    bsg_entries e{ids_.data(), prompt_.data(), est_.data(), prefill_.data(), decoded_.data()};
    bsg_result r{};
    const bsg_status st = bsg_predict_batch(ctx_, &e, static_cast<int64_t>(prompt_.size()), &sc, 1, &r);
    if (st != BSG_OK) return st;
    if (r.status != BSG_OK) return static_cast<bsg_status>(r.status);
    *e2e = r.e2e_ticks;
    return BSG_OK;
  }

  bsg_status decide(int32_t rid, int32_t* chosen, bool* have_prediction) {
    *have_prediction = false;
    const int n = static_cast<int>(inst_.size());
    switch (spec_.policy) {
      case BSG_POLICY_RANDOM: *chosen = static_cast<int32_t>(rng_.below(n)); return BSG_OK;
      case BSG_POLICY_ROUND_ROBIN: *chosen = static_cast<int32_t>(rr_++ % n); return BSG_OK;
      case BSG_POLICY_MIN_QPM:
      case BSG_POLICY_INFAAS_PP:
      case BSG_POLICY_LLUMNIX_MINUS: {
        double best = std::numeric_limits<double>::infinity();
        int32_t best_id = 0;
        for (int i = 0; i < n; ++i) {
          double score = 0;
          const double used = static_cast<double>(cfg_.total_blocks - free_[i]);
          const double bsz = static_cast<double>(std::max(batch_[i], 1));
          if (spec_.policy == BSG_POLICY_MIN_QPM) {
            score = static_cast<double>(qpm_[i].qpm(now_));
          } else if (spec_.policy == BSG_POLICY_INFAAS_PP) {
            score = used / bsz;  // load_infaas, scheduler.cpp:33-36
          } else {
            int64_t pm = 0;  // load_llumnix, scheduler.cpp:38-46
            for (const Member& m : snaps_wait_[i]) pm += blocks(m.prompt - m.prefill, cfg_.block_size);
            score = (used + static_cast<double>(pm)) / bsz;
          }
          if (i == 0 || score < best) {
            best = score;
            best_id = i;
          }
        }
        *chosen = best_id;
        return BSG_OK;
      }
      default: break;
    }
    // BlockPredictive: per-instance what-ifs on the GPU, argmin with lowest-id ties.
    prompt_.clear();
    est_.clear();
    prefill_.clear();
    decoded_.clear();
    ids_.clear();
    scen_.assign(n, bsg_scenario{});
    inst_ids_.resize(n);
    const Record& r = recs_[rid];
    for (int i = 0; i < n; ++i) {
      bsg_scenario& sc = scen_[i];
      sc.run_off = static_cast<int32_t>(prompt_.size());
      sc.run_n = static_cast<int32_t>(snaps_run_[i].size());
      for (const Member& m : snaps_run_[i]) add(m);
      sc.wait_off = static_cast<int32_t>(prompt_.size());
      sc.wait_n = static_cast<int32_t>(snaps_wait_[i].size());
      for (const Member& m : snaps_wait_[i]) add(m);
      sc.cand_prompt = r.prompt;
      sc.cand_est = r.est;
      sc.cfg = 0;
      inst_ids_[i] = i;
    }
    if (cap_) {
      const int32_t base = static_cast<int32_t>(cap_->prompt.size());
      for (bsg_scenario sc : scen_) {
        sc.run_off += base;
        sc.wait_off += base;
        cap_->scenarios.push_back(sc);
      }
      cap_->id.insert(cap_->id.end(), ids_.begin(), ids_.end());
      cap_->prompt.insert(cap_->prompt.end(), prompt_.begin(), prompt_.end());
      cap_->est.insert(cap_->est.end(), est_.begin(), est_.end());
      cap_->prefill.insert(cap_->prefill.end(), prefill_.begin(), prefill_.end());
      cap_->decoded.insert(cap_->decoded.end(), decoded_.begin(), decoded_.end());
    }
    bsg_entries e{ids_.data(), prompt_.data(), est_.data(), prefill_.data(), decoded_.data()};
    int32_t pick = -1;
    per_.resize(n);
    const bsg_status st = bsg_dispatch(ctx_, &e, static_cast<int64_t>(prompt_.size()), scen_.data(),
                                       inst_ids_.data(), n, 1, spec_.objective, &pick, per_.data());
    if (st != BSG_OK) return st;
    if (pick < 0) {
      for (const bsg_result& x : per_)
        if (x.status != BSG_OK) return static_cast<bsg_status>(x.status);
      return BSG_INVALID_ARGUMENT;
    }
    *chosen = pick;
    *have_prediction = true;
    return BSG_OK;
  }

  void add(const Member& m) {
    ids_.push_back(static_cast<uint64_t>(m.rid));
    prompt_.push_back(m.prompt);
    est_.push_back(m.est);
    prefill_.push_back(m.prefill);
    decoded_.push_back(m.decoded);
  }

  bsg_ctx* ctx_;
  bsg_instance_cfg cfg_;
  bsg_replay_spec spec_;
  std::vector<Record> recs_;
  bsg_capture* cap_;
  Rng rng_;
  uint64_t rr_ = 0;
  std::vector<LiveInstance> inst_;
  std::vector<QpmWindow> qpm_;
  std::vector<bsg_request_outcome> out_;
  std::vector<int32_t> land_inst_;  // overhead mode: the instance a request lands at
  double fm_sum_ = 0, fv_sum_ = 0;
  int64_t n_points_ = 0;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> q_;
  uint64_t seq_ = 0;
  int64_t now_ = 0;
  int64_t preemptions_ = 0;
  int32_t active_ = 0, pending_ = 0, provisioned_total_ = 0, next_instance_id_ = 0;
  int64_t last_provision_ = 0;
  bool has_last_provision_ = false;
  std::vector<int32_t> victims_, firsts_, dones_;
  std::vector<std::vector<Member>> snaps_run_, snaps_wait_;
  std::vector<int32_t> free_, batch_;
  std::vector<int32_t> prompt_, est_, prefill_, decoded_, inst_ids_;
  std::vector<uint64_t> ids_;
  std::vector<bsg_scenario> scen_;
  std::vector<bsg_result> per_;
};

}  // namespace

extern "C" {

bsg_status bsg_mc_lengths(int32_t est, uint64_t request_id, int32_t n_samples, uint64_t seed,
                          double mean_abs_rel_error, int32_t* out) {
  if (!out || n_samples < 0) return BSG_INVALID_ARGUMENT;
  // estimate_length's Noisy branch (workload.cpp:126-136) applied to the
  // predicted length, one SplitMix64 stream per sample.
  const double scale = mean_abs_rel_error * std::sqrt(3.14159265358979323846 / 2.0);
  for (int32_t s = 0; s < n_samples; ++s) {
    Rng rng(mix_seed(seed, request_id * static_cast<uint64_t>(n_samples) + static_cast<uint64_t>(s)));
    const double half = std::abs(rng.normal());
    const double sign = (rng.next() & 1) ? 1.0 : -1.0;
    const double v = std::round(static_cast<double>(est) * (1.0 + sign * half * scale));
    out[s] = static_cast<int32_t>(std::max(1.0, v));
  }
  return BSG_OK;
}

bsg_status bsg_make_workload(const bsg_workload* w, int32_t* prompt, int32_t* output, int32_t* est,
                             int64_t* arrival_ticks) {
  if (!w) return BSG_INVALID_ARGUMENT;
  std::vector<Record> recs;
  const bsg_status st = make_records(*w, &recs);
  if (st != BSG_OK) return st;
  for (size_t i = 0; i < recs.size(); ++i) {
    prompt[i] = recs[i].prompt;
    output[i] = recs[i].output;
    est[i] = recs[i].est;
    arrival_ticks[i] = recs[i].arrival;
  }
  return BSG_OK;
}

bsg_status bsg_make_trace(const bsg_workload* w, bsg_trace_record* out) {
  if (!w || (!out && w->count > 0) || w->count < 0) return BSG_INVALID_ARGUMENT;
  const std::vector<Record> rs = synthetic_trace(*w);
  for (size_t i = 0; i < rs.size(); ++i) {
    out[i] = bsg_trace_record{};
    out[i].id = static_cast<uint64_t>(i);
    out[i].prompt_tokens = rs[i].prompt;
    out[i].output_tokens = rs[i].output;
  }
  return BSG_OK;
}

bsg_status bsg_trace_workload(const bsg_trace_record* recs, int64_t n, const bsg_workload* w,
                              int32_t* prompt, int32_t* output, int32_t* est,
                              int64_t* arrival_ticks, int64_t* n_out, bsg_trace_error* err) {
  if (!w || !n_out) return BSG_INVALID_ARGUMENT;
  std::vector<Record> rs;
  const bsg_status st = records_from_trace(recs, n, *w, &rs, err);
  if (st != BSG_OK) return st;
  for (size_t i = 0; i < rs.size(); ++i) {
    prompt[i] = rs[i].prompt;
    output[i] = rs[i].output;
    est[i] = rs[i].est;
    arrival_ticks[i] = rs[i].arrival;
  }
  *n_out = static_cast<int64_t>(rs.size());
  return BSG_OK;
}

namespace {
bsg_status replay_records(bsg_ctx* ctx, std::vector<Record> recs, const bsg_instance_cfg* cfg,
                          const bsg_replay_spec* spec, bsg_request_outcome* outcomes,
                          bsg_replay_summary* summary, bsg_capture** capture,
                          bsg_run_report* report = nullptr);
}

bsg_status bsg_replay_trace(bsg_ctx* ctx, const bsg_trace_record* recs, int64_t n,
                            const bsg_workload* w, const bsg_instance_cfg* cfg,
                            const bsg_replay_spec* spec, bsg_request_outcome* outcomes,
                            bsg_replay_summary* summary, bsg_trace_error* err) {
  if (!ctx || !w || !cfg || !spec || spec->n_instances < 1) return BSG_INVALID_ARGUMENT;
  std::vector<Record> rs;
  const bsg_status st = records_from_trace(recs, n, *w, &rs, err);
  if (st != BSG_OK) return st;
  return replay_records(ctx, std::move(rs), cfg, spec, outcomes, summary, nullptr);
}

bsg_status bsg_replay(bsg_ctx* ctx, const bsg_workload* w, const bsg_instance_cfg* cfg,
                      const bsg_replay_spec* spec, bsg_request_outcome* outcomes,
                      bsg_replay_summary* summary, bsg_capture** capture) {
  if (!ctx || !w || !cfg || !spec || spec->n_instances < 1) return BSG_INVALID_ARGUMENT;
  std::vector<Record> recs;
  const bsg_status st = make_records(*w, &recs);
  if (st != BSG_OK) return st;
  return replay_records(ctx, std::move(recs), cfg, spec, outcomes, summary, capture);
}

namespace {
bsg_status replay_records(bsg_ctx* ctx, std::vector<Record> recs, const bsg_instance_cfg* cfg,
                          const bsg_replay_spec* spec, bsg_request_outcome* outcomes,
                          bsg_replay_summary* summary, bsg_capture** capture,
                          bsg_run_report* report) {
  // validate_provision_policy (autoscaler.cpp:23-34) and config.cpp:177-180
  if (spec->provision_kind < 0 || spec->provision_kind > 2 || !(spec->threshold_s > 0) ||
      spec->cold_start_s < 0 || spec->cooldown_s < 0 ||
      (spec->provision_kind != 0 && spec->max_instances < spec->n_instances) ||
      !(spec->dispatch_overhead_s >= 0))  // config.cpp:189-190
    return BSG_BAD_CONFIG;
  int32_t bi = 0, fc = 0;
  bsg_status st = bsg_set_configs(ctx, cfg, 1, &bi, &fc);
  if (st != BSG_OK) return st;
  // Workload must be servable at all (config.cpp:197-205).
  for (const Record& r : recs)
    if (blocks(static_cast<int64_t>(r.prompt) + r.output, cfg->block_size) > cfg->total_blocks)
      return BSG_TOO_LARGE_CANDIDATE;
  std::unique_ptr<bsg_capture> cap(capture ? new bsg_capture() : nullptr);
  Replay replay(ctx, *cfg, *spec, std::move(recs), cap.get());
  st = replay.run();
  if (st != BSG_OK) return st;
  if (outcomes)
    std::memcpy(outcomes, replay.outcomes().data(),
                replay.outcomes().size() * sizeof(bsg_request_outcome));
  if (summary) replay.summary(summary);
  if (report) {  // aggregate (metrics.cpp:21-124) incl. the dispatch-point balance
    bsg_replay_summary sm{};
    replay.summary(&sm);
    bsg_aggregate(replay.outcomes().data(), static_cast<int64_t>(replay.outcomes().size()), &sm, report);
    replay.balance(&report->free_blocks_mean_avg, &report->free_blocks_var_avg);
  }
  if (capture) *capture = cap.release();
  return BSG_OK;
}
}  // namespace

void bsg_capture_sizes(const bsg_capture* c, int64_t* n_entries, int64_t* n_scenarios) {
  *n_entries = static_cast<int64_t>(c->prompt.size());
  *n_scenarios = static_cast<int64_t>(c->scenarios.size());
}

void bsg_capture_copy(const bsg_capture* c, uint64_t* id, int32_t* prompt, int32_t* est,
                      int32_t* prefill, int32_t* decoded, bsg_scenario* scenarios) {
  const size_t n = c->prompt.size();
  if (id) std::memcpy(id, c->id.data(), n * sizeof(uint64_t));
  std::memcpy(prompt, c->prompt.data(), n * sizeof(int32_t));
  std::memcpy(est, c->est.data(), n * sizeof(int32_t));
  std::memcpy(prefill, c->prefill.data(), n * sizeof(int32_t));
  std::memcpy(decoded, c->decoded.data(), n * sizeof(int32_t));
  std::memcpy(scenarios, c->scenarios.data(), c->scenarios.size() * sizeof(bsg_scenario));
}

void bsg_capture_free(bsg_capture* c) { delete c; }

}  // extern "C"

namespace {

// percentile_nearest_rank (metrics.cpp:11-19)
double nearest_rank(std::vector<double> v, double p) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double n = static_cast<double>(v.size());
  std::size_t rank = static_cast<std::size_t>(std::ceil(p / 100.0 * n));
  if (rank < 1) rank = 1;
  if (rank > v.size()) rank = v.size();
  return v[rank - 1];
}

double mean_of(const std::vector<double>& v) {
  if (v.empty()) return 0.0;
  double s = 0;
  for (double x : v) s += x;
  return s / static_cast<double>(v.size());
}

}  // namespace

extern "C" bsg_status bsg_aggregate(const bsg_request_outcome* o, int64_t n,
                                    const bsg_replay_summary* summary, bsg_run_report* out) {
  if (!o || !out || n < 0) return BSG_INVALID_ARGUMENT;
  std::memset(out, 0, sizeof(*out));
  std::vector<double> ttft, e2e, overhead;
  int64_t first_arrival = INT64_MAX, last_finish = INT64_MIN;
  for (int64_t i = 0; i < n; ++i) {
    first_arrival = std::min(first_arrival, o[i].arrival_ticks);
    if (o[i].finish_ticks >= 0 && o[i].dispatch_ticks >= 0 && o[i].first_token_ticks >= 0) {
      ttft.push_back(static_cast<double>(o[i].first_token_ticks - o[i].dispatch_ticks) * 1e-9);
      e2e.push_back(static_cast<double>(o[i].finish_ticks - o[i].arrival_ticks) * 1e-9);
      overhead.push_back(static_cast<double>(o[i].dispatch_ticks - o[i].arrival_ticks) * 1e-9);
      last_finish = std::max(last_finish, o[i].finish_ticks);
      ++out->finished_requests;
    } else {
      ++out->censored_requests;
    }
  }
  out->mean_ttft_s = mean_of(ttft);
  out->p50_ttft_s = nearest_rank(ttft, 50.0);
  out->p99_ttft_s = nearest_rank(ttft, 99.0);
  out->mean_e2e_s = mean_of(e2e);
  out->p50_e2e_s = nearest_rank(e2e, 50.0);
  out->p99_e2e_s = nearest_rank(e2e, 99.0);
  out->mean_overhead_s = mean_of(overhead);
  if (n > 0 && out->finished_requests > 0 && last_finish > first_arrival)
    out->throughput_rps = static_cast<double>(out->finished_requests) /
                          (static_cast<double>(last_finish - first_arrival) * 1e-9);
  if (summary) {
    out->total_preemptions = summary->total_preemptions;
    out->instances_provisioned = summary->instances_provisioned;
    out->final_instance_count = summary->final_instance_count;
  }
  return BSG_OK;
}

namespace {

// One capacity-search point: run_experiment(spec_for_cell(base, policy, qps,
// seed)) (driver.cpp:321-331, 409-414) + aggregate; pass iff p99 TTFT < slo
// (metrics.cpp:145-150).
bsg_status run_point(bsg_ctx* ctx, const bsg_workload* base, const bsg_instance_cfg* cfg,
                     const bsg_replay_spec* spec, uint64_t seed, double qps, double slo,
                     bool* passed) {
  bsg_workload w = *base;
  w.qps = qps;
  w.arrival_seed = seed;
  w.estimator_seed = seed;
  bsg_replay_spec sp = *spec;
  sp.policy_seed = seed;
  sp.capture = 0;
  const int32_t n = (w.request_cap >= 0 && w.request_cap < w.count) ? w.request_cap : w.count;
  std::vector<bsg_request_outcome> o(static_cast<size_t>(n));
  bsg_replay_summary summ{};
  const bsg_status st = bsg_replay(ctx, &w, cfg, &sp, o.data(), &summ, nullptr);
  if (st != BSG_OK) return st;
  bsg_run_report rep{};
  bsg_aggregate(o.data(), n, &summ, &rep);
  *passed = rep.p99_ttft_s < slo;
  return BSG_OK;
}

// capacity_search's decision logic (metrics.cpp:151-177) given the integer
// results; returns the tenths to test (empty when bracket_pass == qps_max).
std::vector<double> capacity_bracket(const std::vector<bool>& integer_pass, int32_t qps_min,
                                     int32_t qps_max, bsg_capacity_result* out) {
  int last = 0;
  while (last + 1 < static_cast<int>(integer_pass.size()) && integer_pass[last + 1]) ++last;
  out->monotone = 1;
  for (int i = last + 1; i < static_cast<int>(integer_pass.size()); ++i)
    if (integer_pass[i]) out->monotone = 0;
  out->bracket_pass = qps_min + last;
  out->bracket_fail = out->bracket_pass + 1;
  out->capacity_qps = static_cast<double>(out->bracket_pass);
  std::vector<double> tenths;
  if (out->bracket_pass < qps_max)
    for (int tenth = 1; tenth <= 9; ++tenth)
      tenths.push_back(static_cast<double>(out->bracket_pass * 10 + tenth) / 10.0);
  return tenths;
}

}  // namespace

extern "C" bsg_status bsg_capacity_search(bsg_ctx* ctx, const bsg_workload* base,
                                          const bsg_instance_cfg* cfg, const bsg_replay_spec* spec,
                                          uint64_t seed, int32_t qps_min, int32_t qps_max,
                                          double slo_p99_ttft_s, bsg_capacity_result* out,
                                          double* tested_qps, int32_t* tested_pass,
                                          int32_t tested_cap) {
  if (!ctx || !base || !cfg || !spec || !out) return BSG_INVALID_ARGUMENT;
  if (qps_min > qps_max) return BSG_BAD_CONFIG;  // metrics.cpp:141
  std::memset(out, 0, sizeof(*out));
  auto record = [&](double qps, bool ok) {
    if (out->n_tested < tested_cap) {
      if (tested_qps) tested_qps[out->n_tested] = qps;
      if (tested_pass) tested_pass[out->n_tested] = ok ? 1 : 0;
    }
    ++out->n_tested;
  };
  std::vector<bool> integer_pass;
  for (int32_t q = qps_min; q <= qps_max; ++q) {
    bool ok = false;
    const bsg_status st = run_point(ctx, base, cfg, spec, seed, q, slo_p99_ttft_s, &ok);
    if (st != BSG_OK) return st;
    record(q, ok);
    integer_pass.push_back(ok);
  }
  if (!integer_pass.front()) return BSG_NO_CAPACITY;  // metrics.cpp:153-155
  const std::vector<double> tenths = capacity_bracket(integer_pass, qps_min, qps_max, out);
  for (double qps : tenths) {
    bool ok = false;
    const bsg_status st = run_point(ctx, base, cfg, spec, seed, qps, slo_p99_ttft_s, &ok);
    if (st != BSG_OK) return st;
    record(qps, ok);
    if (ok) out->capacity_qps = std::max(out->capacity_qps, qps);
  }
  return BSG_OK;
}

namespace {

// Runs closed-loop points (cell, qps) as device-resident closed loops
// (bsg_replay_device, one thread block per point) and reports pass/fail per
// point: p99 TTFT < slo (metrics.cpp:145-150). Records are generated on
// `threads` host threads; points are launched longest-first.
struct Point {
  int32_t cell;
  double qps;
};
bsg_status run_points_device(bsg_ctx* ctx, const bsg_sweep_cell* cells, const std::vector<Point>& pts,
                             int32_t threads, std::vector<int8_t>* passed, std::vector<int32_t>* status,
                             std::vector<int64_t>* whatifs) {
  const size_t np = pts.size();
  passed->assign(np, 0);
  status->assign(np, BSG_OK);
  whatifs->assign(np, 0);
  if (np == 0) return BSG_OK;
  std::vector<std::vector<Record>> recs(np);
  std::vector<int32_t> gen_err(np, BSG_OK);
  {
    std::atomic<size_t> next{0};
    auto work = [&]() {
      for (size_t i; (i = next.fetch_add(1)) < np;) {
        bsg_workload w = cells[pts[i].cell].workload;
        w.qps = pts[i].qps;  // spec_for_cell (driver.cpp:321-331)
        w.arrival_seed = cells[pts[i].cell].seed;
        w.estimator_seed = cells[pts[i].cell].seed;
        gen_err[i] = make_records(w, &recs[i]);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  // longest first: blocks are dispatched in index order
  std::vector<size_t> order(np);
  for (size_t i = 0; i < np; ++i) order[i] = i;
  auto cost = [&](size_t i) {
    const double ni = cells[pts[i].cell].spec.n_instances;
    return static_cast<double>(recs[i].size()) * ni * (1.0 + pts[i].qps / ni);
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost(a) > cost(b); });
  std::vector<bsg_closed_loop_run> runs;
  std::vector<size_t> run_pt;
  std::vector<int32_t> p, o, e;
  std::vector<int64_t> t;
  for (size_t i : order) {
    if (gen_err[i] != BSG_OK) {
      (*status)[i] = gen_err[i];
      continue;
    }
    const bsg_sweep_cell& c = cells[pts[i].cell];
    runs.push_back(bsg_closed_loop_run{c.spec.n_instances, c.spec.objective, pts[i].cell,
                                       static_cast<int32_t>(recs[i].size()), static_cast<int64_t>(p.size()),
                                       c.spec.provision_kind, c.spec.max_instances, c.spec.threshold_s,
                                       c.spec.cold_start_s, c.spec.cooldown_s, c.spec.policy, 0,
                                       c.seed /* spec_for_cell: policy seed = seed */,
                                       c.spec.dispatch_overhead_s});
    run_pt.push_back(i);
    for (const Record& r : recs[i]) {
      p.push_back(r.prompt);
      o.push_back(r.output);
      e.push_back(r.est);
      t.push_back(r.arrival);
    }
  }
  // the runs are aggregated on the device (metric pipeline): only their reports come back
  std::vector<bsg_run_report> reps(runs.size());
  std::vector<int32_t> rst(runs.size(), BSG_OK);
  const bsg_status st = bsg_replay_device(ctx, runs.data(), static_cast<int32_t>(runs.size()), p.data(),
                                          o.data(), e.data(), t.data(), static_cast<int64_t>(p.size()),
                                          nullptr, nullptr, rst.data(), reps.data());
  if (st != BSG_OK) return st;
  for (size_t r = 0; r < runs.size(); ++r) {
    const size_t i = run_pt[r];
    (*status)[i] = rst[r];
    (*whatifs)[i] = static_cast<int64_t>(runs[r].n_instances) * runs[r].n_requests;
    if (rst[r] != BSG_OK) continue;
    (*passed)[i] = reps[r].p99_ttft_s < cells[pts[i].cell].slo_p99_ttft_s ? 1 : 0;  // metrics.cpp:145
  }
  return BSG_OK;
}

// bsg_sweep_run on device-resident closed loops: every cell must be a
// BlockPredictive cluster of <= 256 instances (any provisioning kind).
bsg_status sweep_device(int device, const bsg_sweep_cell* cells, int32_t n_cells, int32_t threads,
                        bsg_sweep_out* out) {
  bsg_ctx* ctx = nullptr;
  bsg_status st = bsg_ctx_create(device, &ctx);
  if (st != BSG_OK) return st;
  std::unique_ptr<bsg_ctx, void (*)(bsg_ctx*)> guard(ctx, bsg_ctx_destroy);
  std::vector<bsg_instance_cfg> cfgs(static_cast<size_t>(n_cells));
  for (int32_t c = 0; c < n_cells; ++c) cfgs[c] = cells[c].cfg;
  int32_t bi = 0, fc = 0;
  st = bsg_set_configs(ctx, cfgs.data(), n_cells, &bi, &fc);
  if (st != BSG_OK) return st;
  std::vector<int> err(n_cells, BSG_OK);
  std::vector<std::vector<int8_t>> ipass(n_cells);
  std::vector<double> wall(n_cells, 0.0);
  std::vector<int64_t> scen(n_cells, 0);
  auto phase = [&](const std::vector<Point>& pts, std::vector<int8_t>* passed) -> bsg_status {
    std::vector<int32_t> pst;
    std::vector<int64_t> wi;
    const auto t0 = std::chrono::steady_clock::now();
    const bsg_status s = run_points_device(ctx, cells, pts, threads, passed, &pst, &wi);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (s != BSG_OK) return s;
    for (size_t i = 0; i < pts.size(); ++i) {
      if (pst[i] != BSG_OK) err[pts[i].cell] = pst[i];
      scen[pts[i].cell] += wi[i];
    }
    for (int32_t c = 0; c < n_cells; ++c) wall[c] += dt;  // cells share the batched launch
    return BSG_OK;
  };
  std::vector<Point> pts;
  for (int32_t c = 0; c < n_cells; ++c) {
    std::memset(&out[c], 0, sizeof(out[c]));
    if (cells[c].qps_min > cells[c].qps_max) {
      err[c] = BSG_BAD_CONFIG;
      continue;
    }
    for (int32_t q = cells[c].qps_min; q <= cells[c].qps_max; ++q) pts.push_back(Point{c, static_cast<double>(q)});
  }
  std::vector<int8_t> passed;
  st = phase(pts, &passed);
  if (st != BSG_OK) return st;
  for (size_t i = 0; i < pts.size(); ++i) ipass[pts[i].cell].push_back(passed[i]);
  std::vector<Point> tpts;
  std::vector<std::vector<double>> tenths(n_cells);
  for (int32_t c = 0; c < n_cells; ++c) {
    if (err[c] != BSG_OK) continue;
    std::vector<bool> ip(ipass[c].begin(), ipass[c].end());
    if (!ip.front()) {
      err[c] = BSG_NO_CAPACITY;
      continue;
    }
    tenths[c] = capacity_bracket(ip, cells[c].qps_min, cells[c].qps_max, &out[c].result);
    for (double q : tenths[c]) tpts.push_back(Point{c, q});
  }
  std::vector<int8_t> tpassed;
  st = phase(tpts, &tpassed);
  if (st != BSG_OK) return st;
  std::vector<int32_t> n_tenths(n_cells, 0);
  for (size_t i = 0; i < tpts.size(); ++i) {
    const int32_t c = tpts[i].cell;
    ++n_tenths[c];
    if (tpassed[i]) out[c].result.capacity_qps = std::max(out[c].result.capacity_qps, tpts[i].qps);
  }
  for (int32_t c = 0; c < n_cells; ++c) {
    out[c].status = err[c];
    out[c].whatif_scenarios = scen[c];
    out[c].kernel_launches = 2;
    out[c].wall_s = wall[c];
    out[c].result.n_tested = static_cast<int32_t>(ipass[c].size()) + n_tenths[c];
  }
  return BSG_OK;
}

}  // namespace

extern "C" bsg_status bsg_sweep_run(int device, const bsg_sweep_cell* cells, int32_t n_cells,
                                    int32_t threads, bsg_sweep_out* out) {
  if (!cells || !out || n_cells < 0) return BSG_INVALID_ARGUMENT;
  {
    bool device_ok = n_cells > 0 && std::getenv("BSG_SWEEP_HOST") == nullptr;
    for (int32_t c = 0; c < n_cells && device_ok; ++c)
      device_ok = cells[c].spec.n_instances >= 1 && cells[c].spec.n_instances <= 256 &&
                  (cells[c].spec.provision_kind == 0 || cells[c].spec.max_instances <= 256) &&
                  cells[c].cfg.max_batch_size <= 256;
    if (device_ok) return sweep_device(device, cells, n_cells, threads, out);
  }
  // Every closed loop of every cell is independent, so schedule at (cell, qps)
  // granularity: phase 1 runs all integer points, phase 2 the tenths of each
  // cell's bracket. The per-cell result is then assembled exactly as
  // capacity_search would report it (same tested order and decisions).
  struct Task {
    int32_t cell;
    double qps;
    int32_t slot;  // index into the cell's result vector
  };
  std::vector<std::vector<int8_t>> ipass(n_cells), tpass(n_cells);
  std::vector<std::vector<double>> tenths(n_cells);
  std::vector<std::atomic<int64_t>> scen(n_cells), launches(n_cells);
  std::vector<std::atomic<int64_t>> nanos(n_cells);
  std::vector<int> err(n_cells, BSG_OK);
  for (int32_t c = 0; c < n_cells; ++c) {
    std::memset(&out[c], 0, sizeof(out[c]));
    if (cells[c].qps_min > cells[c].qps_max) err[c] = BSG_BAD_CONFIG;
    ipass[c].assign(std::max(0, cells[c].qps_max - cells[c].qps_min + 1), -1);
    scen[c] = 0;
    launches[c] = 0;
    nanos[c] = 0;
  }
  std::atomic<int> fatal{BSG_OK};
  // Closed loops are host-bound between GPU dispatches: oversubscribing the
  // cores with spin-waiting threads stalls everything, so cap the pool at the
  // hardware threads and let waiting threads yield (BSG_SCHED overrides).
  threads = std::min<int32_t>(threads, std::max(1u, std::thread::hardware_concurrency()));
  {
    const char* sched = std::getenv("BSG_SCHED");
    unsigned flags = cudaDeviceScheduleYield;
    if (sched && std::string(sched) == "spin") flags = cudaDeviceScheduleSpin;
    if (sched && std::string(sched) == "block") flags = cudaDeviceScheduleBlockingSync;
    if (sched && std::string(sched) == "auto") flags = cudaDeviceScheduleAuto;
    cudaSetDevice(device);
    if (cudaSetDeviceFlags(flags) != cudaSuccess) cudaGetLastError();  // context already active
  }
  auto run_tasks = [&](std::vector<Task>& tasks, bool tenth_phase) {
    // longest first: more instances and higher qps mean longer closed loops
    std::stable_sort(tasks.begin(), tasks.end(), [&](const Task& a, const Task& b) {
      const double ca = cells[a.cell].spec.n_instances * a.qps;
      const double cb = cells[b.cell].spec.n_instances * b.qps;
      return ca > cb;
    });
    std::atomic<size_t> next{0};
    const int nt = std::max(1, std::min<int>(threads, static_cast<int>(tasks.size())));
    auto worker = [&]() {
      bsg_ctx* ctx = nullptr;
      const bsg_status cs = bsg_ctx_create(device, &ctx);
      if (cs != BSG_OK) {
        fatal = cs;
        return;
      }
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= tasks.size()) break;
        const Task& t = tasks[i];
        const bsg_sweep_cell& c = cells[t.cell];
        const int64_t s0 = bsg_scenario_count(ctx), l0 = bsg_launch_count(ctx);
        const auto t0 = std::chrono::steady_clock::now();
        bool ok = false;
        const bsg_status st =
            run_point(ctx, &c.workload, &c.cfg, &c.spec, c.seed, t.qps, c.slo_p99_ttft_s, &ok);
        const int64_t dt = std::chrono::duration_cast<std::chrono::nanoseconds>(
                               std::chrono::steady_clock::now() - t0).count();
        nanos[t.cell] += dt;
        if (std::getenv("BSG_SWEEP_TRACE"))
          std::fprintf(stderr, "task cell=%d inst=%d qps=%.1f ms=%.1f scen=%lld\n", t.cell,
                       c.spec.n_instances, t.qps, dt * 1e-6,
                       static_cast<long long>(bsg_scenario_count(ctx) - s0));
        scen[t.cell] += bsg_scenario_count(ctx) - s0;
        launches[t.cell] += bsg_launch_count(ctx) - l0;
        if (st != BSG_OK) {
          if (std::getenv("BSG_SWEEP_TRACE"))
            std::fprintf(stderr, "task cell=%d qps=%.1f failed: status %d (%s)\n", t.cell, t.qps,
                         static_cast<int>(st), bsg_last_error(ctx));
          err[t.cell] = st;
          continue;
        }
        (tenth_phase ? tpass : ipass)[t.cell][t.slot] = ok ? 1 : 0;
      }
      bsg_ctx_destroy(ctx);
    };
    std::vector<std::thread> pool;
    for (int k = 0; k < nt; ++k) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  };
  std::vector<Task> tasks;
  for (int32_t c = 0; c < n_cells; ++c)
    if (err[c] == BSG_OK)
      for (int32_t q = cells[c].qps_min; q <= cells[c].qps_max; ++q)
        tasks.push_back(Task{c, static_cast<double>(q), q - cells[c].qps_min});
  run_tasks(tasks, false);
  if (fatal != BSG_OK) return static_cast<bsg_status>(fatal.load());
  tasks.clear();
  for (int32_t c = 0; c < n_cells; ++c) {
    if (err[c] != BSG_OK) continue;
    std::vector<bool> ip(ipass[c].begin(), ipass[c].end());
    if (!ip.front()) {
      err[c] = BSG_NO_CAPACITY;
      continue;
    }
    tenths[c] = capacity_bracket(ip, cells[c].qps_min, cells[c].qps_max, &out[c].result);
    tpass[c].assign(tenths[c].size(), -1);
    for (size_t j = 0; j < tenths[c].size(); ++j)
      tasks.push_back(Task{c, tenths[c][j], static_cast<int32_t>(j)});
  }
  run_tasks(tasks, true);
  if (fatal != BSG_OK) return static_cast<bsg_status>(fatal.load());
  for (int32_t c = 0; c < n_cells; ++c) {
    bsg_sweep_out& o = out[c];
    o.whatif_scenarios = scen[c];
    o.kernel_launches = launches[c];
    o.wall_s = static_cast<double>(nanos[c]) * 1e-9;  // summed closed-loop time
    o.result.n_tested = static_cast<int32_t>(ipass[c].size() + tpass[c].size());
    o.status = err[c];
    if (err[c] != BSG_OK) continue;
    for (size_t j = 0; j < tenths[c].size(); ++j)
      if (tpass[c][j] == 1) o.result.capacity_qps = std::max(o.result.capacity_qps, tenths[c][j]);
  }
  return BSG_OK;
}

// ---- run_sweep / run_capacity (driver.cpp:333-427) ------------------------------
namespace {

bool fits_device(const bsg_instance_cfg& cfg, const bsg_replay_spec& sp) {
  return sp.n_instances >= 1 && sp.n_instances <= 256 &&
         (sp.provision_kind == 0 || sp.max_instances <= 256) && cfg.max_batch_size <= 256;
}

// spec_for_cell (driver.cpp:321-331): policy, its seed, the workload's qps and
// arrival seed, and the estimator's seed.
void apply_cell(bsg_workload* w, bsg_replay_spec* sp, int32_t policy, double qps, uint64_t seed) {
  w->qps = qps;
  w->arrival_seed = seed;
  w->estimator_seed = seed;
  sp->policy = policy;
  sp->policy_seed = seed;
  sp->capture = 0;
}

// Independent run_experiment points, each aggregated (metrics.cpp:21-124):
// device-resident closed loops (batched launches of bounded arena) when every
// point fits K5, else host closed loops on `threads` threads.
bsg_status run_reports(int device, const bsg_instance_cfg& cfg, const std::vector<bsg_workload>& ws,
                       const std::vector<bsg_replay_spec>& sps, int32_t threads,
                       std::vector<int32_t>* status, std::vector<bsg_run_report>* reps) {
  const size_t np = ws.size();
  status->assign(np, BSG_OK);
  reps->assign(np, bsg_run_report{});
  if (np == 0) return BSG_OK;
  bool device_ok = std::getenv("BSG_SWEEP_HOST") == nullptr;
  for (const bsg_replay_spec& sp : sps) device_ok = device_ok && fits_device(cfg, sp);
  threads = std::max<int32_t>(1, threads);
  if (!device_ok) {
    std::atomic<size_t> next{0};
    std::atomic<int> fatal{BSG_OK};
    auto worker = [&]() {
      bsg_ctx* ctx = nullptr;
      const bsg_status cs = bsg_ctx_create(device, &ctx);
      if (cs != BSG_OK) {
        fatal = cs;
        return;
      }
      for (size_t i; (i = next.fetch_add(1)) < np;) {
        std::vector<Record> recs;
        bsg_status st = make_records(ws[i], &recs);
        if (st == BSG_OK) {
          const size_t n = recs.size();
          std::vector<bsg_request_outcome> o(n);
          bsg_replay_summary sm{};
          st = replay_records(ctx, std::move(recs), &cfg, &sps[i], o.data(), &sm, nullptr, &(*reps)[i]);
        }
        (*status)[i] = st;
      }
      bsg_ctx_destroy(ctx);
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::min<int>(threads, static_cast<int>(np)); ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return static_cast<bsg_status>(fatal.load());
  }
  bsg_ctx* ctx = nullptr;
  bsg_status st = bsg_ctx_create(device, &ctx);
  if (st != BSG_OK) return st;
  std::unique_ptr<bsg_ctx, void (*)(bsg_ctx*)> guard(ctx, bsg_ctx_destroy);
  int32_t bi = 0, fc = 0;
  st = bsg_set_configs(ctx, &cfg, 1, &bi, &fc);
  if (st != BSG_OK) return st;
  std::vector<std::vector<Record>> recs(np);
  std::vector<int32_t> gen_err(np, BSG_OK);
  {
    std::atomic<size_t> next{0};
    auto work = [&]() {
      for (size_t i; (i = next.fetch_add(1)) < np;) gen_err[i] = make_records(ws[i], &recs[i]);
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::min<int>(threads, static_cast<int>(np)); ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  // longest first (blocks are dispatched in index order); launches of bounded arena
  std::vector<size_t> order;
  for (size_t i = 0; i < np; ++i) {
    if (gen_err[i] != BSG_OK) (*status)[i] = gen_err[i];
    else order.push_back(i);
  }
  auto cost = [&](size_t i) {
    const double ni = sps[i].n_instances;
    return static_cast<double>(recs[i].size()) * ni * (1.0 + ws[i].qps / ni);
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost(a) > cost(b); });
  size_t o0 = 0;
  while (o0 < order.size()) {
    std::vector<bsg_closed_loop_run> runs;
    std::vector<int32_t> p, o, e;
    std::vector<int64_t> t;
    int64_t arena = 0;
    size_t o1 = o0;
    for (; o1 < order.size(); ++o1) {
      const size_t i = order[o1];
      const bsg_replay_spec& sp = sps[i];
      const int64_t slots = sp.provision_kind == 0 ? sp.n_instances : sp.max_instances;
      const int64_t need = slots * (2 * static_cast<int64_t>(cfg.max_batch_size) + static_cast<int64_t>(recs[i].size()));
      if (o1 > o0 && arena + need >= (int64_t{1} << 30)) break;
      arena += need;
      runs.push_back(bsg_closed_loop_run{sp.n_instances, sp.objective, 0, static_cast<int32_t>(recs[i].size()),
                                         static_cast<int64_t>(p.size()), sp.provision_kind, sp.max_instances,
                                         sp.threshold_s, sp.cold_start_s, sp.cooldown_s, sp.policy, 0,
                                         sp.policy_seed, sp.dispatch_overhead_s});
      for (const Record& r : recs[i]) {
        p.push_back(r.prompt);
        o.push_back(r.output);
        e.push_back(r.est);
        t.push_back(r.arrival);
      }
    }
    std::vector<bsg_run_report> rr(runs.size());
    std::vector<int32_t> rs(runs.size(), BSG_OK);
    st = bsg_replay_device(ctx, runs.data(), static_cast<int32_t>(runs.size()), p.data(), o.data(), e.data(),
                           t.data(), static_cast<int64_t>(p.size()), nullptr, nullptr, rs.data(), rr.data());
    if (st == BSG_BAD_CONFIG || st == BSG_TOO_LARGE_CANDIDATE || st == BSG_BAD_INPUT) {
      // a descriptor-level rejection: attribute it to every run of the batch
      for (size_t q = o0; q < o1; ++q) (*status)[order[q]] = st;
    } else if (st != BSG_OK) {
      return st;
    } else {
      for (size_t q = o0; q < o1; ++q) {
        (*status)[order[q]] = rs[q - o0];
        (*reps)[order[q]] = rr[q - o0];
      }
    }
    o0 = o1;
  }
  return BSG_OK;
}

void format_percent(double fraction, char* out) {  // driver.cpp:392-396
  std::snprintf(out, 16, "%.1f%%", fraction * 100.0);
}

}  // namespace

extern "C" bsg_status bsg_run_sweep(int device, const bsg_workload* base, const bsg_instance_cfg* cfg,
                                    const bsg_replay_spec* spec, const int32_t* policies, int32_t n_policies,
                                    const double* qps_values, int32_t n_qps, const uint64_t* seeds,
                                    int32_t n_seeds, int32_t threads, bsg_sweep_row* rows) {
  if (!base || !cfg || !spec || !rows || n_policies < 0 || n_qps < 0 || n_seeds < 0 ||
      (n_policies && !policies) || (n_qps && !qps_values) || (n_seeds && !seeds))
    return BSG_INVALID_ARGUMENT;
  std::vector<bsg_workload> ws;
  std::vector<bsg_replay_spec> sps;
  for (int32_t a = 0; a < n_policies; ++a) {
    if (policies[a] < BSG_POLICY_RANDOM || policies[a] > BSG_POLICY_BLOCK_PREDICTIVE) return BSG_BAD_CONFIG;
    for (int32_t b = 0; b < n_qps; ++b)
      for (int32_t c = 0; c < n_seeds; ++c) {  // the reference's cell order (driver.cpp:339-345)
        bsg_workload w = *base;
        bsg_replay_spec sp = *spec;
        apply_cell(&w, &sp, policies[a], qps_values[b], seeds[c]);
        ws.push_back(w);
        sps.push_back(sp);
      }
  }
  std::vector<int32_t> st;
  std::vector<bsg_run_report> reps;
  const bsg_status s = run_reports(device, *cfg, ws, sps, threads, &st, &reps);
  if (s != BSG_OK) return s;
  for (size_t i = 0; i < ws.size(); ++i) {
    bsg_sweep_row& r = rows[i];
    std::memset(&r, 0, sizeof(r));
    r.policy = sps[i].policy;
    r.qps = ws[i].qps;
    r.seed = sps[i].policy_seed;
    r.status = st[i];
    r.ok = st[i] == BSG_OK ? 1 : 0;
    if (!r.ok) continue;
    const bsg_run_report& p = reps[i];
    r.mean_ttft_s = p.mean_ttft_s;
    r.p99_ttft_s = p.p99_ttft_s;
    r.mean_e2e_s = p.mean_e2e_s;
    r.p99_e2e_s = p.p99_e2e_s;
    r.throughput_rps = p.throughput_rps;
    r.total_preemptions = p.total_preemptions;
    r.finished_requests = p.finished_requests;
    r.free_blocks_var_avg = p.free_blocks_var_avg;
  }
  return BSG_OK;
}

extern "C" bsg_status bsg_run_capacity(int device, const bsg_workload* base, const bsg_instance_cfg* cfg,
                                       const bsg_replay_spec* spec, const int32_t* policies,
                                       int32_t n_policies, int32_t baseline, uint64_t seed, int32_t qps_min,
                                       int32_t qps_max, double slo_p99_ttft_s, int32_t threads,
                                       bsg_capacity_row* rows, int32_t* n_rows, double* baseline_capacity) {
  if (!base || !cfg || !spec || !rows || !n_rows || n_policies < 0 || (n_policies && !policies))
    return BSG_INVALID_ARGUMENT;
  std::vector<int32_t> pol(policies, policies + n_policies);
  if (std::find(pol.begin(), pol.end(), baseline) == pol.end()) pol.push_back(baseline);
  for (int32_t p : pol)
    if (p < BSG_POLICY_RANDOM || p > BSG_POLICY_BLOCK_PREDICTIVE) return BSG_BAD_CONFIG;
  // one capacity_search cell per policy (driver.cpp:404-416), all batched together
  std::vector<bsg_sweep_cell> cells(pol.size());
  for (size_t i = 0; i < pol.size(); ++i) {
    bsg_sweep_cell& c = cells[i];
    c.workload = *base;
    c.cfg = *cfg;
    c.spec = *spec;
    c.spec.policy = pol[i];
    c.spec.capture = 0;
    c.seed = seed;
    c.qps_min = qps_min;
    c.qps_max = qps_max;
    c.slo_p99_ttft_s = slo_p99_ttft_s;
  }
  std::vector<bsg_sweep_out> out(pol.size());
  const bsg_status st = bsg_sweep_run(device, cells.data(), static_cast<int32_t>(cells.size()), threads, out.data());
  if (st != BSG_OK) return st;
  double base_cap = 0;
  for (size_t i = 0; i < pol.size(); ++i)
    if (pol[i] == baseline && out[i].status == BSG_OK) base_cap = out[i].result.capacity_qps;
  for (size_t i = 0; i < pol.size(); ++i) {
    bsg_capacity_row& r = rows[i];
    std::memset(&r, 0, sizeof(r));
    r.policy = pol[i];
    r.status = out[i].status;
    r.result = out[i].result;
    if (pol[i] != baseline && base_cap > 0 && out[i].status == BSG_OK) {
      r.has_gain = 1;
      r.gain = (r.result.capacity_qps - base_cap) / base_cap;
      format_percent(r.gain, r.gain_text);
    }
  }
  *n_rows = static_cast<int32_t>(pol.size());
  if (baseline_capacity) *baseline_capacity = base_cap;
  return BSG_OK;
}

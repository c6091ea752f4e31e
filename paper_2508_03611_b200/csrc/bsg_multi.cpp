// bsg_multi.cpp — multi-GPU fan-out of the what-if path inside ONE process
// (SURVEY.md §8(e)): one bsg_ctx per device and one persistent host worker
// thread per context, so each GPU's host->device copies, kernels and
// device->host copies run concurrently over its own PCIe / NVLink-C2C link.
//
// The path shards with no data-path collective: scenarios are independent,
// so bsg_multi_predict_batch splits the batch into contiguous ranges (whole
// arrival groups per device, so every request's argmin stays on one GPU), and
// bsg_multi_dispatch splits requests. The latency mode (one Monte-Carlo
// dispatch over many instances, cfg4) splits instances i % n_devices and
// merges the per-device (score, id) minima on the host — exact, lowest id on
// ties (scheduler.cpp:138-150); within one process this is a 16-byte host
// reduction, so NCCL is not involved (bench.py's multi-process mode reduces
// the same packed key with one NCCL MIN).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bsg_internal.h"

namespace {

// A persistent worker thread bound to one context.
struct Worker {
  bsg_ctx* ctx = nullptr;
  int device = 0;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  std::function<void()> job;
  bool has_job = false, done = false, quit = false;

  void run() {
    for (;;) {
      std::function<void()> j;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return has_job || quit; });
        if (quit) return;
        j = std::move(job);
        has_job = false;
      }
      j();
      {
        std::lock_guard<std::mutex> lk(mu);
        done = true;
      }
      cv.notify_all();
    }
  }
  void submit(std::function<void()> j) {
    {
      std::lock_guard<std::mutex> lk(mu);
      job = std::move(j);
      has_job = true;
      done = false;
    }
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return done; });
  }
};

}  // namespace

struct bsg_multi {
  std::vector<Worker*> w;
  std::mutex mu;  // one call at a time
  std::string last_error;
};

namespace {

// Runs fn(d) on every device's worker concurrently; returns the first failure.
bsg_status run_all(bsg_multi* m, const std::function<bsg_status(int)>& fn) {
  const int n = static_cast<int>(m->w.size());
  std::vector<bsg_status> st(static_cast<size_t>(n), BSG_OK);
  for (int d = 1; d < n; ++d) m->w[d]->submit([&, d] { st[d] = fn(d); });
  st[0] = fn(0);  // the calling thread serves device 0
  for (int d = 1; d < n; ++d) m->w[d]->wait();
  for (int d = 0; d < n; ++d) {
    if (st[d] != BSG_OK) {
      m->last_error = "device " + std::to_string(m->w[d]->device) + ": " + bsg_last_error(m->w[d]->ctx);
      return st[d];
    }
  }
  return BSG_OK;
}

// Contiguous shard [lo, hi) of `units` for shard d of n (balanced to +-1).
inline void shard_range(int64_t units, int d, int n, int64_t* lo, int64_t* hi) {
  *lo = units * d / n;
  *hi = units * (d + 1) / n;
}

}  // namespace

extern "C" {

bsg_status bsg_multi_create(const int* devices, int32_t n_devices, bsg_multi** out) {
  if (!devices || n_devices < 1 || !out) return BSG_INVALID_ARGUMENT;
  *out = nullptr;
  auto* m = new bsg_multi();
  for (int32_t d = 0; d < n_devices; ++d) {
    auto* w = new Worker();
    w->device = devices[d];
    const bsg_status st = bsg_ctx_create(devices[d], &w->ctx);
    if (st != BSG_OK) {
      delete w;
      bsg_multi_destroy(m);
      return st;
    }
    m->w.push_back(w);
    if (d > 0) w->th = std::thread([w] { w->run(); });
  }
  *out = m;
  return BSG_OK;
}

void bsg_multi_destroy(bsg_multi* m) {
  if (!m) return;
  for (Worker* w : m->w) {
    if (w->th.joinable()) {
      {
        std::lock_guard<std::mutex> lk(w->mu);
        w->quit = true;
      }
      w->cv.notify_all();
      w->th.join();
    }
    bsg_ctx_destroy(w->ctx);
    delete w;
  }
  delete m;
}

int32_t bsg_multi_device_count(const bsg_multi* m) { return m ? static_cast<int32_t>(m->w.size()) : 0; }

const char* bsg_multi_last_error(const bsg_multi* m) { return m ? m->last_error.c_str() : ""; }

int64_t bsg_multi_launch_count(const bsg_multi* m) {
  int64_t n = 0;
  if (m)
    for (const Worker* w : m->w) n += bsg_launch_count(w->ctx);
  return n;
}

bsg_status bsg_multi_set_configs(bsg_multi* m, const bsg_instance_cfg* cfgs, int32_t n, int32_t* bad_index,
                                 int32_t* field_code) {
  if (!m) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(m->mu);
  for (Worker* w : m->w) {  // validation is identical on every device: the first verdict stands
    const bsg_status st = bsg_set_configs(w->ctx, cfgs, n, bad_index, field_code);
    if (st != BSG_OK) {
      m->last_error = bsg_last_error(w->ctx);
      return st;
    }
  }
  return BSG_OK;
}

bsg_status bsg_multi_predict_batch(bsg_multi* m, const bsg_entries* entries, int64_t n_entries,
                                   const bsg_scenario* scenarios, int64_t n, int32_t group, bsg_result* out) {
  if (!m || !entries || !scenarios || !out || n < 0 || group < 1) return BSG_INVALID_ARGUMENT;
  if (n == 0) return BSG_OK;
  std::lock_guard<std::mutex> lock(m->mu);
  const int nd = static_cast<int>(m->w.size());
  const int64_t groups = (n + group - 1) / group;
  return run_all(m, [&](int d) -> bsg_status {
    int64_t g0, g1;
    shard_range(groups, d, nd, &g0, &g1);
    const int64_t s0 = std::min(n, g0 * group), s1 = std::min(n, g1 * group);
    if (s1 <= s0) return BSG_OK;
    return bsg_predict_batch(m->w[d]->ctx, entries, n_entries, scenarios + s0, s1 - s0, out + s0);
  });
}

bsg_status bsg_multi_dispatch(bsg_multi* m, const bsg_entries* entries, int64_t n_entries,
                              const bsg_scenario* scenarios, const int32_t* instance_ids, int32_t n_inst,
                              int32_t n_requests, int32_t objective, int32_t* chosen, bsg_result* per_instance) {
  if (!m || !entries || !scenarios || !instance_ids || !chosen) return BSG_INVALID_ARGUMENT;
  if (n_inst <= 0) return BSG_NO_INSTANCES;
  if (n_requests <= 0) return BSG_OK;
  std::lock_guard<std::mutex> lock(m->mu);
  const int nd = static_cast<int>(m->w.size());
  return run_all(m, [&](int d) -> bsg_status {
    int64_t r0, r1;
    shard_range(n_requests, d, nd, &r0, &r1);
    if (r1 <= r0) return BSG_OK;
    const int64_t o = r0 * n_inst;
    return bsg_dispatch(m->w[d]->ctx, entries, n_entries, scenarios + o, instance_ids + o, n_inst,
                        static_cast<int32_t>(r1 - r0), objective, chosen + r0,
                        per_instance ? per_instance + o : nullptr);
  });
}

bsg_status bsg_multi_dispatch_mc_sampled(bsg_multi* m, const bsg_entries* entries, int64_t n_entries,
                                         const bsg_scenario* scenarios, const int32_t* instance_ids,
                                         int32_t n_inst, uint64_t request_id, int32_t n_samples, uint64_t seed,
                                         double mean_abs_rel_error, int32_t objective, int32_t* chosen,
                                         int64_t* scores) {
  if (!m || !entries || !scenarios || !instance_ids || !chosen) return BSG_INVALID_ARGUMENT;
  if (n_inst <= 0) return BSG_NO_INSTANCES;
  std::lock_guard<std::mutex> lock(m->mu);
  const int nd = std::min<int>(static_cast<int>(m->w.size()), n_inst);
  // instance i -> device i % nd; each shard's scenarios / ids gathered per device
  struct Shard {
    std::vector<bsg_scenario> sc;
    std::vector<int32_t> ids, at;
    std::vector<int64_t> score;
    int32_t pick = -1;
  };
  std::vector<Shard> sh(static_cast<size_t>(nd));
  for (int32_t i = 0; i < n_inst; ++i) {
    Shard& s = sh[i % nd];
    s.sc.push_back(scenarios[i]);
    s.ids.push_back(instance_ids[i]);
    s.at.push_back(i);
  }
  const std::vector<Worker*> ws(m->w.begin(), m->w.begin() + nd);
  std::vector<bsg_status> st(static_cast<size_t>(nd), BSG_OK);
  auto job = [&](int d) {
    Shard& s = sh[d];
    s.score.assign(s.sc.size(), 0);
    st[d] = bsg_dispatch_mc_sampled(ws[d]->ctx, entries, n_entries, s.sc.data(), s.ids.data(),
                                    static_cast<int32_t>(s.sc.size()), 1, &request_id, n_samples, seed,
                                    mean_abs_rel_error, objective, &s.pick, s.score.data(), nullptr, nullptr,
                                    nullptr);
  };
  for (int d = 1; d < nd; ++d) ws[d]->submit([&, d] { job(d); });
  job(0);
  for (int d = 1; d < nd; ++d) ws[d]->wait();
  for (int d = 0; d < nd; ++d)
    if (st[d] != BSG_OK) {
      m->last_error = "device " + std::to_string(ws[d]->device) + ": " + bsg_last_error(ws[d]->ctx);
      return st[d];
    }
  // exact cross-device argmin: (score, id) lexicographic; a failed shard fails the request
  int64_t best_v = INT64_MAX;
  int32_t best_id = -1;
  bool fail = false;
  for (int d = 0; d < nd; ++d) {
    const Shard& s = sh[d];
    if (s.pick < 0) fail = true;
    for (size_t k = 0; k < s.sc.size(); ++k) {
      if (scores) scores[s.at[k]] = s.score[k];
      const int64_t v = s.score[k];
      if (best_id < 0 || v < best_v || (v == best_v && s.ids[k] < best_id)) {
        best_v = v;
        best_id = s.ids[k];
      }
    }
  }
  *chosen = fail ? -1 : best_id;
  return BSG_OK;
}

}  // extern "C"

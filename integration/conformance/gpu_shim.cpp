// integration/conformance/gpu_shim.cpp — see gpu_shim.h. Compiled WITHOUT the
// shim macros. One GpuPredictorClient per (thread, config template, cache
// mode): the reference's sweep runs cells on several threads, each with its
// own device context.
#include "gpu_shim.h"

#include <atomic>
#include <cstring>
#include <memory>
#include <vector>

#include "blocksim/error.h"
#include "gpu_predictor_client.h"

namespace {

std::atomic<long long> g_calls{0};  // successful GPU predictions

// LatencyCache does not expose its bucket; every cache the reference builds
// in these suites uses the default 256 (predictor.h:50, config.cpp).
blocksim::GpuPredictorClient& client_for(const blocksim::InstanceConfig& c, blocksim::LatencyCache* cache) {
  struct Entry {
    blocksim::InstanceConfig cfg;
    blocksim::CacheMode mode;
    std::unique_ptr<blocksim::GpuPredictorClient> client;
  };
  thread_local std::vector<Entry> pool;
  const blocksim::CacheMode mode = cache ? cache->mode() : blocksim::CacheMode::kOff;
  for (Entry& e : pool) {
    if (e.mode == mode && e.cfg.total_blocks == c.total_blocks && e.cfg.block_size == c.block_size &&
        e.cfg.max_batch_size == c.max_batch_size && e.cfg.chunk_budget == c.chunk_budget &&
        e.cfg.local_policy == c.local_policy && e.cfg.cost_model.c0_s == c.cost_model.c0_s &&
        e.cfg.cost_model.prefill_s_per_token == c.cost_model.prefill_s_per_token &&
        e.cfg.cost_model.decode_s_per_seq == c.cost_model.decode_s_per_seq &&
        e.cfg.cost_model.context_s_per_token == c.cost_model.context_s_per_token)
      return *e.client;
  }
  pool.push_back(Entry{c, mode, std::make_unique<blocksim::GpuPredictorClient>(c, 0, mode, 256)});
  return *pool.back().client;
}

}  // namespace

namespace blocksim {

GpuLocalPredictorClient::GpuLocalPredictorClient(InstanceConfig config_template, LatencyCache* cache)
    : template_(std::move(config_template)), cache_(cache) {}

std::map<InstanceId, PredictionResult> GpuLocalPredictorClient::predict_across(
    const std::vector<InstanceSnapshot>& snapshots, const CandidateRequest& candidate) {
  return bsg_shim::predict_across(snapshots, candidate, template_, cache_);
}

}  // namespace blocksim

namespace bsg_shim {

blocksim::PredictionResult predict(const blocksim::PredictionRequest& request, blocksim::LatencyCache* cache) {
  blocksim::validate_instance_config(request.instance_config);  // before any client exists
  blocksim::PredictionResult r = client_for(request.instance_config, cache).predict(request);
  ++g_calls;
  return r;
}

std::map<blocksim::InstanceId, blocksim::PredictionResult> predict_across(
    const std::vector<blocksim::InstanceSnapshot>& snapshots, const blocksim::CandidateRequest& candidate,
    const blocksim::InstanceConfig& config_template, blocksim::LatencyCache* cache) {
  if (snapshots.empty()) throw blocksim::NoInstancesError("predict_across needs at least one snapshot");
  auto r = client_for(config_template, cache).predict_across(snapshots, candidate);
  ++g_calls;
  return r;
}

long long gpu_calls() { return g_calls.load(); }

}  // namespace bsg_shim

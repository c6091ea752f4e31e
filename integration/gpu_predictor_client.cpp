// integration/gpu_predictor_client.cpp — see gpu_predictor_client.h.
#include "gpu_predictor_client.h"

#include <algorithm>
#include <string>

#include "blocksim/error.h"

namespace blocksim {

namespace {

bsg_instance_cfg to_abi(const InstanceConfig& c, CacheMode cache, TokenCount bucket) {
  bsg_instance_cfg a{};
  a.total_blocks = c.total_blocks;
  a.block_size = c.block_size;
  a.max_batch_size = c.max_batch_size;
  a.chunk_budget = c.chunk_budget;
  a.local_policy = c.local_policy == LocalPolicy::kPrefillPriority ? BSG_PREFILL_PRIORITY
                                                                   : BSG_CHUNKED_PREFILL;
  a.cache_mode = cache == CacheMode::kBucketed ? BSG_CACHE_BUCKETED
                                               : (cache == CacheMode::kExact ? BSG_CACHE_EXACT
                                                                             : BSG_CACHE_OFF);
  a.context_bucket = bucket;
  a.c0_s = c.cost_model.c0_s;
  a.prefill_s_per_token = c.cost_model.prefill_s_per_token;
  a.decode_s_per_seq = c.cost_model.decode_s_per_seq;
  a.context_s_per_token = c.cost_model.context_s_per_token;
  return a;
}

const char* kConfigFields[] = {"",
                               "total_blocks",
                               "block_size",
                               "max_batch_size",
                               "chunk_budget",
                               "cost_model.c0_s",
                               "cost_model.prefill_s_per_token",
                               "cost_model.decode_s_per_seq",
                               "cost_model.context_s_per_token"};
const char* kConfigWhat[] = {"", "must be >= 1", "must be >= 1", "must be >= 1",
                             "must be >= block_size", "must be > 0", "must be >= 0",
                             "must be >= 0", "must be >= 0"};

}  // namespace

GpuPredictorClient::GpuPredictorClient(InstanceConfig config_template, int device,
                                       CacheMode cache, TokenCount context_bucket)
    : template_(std::move(config_template)) {
  // validate_instance_config semantics (types.cpp:47-61) happen on the host
  // before any device work, exactly like the Instance constructor.
  validate_instance_config(template_);
  if (bsg_ctx_create(device, &ctx_) != BSG_OK) {
    ctx_ = nullptr;
    return;  // predict_across will report PredictorUnavailableError
  }
  const bsg_instance_cfg cfg = to_abi(template_, cache, context_bucket);
  int32_t bad = 0, field = 0;
  const bsg_status st = bsg_set_configs(ctx_, &cfg, 1, &bad, &field);
  if (st == BSG_BAD_CONFIG) throw ConfigError(kConfigFields[field], kConfigWhat[field]);
  if (st != BSG_OK) {
    bsg_ctx_destroy(ctx_);
    ctx_ = nullptr;
  }
}

GpuPredictorClient::~GpuPredictorClient() { bsg_ctx_destroy(ctx_); }

std::int64_t GpuPredictorClient::kernel_launches() const { return bsg_launch_count(ctx_); }

std::map<InstanceId, PredictionResult> GpuPredictorClient::predict_across(
    const std::vector<InstanceSnapshot>& snapshots, const CandidateRequest& candidate) {
  if (snapshots.empty()) throw NoInstancesError("predict_across needs at least one snapshot");
  if (ctx_ == nullptr) throw PredictorUnavailableError("no CUDA device for the GPU predictor");
  id_.clear();
  prompt_.clear();
  est_.clear();
  prefill_.clear();
  decoded_.clear();
  scen_.assign(snapshots.size(), bsg_scenario{});
  auto push = [&](const SnapshotRequest& r) {
    id_.push_back(r.id);
    prompt_.push_back(r.prompt_tokens);
    est_.push_back(r.estimated_output_tokens);
    prefill_.push_back(r.prefill_progress);
    decoded_.push_back(r.decoded_tokens);
  };
  for (std::size_t i = 0; i < snapshots.size(); ++i) {
    const InstanceSnapshot& s = snapshots[i];
    bsg_scenario& sc = scen_[i];
    sc.run_off = static_cast<int32_t>(prompt_.size());
    sc.run_n = static_cast<int32_t>(s.running.size());
    for (const auto& r : s.running) push(r);
    sc.wait_off = static_cast<int32_t>(prompt_.size());
    sc.wait_n = static_cast<int32_t>(s.waiting.size());
    for (const auto& r : s.waiting) push(r);
    sc.cand_prompt = candidate.prompt_tokens;
    sc.cand_est = candidate.estimated_output_tokens;
    sc.cfg = 0;
  }
  res_.resize(snapshots.size());
  const bsg_entries e{id_.data(), prompt_.data(), est_.data(), prefill_.data(), decoded_.data()};
  const bsg_status st = bsg_predict_batch(ctx_, &e, static_cast<int64_t>(prompt_.size()),
                                          scen_.data(), static_cast<int64_t>(scen_.size()),
                                          res_.data());
  if (st != BSG_OK) {
    throw PredictorUnavailableError(std::string("GPU predictor failed: ") + bsg_last_error(ctx_));
  }
  std::map<InstanceId, PredictionResult> out;
  for (std::size_t i = 0; i < snapshots.size(); ++i) {
    const InstanceSnapshot& s = snapshots[i];
    const bsg_result& r = res_[i];
    if (r.status != BSG_OK) {
      // Reconstruct the reference's messages (predictor.cpp:103-135, backend.cpp:42-83, 275).
      auto cand_id = [&]() {
        RequestId m = 0;
        for (const auto& x : s.running) m = std::max(m, x.id);
        for (const auto& x : s.waiting) m = std::max(m, x.id);
        return m + 1;
      };
      const std::string tag = "instance " + std::to_string(s.instance_id) + ": ";
      switch (r.status) {
        case BSG_TOO_LARGE_RUNNING:
          throw PredictionError(tag + "candidate does not fit the instance: snapshot running set "
                                      "exceeds total memory blocks");
        case BSG_TOO_LARGE_CANDIDATE:
          throw PredictionError(tag + "candidate does not fit the instance: request " +
                                std::to_string(cand_id()) + " needs " + std::to_string(r.detail) +
                                " blocks, instance has " + std::to_string(template_.total_blocks));
        case BSG_DEADLOCK: {
          const RequestId who =
              r.detail < 0 ? cand_id()
                           : (r.detail < static_cast<int32_t>(s.running.size())
                                  ? s.running[r.detail].id
                                  : s.waiting[r.detail - s.running.size()].id);
          throw PredictionError(tag + "backend deadlock during forward simulation: request " +
                                std::to_string(who) + " cannot proceed with the whole memory free");
        }
        case BSG_STEP_LIMIT:
          throw PredictionError(tag + "forward simulation exceeded the step limit");
        case BSG_VANISHED:
          throw PredictionError(tag + "candidate vanished from the forward simulation");
        case BSG_EMPTY_PLAN:
          throw EmptyPlanError("no runnable work fits the batch");
        case BSG_BAD_INPUT:
          // outside the GPU simulator's integer domain: a prediction
          // failure the caller sees, never a silent switch to the fallback policy
          throw PredictionError(tag + "snapshot outside the GPU simulator's supported domain "
                                      "(prompt <= 2^22, estimate <= 2^24, member capacity <= 256)");
        default:
          throw PredictorUnavailableError("GPU predictor rejected the input (status " +
                                          std::to_string(r.status) + ")");
      }
    }
    PredictionResult pr;
    pr.metrics["predicted_e2e_latency"] = SimTime::from_ticks(r.e2e_ticks).seconds();
    pr.metrics["predicted_ttft"] = SimTime::from_ticks(r.ttft_ticks).seconds();
    pr.metrics["predicted_queueing_delay"] = SimTime::from_ticks(r.qdelay_ticks).seconds();
    pr.simulated_steps = r.steps;
    out[s.instance_id] = std::move(pr);
  }
  return out;
}

}  // namespace blocksim

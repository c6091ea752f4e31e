// integration/gpu_predictor_client.cpp — see gpu_predictor_client.h.
#include "gpu_predictor_client.h"

#include <algorithm>
#include <cstring>
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
    : GpuPredictorClient(std::move(config_template), std::vector<int>{device}, cache, context_bucket) {}

GpuPredictorClient::GpuPredictorClient(InstanceConfig config_template, const std::vector<int>& devices,
                                       CacheMode cache, TokenCount context_bucket)
    : cache_(cache), bucket_(context_bucket), template_(std::move(config_template)) {
  // validate_instance_config semantics (types.cpp:47-61) happen on the host
  // before any device work, exactly like the Instance constructor.
  validate_instance_config(template_);
  bsg_status st = BSG_CUDA_ERROR;
  if (devices.size() > 1) {
    st = bsg_multi_create(devices.data(), static_cast<int32_t>(devices.size()), &multi_);
    if (st != BSG_OK) multi_ = nullptr;
  } else if (!devices.empty()) {
    st = bsg_ctx_create(devices[0], &ctx_);
    if (st != BSG_OK) ctx_ = nullptr;
  }
  if (st != BSG_OK) return;  // predict_across will report PredictorUnavailableError
  if (config_index(template_) < 0) {
    bsg_ctx_destroy(ctx_);
    bsg_multi_destroy(multi_);
    ctx_ = nullptr;
    multi_ = nullptr;
  }
}

GpuPredictorClient::~GpuPredictorClient() {
  bsg_ctx_destroy(ctx_);
  bsg_multi_destroy(multi_);
}

std::int64_t GpuPredictorClient::kernel_launches() const {
  return multi_ ? bsg_multi_launch_count(multi_) : bsg_launch_count(ctx_);
}

int32_t GpuPredictorClient::config_index(const InstanceConfig& c) {
  const bsg_instance_cfg a = to_abi(c, cache_, bucket_);
  for (size_t i = 0; i < cfgs_.size(); ++i)
    if (std::memcmp(&cfgs_[i], &a, sizeof(a)) == 0) return static_cast<int32_t>(i);
  cfgs_.push_back(a);
  int32_t bad = 0, field = 0;
  const bsg_status st = multi_ ? bsg_multi_set_configs(multi_, cfgs_.data(), static_cast<int32_t>(cfgs_.size()),
                                                       &bad, &field)
                               : bsg_set_configs(ctx_, cfgs_.data(), static_cast<int32_t>(cfgs_.size()), &bad,
                                                 &field);
  if (st != BSG_OK) {
    cfgs_.pop_back();
    if (!cfgs_.empty()) {  // restore the registered set
      if (multi_) bsg_multi_set_configs(multi_, cfgs_.data(), static_cast<int32_t>(cfgs_.size()), &bad, &field);
      else bsg_set_configs(ctx_, cfgs_.data(), static_cast<int32_t>(cfgs_.size()), &bad, &field);
    }
    if (st == BSG_BAD_CONFIG) throw ConfigError(kConfigFields[field], kConfigWhat[field]);
    if (st == BSG_BAD_INPUT)
      throw PredictionError("instance config outside the GPU simulator's supported domain "
                            "(total_blocks * block_size <= 2^30, block_size <= 2^20, chunk_budget <= 2^30)");
    return -1;
  }
  return static_cast<int32_t>(cfgs_.size()) - 1;
}

void GpuPredictorClient::pack(const InstanceSnapshot& s, const CandidateRequest& c, int32_t cfg) {
  auto push = [&](const SnapshotRequest& r) {
    id_.push_back(r.id);
    prompt_.push_back(r.prompt_tokens);
    est_.push_back(r.estimated_output_tokens);
    prefill_.push_back(r.prefill_progress);
    decoded_.push_back(r.decoded_tokens);
  };
  bsg_scenario sc{};
  sc.run_off = static_cast<int32_t>(prompt_.size());
  sc.run_n = static_cast<int32_t>(s.running.size());
  for (const auto& r : s.running) push(r);
  sc.wait_off = static_cast<int32_t>(prompt_.size());
  sc.wait_n = static_cast<int32_t>(s.waiting.size());
  for (const auto& r : s.waiting) push(r);
  sc.cand_prompt = c.prompt_tokens;
  sc.cand_est = c.estimated_output_tokens;
  sc.cfg = cfg;
  scen_.push_back(sc);
}

bool GpuPredictorClient::run_batch() {
  res_.resize(scen_.size());
  const bsg_entries e{id_.data(), prompt_.data(), est_.data(), prefill_.data(), decoded_.data()};
  const bsg_status st =
      multi_ ? bsg_multi_predict_batch(multi_, &e, static_cast<int64_t>(prompt_.size()), scen_.data(),
                                       static_cast<int64_t>(scen_.size()), 1, res_.data())
             : bsg_predict_batch(ctx_, &e, static_cast<int64_t>(prompt_.size()), scen_.data(),
                                 static_cast<int64_t>(scen_.size()), res_.data());
  return st == BSG_OK;
}

void GpuPredictorClient::raise(const InstanceSnapshot& s, const bsg_result& r, const std::string& tag,
                               TokenCount total_blocks) const {
  // Reconstruct the reference's messages (predictor.cpp:103-135, backend.cpp:42-83, 275).
  auto cand_id = [&]() {
    RequestId m = 0;
    for (const auto& x : s.running) m = std::max(m, x.id);
    for (const auto& x : s.waiting) m = std::max(m, x.id);
    return m + 1;
  };
  switch (r.status) {
    case BSG_TOO_LARGE_RUNNING:
      throw PredictionError(tag + "candidate does not fit the instance: snapshot running set "
                                  "exceeds total memory blocks");
    case BSG_TOO_LARGE_CANDIDATE:
      throw PredictionError(tag + "candidate does not fit the instance: request " +
                            std::to_string(cand_id()) + " needs " + std::to_string(r.detail) +
                            " blocks, instance has " + std::to_string(total_blocks));
    case BSG_DEADLOCK: {
      const RequestId who = r.detail < 0 ? cand_id()
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
      throw PredictorUnavailableError("GPU predictor rejected the input (status " + std::to_string(r.status) +
                                      ")");
  }
}

namespace {

PredictionResult to_result(const bsg_result& r) {
  PredictionResult pr;
  pr.metrics["predicted_e2e_latency"] = SimTime::from_ticks(r.e2e_ticks).seconds();
  pr.metrics["predicted_ttft"] = SimTime::from_ticks(r.ttft_ticks).seconds();
  pr.metrics["predicted_queueing_delay"] = SimTime::from_ticks(r.qdelay_ticks).seconds();
  pr.simulated_steps = r.steps;
  return pr;
}

}  // namespace

std::map<InstanceId, PredictionResult> GpuPredictorClient::predict_across(
    const std::vector<InstanceSnapshot>& snapshots, const CandidateRequest& candidate) {
  if (snapshots.empty()) throw NoInstancesError("predict_across needs at least one snapshot");
  if (ctx_ == nullptr && multi_ == nullptr) throw PredictorUnavailableError("no CUDA device for the GPU predictor");
  id_.clear();
  prompt_.clear();
  est_.clear();
  prefill_.clear();
  decoded_.clear();
  scen_.clear();
  for (const InstanceSnapshot& s : snapshots) pack(s, candidate, 0);  // config 0: the template
  if (!run_batch()) {
    throw PredictorUnavailableError(std::string("GPU predictor failed: ") +
                                    (multi_ ? bsg_multi_last_error(multi_) : bsg_last_error(ctx_)));
  }
  std::map<InstanceId, PredictionResult> out;
  for (std::size_t i = 0; i < snapshots.size(); ++i) {
    const InstanceSnapshot& s = snapshots[i];
    if (res_[i].status != BSG_OK)
      raise(s, res_[i], "instance " + std::to_string(s.instance_id) + ": ", template_.total_blocks);
    out[s.instance_id] = to_result(res_[i]);
  }
  return out;
}

PredictionResult GpuPredictorClient::predict(const PredictionRequest& request) {
  validate_instance_config(request.instance_config);  // the Instance ctor's check (backend.cpp:16-18)
  if (ctx_ == nullptr && multi_ == nullptr) throw PredictorUnavailableError("no CUDA device for the GPU predictor");
  const int32_t cfg = config_index(request.instance_config);
  if (cfg < 0) throw PredictorUnavailableError("GPU predictor failed to register the instance config");
  id_.clear();
  prompt_.clear();
  est_.clear();
  prefill_.clear();
  decoded_.clear();
  scen_.clear();
  pack(request.snapshot, request.candidate, cfg);
  if (!run_batch()) {
    throw PredictorUnavailableError(std::string("GPU predictor failed: ") +
                                    (multi_ ? bsg_multi_last_error(multi_) : bsg_last_error(ctx_)));
  }
  if (res_[0].status != BSG_OK) raise(request.snapshot, res_[0], "", request.instance_config.total_blocks);
  return to_result(res_[0]);
}

}  // namespace blocksim

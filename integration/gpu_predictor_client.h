// integration/gpu_predictor_client.h — the reference-side binding.
//
// This is the file a blocksim maintainer adds to the reference to route
// BlockPredictive what-if simulation onto a B200: a PredictorClient
// (core/include/blocksim/scheduler.h:53-61) whose predict_across() packs the
// snapshots into the C-ABI's SoA buffers (include/blocksim_b200.h) and runs
// every per-instance predict() in one kernel launch. It is written against the
// reference's own headers and types; Dispatcher::dispatch
// (core/src/scheduler.cpp:115-152) uses it unchanged.
//
// Error behaviour matches LocalPredictorClient -> predict_across
// (core/src/predictor.cpp:139-157): PredictionError messages re-tagged
// "instance N: ..." for the first failing snapshot in input order,
// EmptyPlanError / ConfigError propagate as themselves, NoInstancesError on an
// empty fan-out, and any device failure surfaces as PredictorUnavailableError
// so the Dispatcher's Llumnix- fallback engages (scheduler.cpp:129-136). A
// snapshot outside the GPU simulator's integer domain is a PredictionError
// (it propagates out of dispatch), never a silent fallback.
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "blocksim/predictor.h"
#include "blocksim/scheduler.h"
#include "blocksim_b200.h"

namespace blocksim {

class GpuPredictorClient : public PredictorClient {
 public:
  // cache: kOff / kExact price exactly (the exact cache is transparent,
  // predictor.cpp:43-47); kBucketed rounds the context like LatencyCache.
  explicit GpuPredictorClient(InstanceConfig config_template, int device = 0,
                              CacheMode cache = CacheMode::kExact, TokenCount context_bucket = 256);
  // Fan-out over several GPUs of the box (bsg_multi_*: one context + host
  // worker thread per device; a fan-out's snapshots are split across them).
  GpuPredictorClient(InstanceConfig config_template, const std::vector<int>& devices,
                     CacheMode cache = CacheMode::kExact, TokenCount context_bucket = 256);
  ~GpuPredictorClient() override;
  GpuPredictorClient(const GpuPredictorClient&) = delete;
  GpuPredictorClient& operator=(const GpuPredictorClient&) = delete;

  std::map<InstanceId, PredictionResult> predict_across(
      const std::vector<InstanceSnapshot>& snapshots, const CandidateRequest& candidate) override;

  // predict() (predictor.cpp:76-137) for the reference's direct callers — preempt
  // provisioning (driver.cpp:204-208) and the predictor role (service.cpp:232):
  // the request's own instance_config, same results and exceptions (PredictionError
  // messages untagged, ConfigError / EmptyPlanError as themselves).
  PredictionResult predict(const PredictionRequest& request);

  std::int64_t kernel_launches() const;

 private:
  // one batch over the packed scenarios; returns false when the device failed
  bool run_batch();
  // the config index of `c` (registered on the device on first use)
  int32_t config_index(const InstanceConfig& c);
  void pack(const InstanceSnapshot& s, const CandidateRequest& c, int32_t cfg);
  // throws the reference's exception for a failed scenario (tag: "instance N: " or "")
  [[noreturn]] void raise(const InstanceSnapshot& s, const bsg_result& r, const std::string& tag,
                          TokenCount total_blocks) const;

  bsg_ctx* ctx_ = nullptr;
  bsg_multi* multi_ = nullptr;
  CacheMode cache_ = CacheMode::kExact;
  TokenCount bucket_ = 256;
  std::vector<bsg_instance_cfg> cfgs_;
  InstanceConfig template_;
  std::vector<std::uint64_t> id_;
  std::vector<std::int32_t> prompt_, est_, prefill_, decoded_;
  std::vector<bsg_scenario> scen_;
  std::vector<bsg_result> res_;
};

}  // namespace blocksim

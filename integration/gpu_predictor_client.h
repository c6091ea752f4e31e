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
  ~GpuPredictorClient() override;
  GpuPredictorClient(const GpuPredictorClient&) = delete;
  GpuPredictorClient& operator=(const GpuPredictorClient&) = delete;

  std::map<InstanceId, PredictionResult> predict_across(
      const std::vector<InstanceSnapshot>& snapshots, const CandidateRequest& candidate) override;

  std::int64_t kernel_launches() const;

 private:
  bsg_ctx* ctx_ = nullptr;
  InstanceConfig template_;
  std::vector<std::uint64_t> id_;
  std::vector<std::int32_t> prompt_, est_, prefill_, decoded_;
  std::vector<bsg_scenario> scen_;
  std::vector<bsg_result> res_;
};

}  // namespace blocksim

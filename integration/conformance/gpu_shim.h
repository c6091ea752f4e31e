// integration/conformance/gpu_shim.h — force-included (g++ -include) into the
// reference's translation units and its own unit tests to run them with the
// GPU predictor in place of the CPU one, without editing a line of either:
//
//   * LocalPredictorClient (scheduler.h:63-75; constructed by SimulationDriver,
//     driver.cpp:29/72) becomes GpuLocalPredictorClient, a PredictorClient over
//     GpuPredictorClient — so every BlockPredictive dispatch and probe of the
//     reference's own driver runs its what-ifs on the B200;
//   * with BSG_SHIM_PREDICT, calls of the free function predict(...)
//     (predictor.h:94; the direct caller driver.cpp:208 and test_predictor.cpp)
//     go to bsg_shim::predict = GpuPredictorClient::predict;
//   * with BSG_SHIM_PREDICT_ACROSS, calls of predict_across(...) (predictor.h)
//     go to the GPU too (test_predictor.cpp only: other TUs name methods so).
//
// The real headers are included first, so their own declarations are parsed
// unchanged; the macros only rewrite later uses.
#pragma once

#include <map>
#include <vector>

#include "blocksim/predictor.h"
#include "blocksim/scheduler.h"

namespace blocksim {

class GpuLocalPredictorClient : public PredictorClient {
 public:
  GpuLocalPredictorClient(InstanceConfig config_template, LatencyCache* cache);
  std::map<InstanceId, PredictionResult> predict_across(const std::vector<InstanceSnapshot>& snapshots,
                                                        const CandidateRequest& candidate) override;

 private:
  InstanceConfig template_;
  LatencyCache* cache_;
};

}  // namespace blocksim

namespace bsg_shim {

blocksim::PredictionResult predict(const blocksim::PredictionRequest& request,
                                   blocksim::LatencyCache* cache = nullptr);
std::map<blocksim::InstanceId, blocksim::PredictionResult> predict_across(
    const std::vector<blocksim::InstanceSnapshot>& snapshots, const blocksim::CandidateRequest& candidate,
    const blocksim::InstanceConfig& config_template, blocksim::LatencyCache* cache = nullptr);
// GPU predictions served so far (all threads) — the run proves the GPU path ran.
long long gpu_calls();

}  // namespace bsg_shim

#define LocalPredictorClient GpuLocalPredictorClient
#ifdef BSG_SHIM_PREDICT
#define predict(...) ::bsg_shim::predict(__VA_ARGS__)
#endif
#ifdef BSG_SHIM_PREDICT_ACROSS
#define predict_across(...) ::bsg_shim::predict_across(__VA_ARGS__)
#endif

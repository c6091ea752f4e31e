// integration/dispatch_parity_main.cpp — the reference's own Dispatcher
// (core/src/scheduler.cpp:115-152) driven by GpuPredictorClient versus the
// reference's LocalPredictorClient (scheduler.h:63-75), on the reference's own
// fixtures (acceptance C11, test_scheduler.cpp:178-214, test_predictor.cpp)
// and on captured closed-loop snapshots. Predictions must be equal as doubles,
// decisions identical, and errors of the same type with the same message.
// Exit code 0 iff every check passes. Built by integration/Makefile against
// the reference headers and the reference compiled in oracle/_ref.
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "blocksim/backend.h"
#include "blocksim/predictor.h"
#include "blocksim/error.h"
#include "blocksim/scheduler.h"
#include "blocksim/workload.h"
#include "gpu_predictor_client.h"

using namespace blocksim;

namespace {

int g_fail = 0, g_pass = 0;

void check(bool ok, const std::string& what) {
  if (ok) {
    ++g_pass;
  } else {
    ++g_fail;
    std::printf("FAIL %s\n", what.c_str());
  }
}

InstanceConfig reference_config() {
  InstanceConfig cfg;
  cfg.total_blocks = 1056;
  cfg.block_size = 16;
  cfg.max_batch_size = 48;
  cfg.chunk_budget = 512;
  return cfg;
}

InstanceSnapshot snapshot_with(InstanceId id, std::vector<SnapshotRequest> running,
                               std::vector<SnapshotRequest> waiting) {
  InstanceSnapshot s;
  s.instance_id = id;
  s.batch_size = static_cast<int>(running.size());
  std::int64_t held = 0;
  for (const auto& r : running) held += blocks_needed(r.prefill_progress + r.decoded_tokens, 16);
  s.free_blocks = static_cast<int>(1056 - held);
  s.running = std::move(running);
  s.waiting = std::move(waiting);
  return s;
}

bool same(const std::map<InstanceId, PredictionResult>& a,
          const std::map<InstanceId, PredictionResult>& b) {
  if (a.size() != b.size()) return false;
  for (const auto& [id, r] : a) {
    auto it = b.find(id);
    if (it == b.end() || it->second.metrics != r.metrics ||
        it->second.simulated_steps != r.simulated_steps)
      return false;
  }
  return true;
}

// Runs both clients; compares results or the thrown exception (type + what()).
void compare(PredictorClient& gpu, PredictorClient& local, const std::vector<InstanceSnapshot>& s,
             const CandidateRequest& c, const std::string& name) {
  std::string eg, el, tg, tl;
  std::map<InstanceId, PredictionResult> rg, rl;
  auto run = [&](PredictorClient& p, std::map<InstanceId, PredictionResult>& r, std::string& e,
                 std::string& t) {
    try {
      r = p.predict_across(s, c);
    } catch (const PredictionError& x) {
      t = "PredictionError";
      e = x.what();
    } catch (const EmptyPlanError& x) {
      t = "EmptyPlanError";
      e = x.what();
    } catch (const NoInstancesError& x) {
      t = "NoInstancesError";
      e = x.what();
    }
  };
  run(gpu, rg, eg, tg);
  run(local, rl, el, tl);
  check(tg == tl && eg == el, name + ": exception " + tg + " '" + eg + "' vs " + tl + " '" + el + "'");
  check(same(rg, rl), name + ": predictions differ");
  Dispatcher dg({PolicyKind::kBlockPredictive, 0, LatencyObjective::kE2e}, reference_config());
  Dispatcher dl({PolicyKind::kBlockPredictive, 0, LatencyObjective::kE2e}, reference_config());
  if (tg.empty() && !s.empty()) {
    check(dg.dispatch(c, s, &gpu).instance_id == dl.dispatch(c, s, &local).instance_id,
          name + ": decision differs");
    Dispatcher tg2({PolicyKind::kBlockPredictive, 0, LatencyObjective::kTtft}, reference_config());
    Dispatcher tl2({PolicyKind::kBlockPredictive, 0, LatencyObjective::kTtft}, reference_config());
    check(tg2.dispatch(c, s, &gpu).instance_id == tl2.dispatch(c, s, &local).instance_id,
          name + ": ttft decision differs");
  }
}

}  // namespace

int main() {
  const InstanceConfig cfg = reference_config();
  LatencyCache cache;  // the reference default (exact): transparent
  LocalPredictorClient local(cfg, &cache);
  GpuPredictorClient gpu(cfg, 0);

  // acceptance_main.cpp:675-699 — criterion 11 fixtures, candidate (300, 80)
  std::vector<std::vector<InstanceSnapshot>> fixtures;
  fixtures.push_back({snapshot_with(0, {}, {}), snapshot_with(1, {}, {})});
  fixtures.push_back({snapshot_with(0, {{1, 64, 300, 64, 10}, {2, 64, 300, 64, 20}}, {}),
                      snapshot_with(1, {{3, 64, 50, 64, 45}}, {}), snapshot_with(2, {}, {})});
  fixtures.push_back({snapshot_with(0, {{1, 96, 100, 96, 120}}, {{2, 800, 100, 0, 0}}),
                      snapshot_with(1, {{3, 96, 100, 96, 20}}, {{4, 100, 50, 60, 0}})});
  {
    std::vector<SnapshotRequest> big;
    for (RequestId id = 0; id < 40; ++id) big.push_back({id, 128, 260, 128, 40});
    fixtures.push_back({snapshot_with(0, std::move(big), {}), snapshot_with(1, {{50, 64, 400, 64, 5}}, {}),
                        snapshot_with(2, {}, {{60, 4000, 800, 0, 0}})});
  }
  fixtures.push_back({snapshot_with(3, {}, {{9, 900, 300, 0, 0}, {10, 200, 60, 0, 0}}),
                      snapshot_with(7, {{11, 300, 200, 300, 199}}, {})});
  for (std::size_t i = 0; i < fixtures.size(); ++i)
    compare(gpu, local, fixtures[i], {300, 80}, "c11_fixture_" + std::to_string(i));

  // test_scheduler.cpp:178-203 flavour: 12 instances, identical pairs tie -> lowest id
  {
    std::vector<InstanceSnapshot> snaps;
    for (InstanceId id = 0; id < 12; ++id) {
      std::vector<SnapshotRequest> run;
      for (RequestId r = 0; r < static_cast<RequestId>((id * 5) % 12); ++r) run.push_back({r, 64, 200, 64, 20});
      snaps.push_back(snapshot_with(id, run, {}));
    }
    snaps[9] = snapshot_with(9, snaps[4].running, {});
    compare(gpu, local, snaps, {128, 32}, "brute_force_12_with_tie");
    std::vector<InstanceSnapshot> rev(snaps.rbegin(), snaps.rend());
    compare(gpu, local, rev, {128, 32}, "brute_force_12_reversed");
  }
  // error behaviour: candidate too large, running set too large, deadlock, empty fan-out
  compare(gpu, local, {snapshot_with(0, {}, {})}, {16000, 2000}, "too_large_candidate");
  {
    std::vector<SnapshotRequest> run;
    for (RequestId id = 0; id < 40; ++id) run.push_back({id, 512, 600, 512, 20});  // 40*33 > 1056
    compare(gpu, local, {snapshot_with(0, {}, {}), snapshot_with(5, run, {})}, {10, 10},
            "too_large_running_second_instance");
  }
  compare(gpu, local, {snapshot_with(2, {}, {{7, 17000, 10, 0, 0}})}, {10, 10},
          "empty_plan_oversized_waiting_head");
  compare(gpu, local, {}, {10, 10}, "no_instances");

  // captured closed-loop snapshots: replay the reference driver loop for 12
  // instances, 600 requests at 27 QPS, and compare every arrival's fan-out.
  {
    SyntheticTraceSpec t;
    t.count = 600;
    t.seed = 1234;
    const auto records = make_synthetic_trace(t);
    const auto arrivals = generate_arrivals(records, 27.0, 1);
    std::vector<Instance> inst;
    for (int i = 0; i < 12; ++i) {
      InstanceConfig c = cfg;
      c.instance_id = i;
      inst.emplace_back(c);
    }
    // simple fixed-step drive: advance every instance one step between arrivals
    int compared = 0;
    for (std::size_t a = 0; a < arrivals.size(); ++a) {
      std::vector<InstanceSnapshot> snaps;
      for (const auto& in : inst) snaps.push_back(in.snapshot(SimTime::zero()));
      const CandidateRequest c{arrivals[a].record.prompt_tokens, arrivals[a].record.output_tokens};
      Dispatcher dl({PolicyKind::kBlockPredictive, 0, LatencyObjective::kE2e}, cfg);
      const auto d = dl.dispatch(c, snaps, &local);
      if (a % 7 == 0) {
        compare(gpu, local, snaps, c, "replay_arrival_" + std::to_string(a));
        ++compared;
      }
      inst[static_cast<std::size_t>(d.instance_id)].admit(a, c.prompt_tokens, c.estimated_output_tokens,
                                                          c.estimated_output_tokens);
      for (auto& in : inst)
        if (in.has_work()) in.execute_step();
    }
    check(compared > 50, "replay compared enough arrivals");
  }

  // the same fixtures through a client fanning out over several contexts
  // (bsg_multi_*; two contexts on device 0 here: the splitting is under test)
  {
    GpuPredictorClient multi(cfg, std::vector<int>{0, 0});
    for (std::size_t i = 0; i < fixtures.size(); ++i)
      compare(multi, local, fixtures[i], {300, 80}, "multi_c11_fixture_" + std::to_string(i));
    compare(multi, local, {snapshot_with(0, {}, {})}, {16000, 2000}, "multi_too_large_candidate");
  }

  // direct predict() callers (driver.cpp:204-208 preempt provisioning, service.cpp:232):
  // GpuPredictorClient::predict vs the reference predict(), per request config,
  // results and exception messages identical
  {
    auto direct = [&](const PredictionRequest& req, const std::string& name) {
      std::string eg, el, tg, tl;
      PredictionResult rg, rl;
      auto run = [&](const std::function<PredictionResult()>& f, PredictionResult& r, std::string& e,
                     std::string& t) {
        try {
          r = f();
        } catch (const PredictionError& x) {
          t = "PredictionError";
          e = x.what();
        } catch (const EmptyPlanError& x) {
          t = "EmptyPlanError";
          e = x.what();
        } catch (const ConfigError& x) {
          t = "ConfigError";
          e = x.what();
        }
      };
      run([&] { return gpu.predict(req); }, rg, eg, tg);
      run([&] { return predict(req, &cache); }, rl, el, tl);
      check(tg == tl && eg == el, name + ": exception " + tg + " '" + eg + "' vs " + tl + " '" + el + "'");
      check(rg.metrics == rl.metrics && rg.simulated_steps == rl.simulated_steps, name + ": prediction differs");
    };
    int k = 0;
    for (const auto& fx : fixtures)
      for (const auto& snap : fx) {
        PredictionRequest req;
        req.snapshot = snap;
        req.candidate = {300, 80};
        req.instance_config = cfg;
        direct(req, "direct_" + std::to_string(k));
        req.instance_config.total_blocks = 700 + 37 * k;  // a different config per request
        req.instance_config.max_batch_size = 24 + k;
        req.instance_config.local_policy = k % 2 ? LocalPolicy::kPrefillPriority : LocalPolicy::kChunkedPrefill;
        direct(req, "direct_cfg_" + std::to_string(k));
        ++k;
      }
    PredictionRequest bad;
    bad.snapshot = snapshot_with(0, {}, {});
    bad.candidate = {10, 10};
    bad.instance_config = cfg;
    bad.instance_config.chunk_budget = 8;  // < block_size: ConfigError
    direct(bad, "direct_config_error");
    bad.instance_config = cfg;
    bad.candidate = {16000, 2000};
    direct(bad, "direct_too_large");
  }

  // predictor unavailable -> the Dispatcher's own Llumnix- fallback
  {
    GpuPredictorClient down(cfg, 1 << 20);  // no such device
    Dispatcher d({PolicyKind::kBlockPredictive, 0, LatencyObjective::kE2e}, cfg);
    std::vector<InstanceSnapshot> snaps = {snapshot_with(0, {{1, 900, 10, 900, 1}}, {}),
                                           snapshot_with(1, {{2, 100, 10, 100, 1}}, {})};
    const auto dec = d.dispatch({10, 10}, snaps, &down);
    check(dec.used_fallback && d.fallback_count() == 1 && dec.instance_id == 1,
          "unavailable GPU predictor falls back to llumnix-");
  }

  std::printf("dispatch parity: %d passed, %d failed, %lld GPU launches\n", g_pass, g_fail,
              static_cast<long long>(gpu.kernel_launches()));
  return g_fail == 0 ? 0 : 1;
}

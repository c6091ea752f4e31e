// bsg_capi.cu — C-ABI (include/blocksim_b200.h) over the sm_100a kernels.
//
// Host-side responsibilities only: config validation (validate_instance_config,
// types.cpp:47-61), device buffer management, kernel selection by member
// capacity, and stream-ordered launches. No simulation happens on the host;
// without a CUDA device every entry point fails with BSG_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bsg_internal.h"
#include "mc_sampler.cuh"
#include "scenario_sim.cuh"

namespace bsg {

constexpr int kWarpsPerBlock = 4;
// predict_kernel: warps per block (one scenario per warp). Small blocks let
// the block scheduler refill a warp slot as soon as its scenario finishes
// (scenario costs vary ~100x), instead of holding it until the block's
// slowest warp is done.
#ifndef BSG_WPB
#define BSG_WPB 4
#endif
constexpr int kPredictWarps = BSG_WPB;

// Resident-warp target per SM for the 32-member kernels: 28 warps/SM = 72
// registers/thread (measured on cfg2 with the config in the constant bank:
// 28 -> 249 M/s, 32 -> 246.5 M/s); the optimistic narrow passes of wide sets
// keep 32 (64 registers; cfg3 7.44 ms at 28 vs 7.32 ms at 32).
#ifndef BSG_K1_WARPS_PER_SM
#define BSG_K1_WARPS_PER_SM 28
#endif
#ifndef BSG_OPT_WARPS_PER_SM
#define BSG_OPT_WARPS_PER_SM 32
#endif
// ... and for the 64-member kernels: they run small sets (below the queue
// threshold: one wave, bound by the longest scenario) and the optimistic
// passes' retries, so registers beat warps — 16 warps/SM, 119 registers, no
// spills (24 warps: 80 registers, 154/192 B spills): cfg1 200 -> 176 us, cfg3 flat.
#ifndef BSG_K2_WARPS_PER_SM
#define BSG_K2_WARPS_PER_SM 16
#endif
constexpr int min_blocks(int k, bool opt = false) {
  return opt ? BSG_OPT_WARPS_PER_SM / kPredictWarps
             : k == 1 ? BSG_K1_WARPS_PER_SM / kPredictWarps
                      : (k == 2 ? BSG_K2_WARPS_PER_SM / kPredictWarps : 1);
}

// ---- cost-ordered launch (LPT) ----------------------------------------------------
// Scenario costs vary ~100x (a scenario runs until its candidate completes, so
// its step count is ~ the candidate's estimate plus its queueing) and one long
// scenario that starts late is the kernel's tail. Blocks are dispatched in
// index order, so order_kernel counting-sorts the scenarios by cost bucket,
// most expensive first (longest-processing-time order), into a scratch copy of
// the scenario rows whose `reserved` word carries the caller's index;
// predict_kernel's warp w runs sorted row w and writes result `reserved`. The
// copy keeps the row one dependent load away (an index array in between would
// add one more load latency to every scenario's start). Measured with the
// per-scenario timeline (tools/tlprobe.py, cfg2): the round-2 heavy-first list
// (top n/128 only) left a 38 us tail of medium scenarios started late (span
// 220 us, active warps < 90 % of peak for the last 17 %).
constexpr int kCostBuckets = 128;
// A scenario queued behind more than kDeepWait waiting entries admits/preempts
// often, so its pure-decode windows are short: the optimistic pass runs 32-step
// windows when such scenarios are >= 1/4 of the set, 128-step windows otherwise
// (cfg3 8.1 ms with 32 vs 9.6 ms with 128; cfg1 310 vs 238 us).
constexpr int32_t kDeepWait = 8;
// Cost proxy: the candidate's estimate plus BSG_COST_WAIT tokens per waiting
// entry queued ahead of it (cfg2: duration vs cand_est correlation 0.98; cfg1,
// with queues: 0.53 on cand_est alone, 0.83 with 100 per waiting entry).
#ifndef BSG_COST_WAIT
#define BSG_COST_WAIT 250
#endif

__device__ __forceinline__ int cost_bucket(const bsg_scenario& s) {
  const int64_t c = static_cast<int64_t>(max(s.cand_est, 0)) +
                    static_cast<int64_t>(BSG_COST_WAIT) * max(s.wait_n, 0);
  const uint32_t x = static_cast<uint32_t>(c < 0x7ffffffe ? c : 0x7ffffffe) + 1u;
  const int l = 31 - __clz(x);
  const int f = l >= 2 ? static_cast<int>((x >> (l - 2)) & 3u) : static_cast<int>((x << (2 - l)) & 3u);
  return min(4 * l + f, kCostBuckets - 1);
}

// Work-queue state of one launch (zeroed before it), followed in the same
// allocation by bsg_scenario sorted[n] and int32_t retry[n].
struct WorkQueue {
  int32_t arrive;       // order_kernel's grid barrier
  int32_t retry_count;
  int32_t deep_wait, use_wide;  // window-width vote of the optimistic pass
  int32_t hist[kCostBuckets];
  int32_t cursor[kCostBuckets];
};
constexpr size_t kQueueHeader = (sizeof(WorkQueue) + 127) / 128 * 128;
__device__ __forceinline__ bsg_scenario* sorted_rows(WorkQueue* q) {
  return reinterpret_cast<bsg_scenario*>(reinterpret_cast<char*>(q) + kQueueHeader);
}
__device__ __forceinline__ int32_t* retry_list(WorkQueue* q, int64_t n) {
  return reinterpret_cast<int32_t*>(sorted_rows(q) + n);
}

#ifdef BSG_PROFILE_TIMELINE
constexpr int64_t kTimelineCap = 1 << 17;
__device__ uint64_t g_timeline[3 * kTimelineCap];
#endif

// One launch, grid <= one block per SM (all co-resident): bucket histogram,
// one grid barrier, then every block derives the descending bucket offsets and
// scatters its own rows (warp-aggregated cursor atomics; order inside a bucket
// is arbitrary — each row carries its result index). Block 0 also casts the
// optimistic pass's window-width vote.
__global__ void __launch_bounds__(256) order_kernel(const bsg_scenario* __restrict__ sc, int64_t n,
                                                    WorkQueue* q, int32_t force_vote) {
  __shared__ int32_t h[kCostBuckets];
  __shared__ int32_t base[kCostBuckets];
  for (int b = threadIdx.x; b < kCostBuckets; b += blockDim.x) h[b] = 0;
  __syncthreads();
  // contiguous range per block
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t hi = min(n, lo + per);
  int32_t deep = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    atomicAdd(&h[cost_bucket(sc[i])], 1);
    deep += sc[i].wait_n > kDeepWait ? 1 : 0;
  }
  deep = static_cast<int32_t>(__reduce_add_sync(kFull, static_cast<uint32_t>(deep)));
  if ((threadIdx.x & 31) == 0 && deep) atomicAdd(&q->deep_wait, deep);
  __syncthreads();
  for (int b = threadIdx.x; b < kCostBuckets; b += blockDim.x)
    if (h[b]) atomicAdd(&q->hist[b], h[b]);
  // grid barrier (the grid is at most one block per SM, so every block is resident)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&q->arrive, 1);
    while (atomicAdd(&q->arrive, 0) < static_cast<int32_t>(gridDim.x)) __nanosleep(64);
  }
  __syncthreads();
  __threadfence();
  if (threadIdx.x < 32) {
    // exclusive offsets, highest bucket first: 4 buckets per lane
    const int lane = threadIdx.x;
    int32_t c[4], tot = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      c[j] = __ldcg(&q->hist[kCostBuckets - 1 - (lane * 4 + j)]);
      tot += c[j];
    }
    int32_t acc = warp_incl_scan(tot) - tot;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      base[kCostBuckets - 1 - (lane * 4 + j)] = acc;
      acc += c[j];
    }
    if (blockIdx.x == 0 && lane == 0)
      q->use_wide = force_vote >= 0 ? force_vote
                                    : (static_cast<int64_t>(__ldcg(&q->deep_wait)) * 4 < n ? 1 : 0);
  }
  __syncthreads();
  bsg_scenario* out = sorted_rows(q);
  const int lane = threadIdx.x & 31;
  const unsigned lanes_lt = (1u << lane) - 1u;
  for (int64_t i0 = lo + (threadIdx.x & ~31); i0 < hi; i0 += blockDim.x) {
    const int64_t i = i0 + lane;
    const bool in = i < hi;
    bsg_scenario r{};
    int b = -1;
    if (in) {
      r = sc[i];
      b = cost_bucket(r);
    }
    const unsigned peers = __match_any_sync(kFull, b);
    const int leader = __ffs(peers) - 1;
    int32_t pos = 0;
    if (in && lane == leader) pos = atomicAdd(&q->cursor[b], __popc(peers));
    pos = __shfl_sync(kFull, pos, leader);
    if (in) {
      r.reserved = static_cast<int32_t>(i);
      out[base[b] + pos + __popc(peers & lanes_lt)] = r;
    }
  }
}

// One pass of the predict kernels serves the scenarios of ONE instance config,
// passed by value as a __grid_constant__ kernel parameter: its fields stay in
// the constant bank and feed the integer / FP64 instructions as c[][] operands
// instead of occupying ~14 registers for the whole simulation (measured on
// cfg2: spills 172/356 B -> 74/84 B, 222 -> 247 M scenarios/s). Sets that mix
// configs run one pass per config in use; the other scenarios' warps exit at
// once. Returns false when this pass does not own the scenario.
template <int K, bool POW2, bool OPT, int WJ, bool CYC>
__device__ __forceinline__ bool predict_one(const DevCfg& cfg, int32_t cfg_sel, int32_t ncfg,
                                            const int32_t* __restrict__ prompt,
                                            const int32_t* __restrict__ est,
                                            const int32_t* __restrict__ prefill,
                                            const int32_t* __restrict__ decoded,
                                            const bsg_scenario& sc, int32_t* smem,
                                            bsg_result* __restrict__ o) {
  if (sc.cfg < 0 || sc.cfg >= ncfg) {  // every pass writes the same verdict
    if ((threadIdx.x & 31) == 0) {
      bsg_result r{};
      r.status = BSG_INVALID_ARGUMENT;
      *o = r;
    }
    return false;
  }
  if (sc.cfg != cfg_sel) return false;
  const int32_t need = max(sc.run_n, min(cfg.max_batch_size, sc.run_n + sc.wait_n + 1));
  if ((!OPT && need > 32 * K) || sc.run_n < 0 || sc.wait_n < 0) {
    if ((threadIdx.x & 31) == 0) {
      bsg_result r{};
      r.status = BSG_BAD_INPUT;
      *o = r;
    }
    return false;
  }
  // One window width per kernel (a second instantiation costs more in spills
  // than it saves): 128-step windows for 32-member sets, 32-step windows for
  // wide / KV-pressure sets, where admissions and preemptions cut windows short
  // (measured: cfg3 8.1 ms at J=1 vs 9.6 ms at J=4; cfg1 prefers J=4, 238 vs 310 us).
  simulate_scenario<K, false, false, POW2, true, OPT, WJ, CYC>(cfg, prompt, est, prefill, decoded, sc, smem, o,
                                                              TraceSink{nullptr, 0});
  return true;
}

// WJ: event-skipping window width (steps per lane). Measured choices: 128-step
// windows for 32-member sets and for latency-bound small sets (one wave: the
// longest scenario is the critical path), 32-step windows for large wide sets
// and KV pressure, where admissions/preemptions cut windows short.
template <int K, bool POW2, bool OPT, int WJ>
__global__ void __launch_bounds__(kPredictWarps * 32, min_blocks(K, OPT))
    predict_kernel(__grid_constant__ const DevCfg cfg, int32_t cfg_sel, int32_t ncfg,
                   const int32_t* __restrict__ prompt, const int32_t* __restrict__ est,
                   const int32_t* __restrict__ prefill, const int32_t* __restrict__ decoded,
                   const bsg_scenario* __restrict__ scen, int64_t n, WorkQueue* __restrict__ q,
                   bsg_result* __restrict__ out) {
  __shared__ int32_t smem_all[kPredictWarps * smem_words(K, WJ)];
  const int warp = threadIdx.x >> 5;
  int32_t* smem = smem_all + warp * smem_words(K, WJ);
  if constexpr (OPT) {  // two optimistic passes are launched; the vote keeps one
    static_assert(BSG_WIN_J_WIDE != BSG_WIN_J_PREDICT, "the two optimistic passes need distinct widths");
    // use_wide = the vote chose wide (BSG_WIN_J_PREDICT-step) windows; else the
    // BSG_WIN_J_WIDE pass (the width for wide member sets) runs
    if ((__ldcg(&q->use_wide) != 0) != (WJ == BSG_WIN_J_PREDICT)) return;
  }
  // warp w runs the w-th row in cost order (order_kernel), whose result index
  // rides in its reserved word; without a queue, scenario w in caller order
  int64_t w = static_cast<int64_t>(blockIdx.x) * kPredictWarps + warp;
  if (w >= n) return;
  const bsg_scenario sc = q ? sorted_rows(q)[w] : scen[w];
  if (q) w = sc.reserved;
#ifdef BSG_PROFILE_TIMELINE
  uint64_t tl_t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl_t0));
#endif
  // admit / self-preempt cycle absorption (scenario_sim.cuh) only where queues
  // are deep (KV-pressure / wide sets): it costs the 32-member kernel registers
  const bool ran = predict_one<K, POW2, OPT, WJ, (OPT || K >= 2)>(cfg, cfg_sel, ncfg, prompt, est, prefill, decoded, sc,
                                                  smem, out + w);
#ifdef BSG_PROFILE_TIMELINE
  // debug: per-scenario (start, end, SM) on the global timer (tools/tlprobe.py)
  if (ran && (threadIdx.x & 31) == 0 && w < kTimelineCap) {
    uint64_t tl_t1;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl_t1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_timeline[3 * w] = tl_t0;
    g_timeline[3 * w + 1] = tl_t1;
    g_timeline[3 * w + 2] = smid;
  }
#endif
  if constexpr (OPT) {  // too wide for this pass: list it for the wide kernel
    __syncwarp();
    if (ran && (threadIdx.x & 31) == 0 && out[w].status == kStatusRetryWider)
      retry_list(q, n)[atomicAdd(&q->retry_count, 1)] = static_cast<int32_t>(w);
  }
}

// The wide pass over the scenarios the optimistic narrow pass handed back.
template <int K, bool POW2>
__global__ void __launch_bounds__(kPredictWarps * 32, min_blocks(K))
    predict_retry_kernel(__grid_constant__ const DevCfg cfg, int32_t cfg_sel, int32_t ncfg,
                         const int32_t* __restrict__ prompt, const int32_t* __restrict__ est,
                         const int32_t* __restrict__ prefill, const int32_t* __restrict__ decoded,
                         const bsg_scenario* __restrict__ scen, int64_t n, WorkQueue* __restrict__ q,
                         bsg_result* __restrict__ out) {
  __shared__ int32_t smem_all[kPredictWarps * smem_words(K, BSG_WIN_J_WIDE)];
  const int warp = threadIdx.x >> 5;
  int32_t* smem = smem_all + warp * smem_words(K, BSG_WIN_J_WIDE);
  const int32_t cnt = __ldcg(&q->retry_count);
  const int32_t* rl = retry_list(q, n);
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * kPredictWarps + warp; j < cnt;
       j += static_cast<int64_t>(gridDim.x) * kPredictWarps) {
    const int64_t w = __ldcg(&rl[j]);
    const bsg_scenario sc = scen[w];
    predict_one<K, POW2, false, BSG_WIN_J_WIDE, true>(cfg, cfg_sel, ncfg, prompt, est, prefill, decoded, sc, smem,
                                                out + w);
  }
}

template <int K, bool POW2, int WJ, bool CYC>
__global__ void __launch_bounds__(32)
    trace_kernel(const DevCfg* __restrict__ cfgs, const int32_t* __restrict__ prompt,
                 const int32_t* __restrict__ est, const int32_t* __restrict__ prefill,
                 const int32_t* __restrict__ decoded, const bsg_scenario* __restrict__ scen,
                 bsg_result* __restrict__ out, bsg_step_record* rec, int64_t cap) {
  __shared__ int32_t smem[smem_words(K, WJ)];
  const bsg_scenario sc = scen[0];
  const DevCfg cfg = cfgs[sc.cfg];
  simulate_scenario<K, true, false, POW2, true, false, WJ, CYC>(cfg, prompt, est, prefill, decoded, sc, smem,
                                                              out, TraceSink{rec, cap});
}

// BlockPredictive argmin (scheduler.cpp:138-150): one warp per request, value
// compared as int64 ticks (== comparing ticks*1e-9 doubles),
// ties to the lowest instance id. A failing scenario poisons its request.
__global__ void argmin_kernel(const bsg_result* __restrict__ res,
                              const int32_t* __restrict__ inst_ids, int32_t n_inst,
                              int32_t n_req, int32_t objective, int32_t* __restrict__ chosen) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n_req) return;
  const int lane = threadIdx.x & 31;
  int64_t best_v = INT64_MAX;
  int32_t best_id = INT32_MAX;
  bool fail = false;
  for (int32_t i = lane; i < n_inst; i += 32) {
    const bsg_result& x = res[r * n_inst + i];
    const int32_t id = inst_ids[r * n_inst + i];
    if (x.status != BSG_OK) fail = true;
    const int64_t v = objective == 1 ? x.ttft_ticks : x.e2e_ticks;
    if (v < best_v || (v == best_v && id < best_id)) {
      best_v = v;
      best_id = id;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const int64_t ov = __shfl_xor_sync(kFull, best_v, d);
    const int32_t oi = __shfl_xor_sync(kFull, best_id, d);
    if (ov < best_v || (ov == best_v && oi < best_id)) {
      best_v = ov;
      best_id = oi;
    }
  }
  fail = __any_sync(kFull, fail);
  if (lane == 0) chosen[r] = fail ? -1 : best_id;
}

// Per-request MC sampling arguments of the device-sampled dispatch.
struct McSampling {
  const uint64_t* request_id;  // [n_req], nullptr: lengths are given (sorted_len)
  uint64_t seed;
  double scale;                // mean_abs_rel_error * sqrt(pi / 2), computed on the host
  int32_t* lengths_out;        // optional [n_req * S], sample order
};

// Packed cross-GPU argmin key: min(score, 2^47 - 1) << 16 | id,
// -1 when the request failed on this shard (the MIN reduction then fails it).
constexpr int64_t kKeySat = (int64_t{1} << 47) - 1;

// Monte-Carlo BlockPredictive dispatch (cfg4): warp w simulates instance
// w % n_inst of request w / n_inst once, with the request's sorted sample
// lengths staged in shared memory (prefix sharing), and the
// last warp of each request to finish takes the argmin over the per-instance
// scores (sum of per-sample e2e ticks), lowest instance id on ties
// (scheduler.cpp:138-150). SAMPLE: each warp draws the request's S samples
// itself (K3 above, lane-parallel) and bitonic-sorts them in shared memory,
// so sampling is inside the call with no extra launch or host pass.
template <int K, bool POW2, bool SAMPLE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    dispatch_mc_kernel(const DevCfg* __restrict__ cfgs, int32_t ncfg,
                       const int32_t* __restrict__ prompt, const int32_t* __restrict__ est,
                       const int32_t* __restrict__ prefill, const int32_t* __restrict__ decoded,
                       const bsg_scenario* __restrict__ scen, const int32_t* __restrict__ inst_ids,
                       int32_t n_inst, int32_t n_req, const int32_t* __restrict__ sorted_len,
                       int32_t S, int32_t objective, int64_t* __restrict__ scores,
                       int64_t* __restrict__ sample_e2e, bsg_result* __restrict__ res,
                       unsigned* __restrict__ counters, int32_t* __restrict__ chosen,
                       McSampling smp, int64_t* __restrict__ keys) {
  extern __shared__ int32_t dsm[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp;
  if (w >= static_cast<int64_t>(n_inst) * n_req) return;
  const int32_t r = static_cast<int32_t>(w / n_inst);
  const int32_t Sp = SAMPLE ? pow2_ceil(S) : S;
  int32_t* smem = dsm + warp * (smem_words(K, BSG_WIN_J_LATENCY) + Sp);
  int32_t* len = smem + smem_words(K, BSG_WIN_J_LATENCY);
  const bsg_scenario sc = scen[w];
  if constexpr (SAMPLE) {
    stage_mc_samples(len, sc.cand_est, smp.request_id[r], S, smp.seed, smp.scale,
                     (smp.lengths_out && w % n_inst == 0) ? smp.lengths_out + static_cast<int64_t>(r) * S : nullptr);
  } else {
    for (int32_t j = lane; j < S; j += 32) len[j] = sorted_len[static_cast<int64_t>(r) * S + j];
    __syncwarp();
  }
  bsg_result* o = res + w;
  if (sc.cfg < 0 || sc.cfg >= ncfg) {
    if (lane == 0) {
      bsg_result x{};
      x.status = BSG_INVALID_ARGUMENT;
      *o = x;
      scores[w] = INT64_MAX;
    }
  } else {
    const DevCfg cfg = cfgs[sc.cfg];
    const int32_t need = max(sc.run_n, min(cfg.max_batch_size, sc.run_n + sc.wait_n + 1));
    if (need > 32 * K || sc.run_n < 0 || sc.wait_n < 0) {
      if (lane == 0) {
        bsg_result x{};
        x.status = BSG_BAD_INPUT;
        *o = x;
        scores[w] = INT64_MAX;
      }
    } else {
      simulate_scenario<K, false, true, POW2, true, false, BSG_WIN_J_LATENCY, BSG_CYC_LATENCY>(
          cfg, prompt, est, prefill, decoded, sc, smem, o, TraceSink{nullptr, 0},
          McArgs{len, S, sample_e2e ? sample_e2e + w * S : nullptr, scores + w, objective});
    }
  }
  // fused per-request argmin by the last warp to finish
  __threadfence();
  unsigned prev = 0;
  if (lane == 0) prev = atomicAdd(&counters[r], 1u);
  prev = __shfl_sync(kFull, prev, 0);
  if (prev != static_cast<unsigned>(n_inst - 1)) return;
  __threadfence();
  int64_t best_v = INT64_MAX;
  int32_t best_id = INT32_MAX;
  bool fail = false;
  for (int32_t i = lane; i < n_inst; i += 32) {
    const int64_t q = static_cast<int64_t>(r) * n_inst + i;
    const int32_t st = __ldcg(&res[q].status);
    const int64_t v = __ldcg(&scores[q]);
    const int32_t id = inst_ids[q];
    if (st != BSG_OK) fail = true;
    if (v < best_v || (v == best_v && id < best_id)) {
      best_v = v;
      best_id = id;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const int64_t ov = __shfl_xor_sync(kFull, best_v, d);
    const int32_t oi = __shfl_xor_sync(kFull, best_id, d);
    if (ov < best_v || (ov == best_v && oi < best_id)) {
      best_v = ov;
      best_id = oi;
    }
  }
  fail = __any_sync(kFull, fail);
  if (lane == 0) {
    chosen[r] = fail ? -1 : best_id;
    if (keys) keys[r] = fail ? -1 : ((best_v < kKeySat ? best_v : kKeySat) << 16) | best_id;
    counters[r] = 0;  // ready for the next call
  }
}

}  // namespace bsg

using namespace bsg;

#include "bsg_ctx.cuh"

namespace {

bsg_status cuda_fail(bsg_ctx* ctx, cudaError_t e, const char* what) {
  if (ctx) ctx->last_error = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();  // a non-sticky error must not poison the context's next call
  return BSG_CUDA_ERROR;
}

}  // namespace

bsg_status bsg_cuda_fail(bsg_ctx* ctx, cudaError_t e, const char* what) { return cuda_fail(ctx, e, what); }

namespace {

#define BSG_CUDA(ctx, call)                                  \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call); \
  } while (0)

DevCfg to_dev(const bsg_instance_cfg& c) {
  DevCfg d{};
  d.total_blocks = c.total_blocks;
  d.block_size = c.block_size;
  d.max_batch_size = c.max_batch_size;
  d.chunk_budget = c.chunk_budget;
  d.local_policy = c.local_policy;
  d.cache_mode = c.cache_mode;
  d.context_bucket = c.context_bucket;
  const uint32_t bs = static_cast<uint32_t>(c.block_size);
  if ((bs & (bs - 1)) == 0) {
    d.div_magic = 0;
    d.div_shift = __builtin_ctz(bs);
  } else {
    // N = 31-bit dividends: l = ceil(log2 bs), m = floor(2^(31+l)/bs) + 1 < 2^32,
    // q = umulhi(n, m) >> (l - 1).
    int l = 0;
    while ((1u << l) < bs) ++l;
    const unsigned __int128 two = static_cast<unsigned __int128>(1) << (31 + l);
    d.div_magic = static_cast<uint32_t>(two / bs + 1);
    d.div_shift = l - 1;
  }
  d.c0 = c.c0_s;
  d.cp = c.prefill_s_per_token;
  d.cd = c.decode_s_per_seq;
  d.cc = c.context_s_per_token;
  return d;
}

int capacity_k(int32_t need) {
  if (need <= 32) return 1;
  if (need <= 64) return 2;
  if (need <= 128) return 4;
  if (need <= 256) return 8;
  return 0;
}

// The queue path (cost order + optimistic narrow pass + retry) serves wide
// member sets (K > 1) of several waves. 32-member sets (cfg2 shape) and one-wave
// sets run in the caller's order: measured, the cost order's pre-pass costs
// more than it saves there (cfg2 229 us plain vs 249 us LPT-ordered and 243 us
// with round 2's heavy-first list; cfg1 181 vs 186 us) — cand_est misjudges
// scenarios whose candidate waits for KV blocks, and those end up in the tail.
#ifndef BSG_QUEUE_MIN
#define BSG_QUEUE_MIN 8192
#endif

// One pass: the scenarios of config cfg_sel (see predict_one).
template <int K, bool POW2>
bsg_status launch_predict_t(bsg_ctx* ctx, int32_t cfg_sel, int64_t n, const bsg_entries& e,
                            const bsg_scenario* sc, bsg_result* out, cudaStream_t s) {
  static const bool no_queue = std::getenv("BSG_NO_QUEUE") != nullptr;
  const DevCfg& cf = ctx->dev_cfgs_host[cfg_sel];
  const int64_t blocks = (n + kPredictWarps - 1) / kPredictWarps;
  const std::string tp = std::string(POW2 ? "true" : "false");
#ifndef BSG_QUEUE_K1
#define BSG_QUEUE_K1 0  // 1: cost order for 32-member sets too (A/B builds)
#endif
  const bool queue = !no_queue && n >= BSG_QUEUE_MIN && (K > 1 || BSG_QUEUE_K1);
  if (!queue) {
    ctx->last_launch = "predict_kernel<" + std::to_string(K) + "," + tp + ",false," +
                       std::to_string(BSG_WIN_J_PREDICT) + ">";
    predict_kernel<K, POW2, false, BSG_WIN_J_PREDICT><<<static_cast<unsigned>(blocks), kPredictWarps * 32, 0, s>>>(
        cf, cfg_sel, ctx->ncfg, e.prompt, e.est, e.prefill, e.decoded, sc, n, nullptr, out);
    ctx->launches += 1;
    BSG_CUDA(ctx, cudaGetLastError());
    return BSG_OK;
  }
  // stream-ordered scratch: safe for concurrent calls on different streams
  void* mem = nullptr;
  BSG_CUDA(ctx, cudaMallocAsync(&mem, kQueueHeader + n * (sizeof(bsg_scenario) + sizeof(int32_t)), s));
  auto* q = static_cast<WorkQueue*>(mem);
  BSG_CUDA(ctx, cudaMemsetAsync(q, 0, sizeof(WorkQueue), s));
  const int64_t hb = std::min<int64_t>((n + 1023) / 1024, 148);
  // BSG_FORCE_VOTE=0/1 pins the optimistic pass's window-width vote (parity
  // tests run both passes on the same sets); unset: the vote decides
  const char* fv = std::getenv("BSG_FORCE_VOTE");
  const int32_t force_vote = fv ? (std::atoi(fv) != 0 ? 1 : 0) : -1;
  order_kernel<<<static_cast<unsigned>(hb), 256, 0, s>>>(sc, n, q, force_vote);
  const int64_t pb = blocks;
  static const bool no_opt = std::getenv("BSG_NO_OPT") != nullptr;
  if constexpr (K > 1) {
    if (!no_opt) {
      // Optimistic narrow pass: most scenarios' resident lists fit 32 slots even when
      // the batch cap admits more (KV pressure keeps running sets small); the
      // 32-slot kernel runs at 32 warps/SM with half the per-member work, and hands
      // the rest to the wide kernel.
      predict_kernel<1, POW2, true, BSG_WIN_J_PREDICT><<<static_cast<unsigned>(pb), kPredictWarps * 32, 0, s>>>(
          cf, cfg_sel, ctx->ncfg, e.prompt, e.est, e.prefill, e.decoded, sc, n, q, out);
      predict_kernel<1, POW2, true, BSG_WIN_J_WIDE><<<static_cast<unsigned>(pb), kPredictWarps * 32, 0, s>>>(
          cf, cfg_sel, ctx->ncfg, e.prompt, e.est, e.prefill, e.decoded, sc, n, q, out);
      ctx->last_launch = "predict_kernel<1," + tp + ",true," + std::to_string(BSG_WIN_J_PREDICT) + "|" +
                         std::to_string(BSG_WIN_J_WIDE) + "> (vote) + predict_retry_kernel<" +
                         std::to_string(K) + "," + tp + ">";
      const int64_t rb = std::min<int64_t>(pb, 148 * 8);
      predict_retry_kernel<K, POW2><<<static_cast<unsigned>(rb), kPredictWarps * 32, 0, s>>>(
          cf, cfg_sel, ctx->ncfg, e.prompt, e.est, e.prefill, e.decoded, sc, n, q, out);
      ctx->launches += 4;
      BSG_CUDA(ctx, cudaGetLastError());
      BSG_CUDA(ctx, cudaFreeAsync(mem, s));
      return BSG_OK;
    }
  }
  ctx->last_launch = "predict_kernel<" + std::to_string(K) + "," + tp + ",false," +
                     std::to_string(BSG_WIN_J_WIDE) + ">";
  predict_kernel<K, POW2, false, K == 1 ? BSG_WIN_J_PREDICT : BSG_WIN_J_WIDE>
      <<<static_cast<unsigned>(pb), kPredictWarps * 32, 0, s>>>(
      cf, cfg_sel, ctx->ncfg, e.prompt, e.est, e.prefill, e.decoded, sc, n, q, out);
  ctx->launches += 2;
  BSG_CUDA(ctx, cudaGetLastError());
  BSG_CUDA(ctx, cudaFreeAsync(mem, s));
  return BSG_OK;
}

// One pass per config in use (used == nullptr: every config); a pass is
// specialised on its own block size (shift/mask when it is a power of two).
template <int K>
bsg_status launch_predict(bsg_ctx* ctx, int64_t n, const bsg_entries& e, const bsg_scenario* sc,
                          bsg_result* out, cudaStream_t s, const std::vector<uint8_t>* used) {
  bool any = false;
  for (int32_t c = 0; c < ctx->ncfg; ++c) any |= !used || (*used)[c];
  for (int32_t c = 0; c < ctx->ncfg; ++c) {
    if (used && !(*used)[c] && (any || c > 0)) continue;  // >= 1 pass: it writes bad-cfg verdicts
    const bsg_status st = ctx->dev_cfgs_host[c].div_magic == 0
                              ? launch_predict_t<K, true>(ctx, c, n, e, sc, out, s)
                              : launch_predict_t<K, false>(ctx, c, n, e, sc, out, s);
    if (st != BSG_OK) return st;
  }
  return BSG_OK;
}

bsg_status launch_predict_k(bsg_ctx* ctx, int k, int64_t n, const bsg_entries& e,
                            const bsg_scenario* sc, bsg_result* out, cudaStream_t s,
                            const std::vector<uint8_t>* used) {
  if (n == 0) return BSG_OK;
  ctx->scenarios += n;
  switch (k) {
    case 1: return launch_predict<1>(ctx, n, e, sc, out, s, used);
    case 2: return launch_predict<2>(ctx, n, e, sc, out, s, used);
    case 4: return launch_predict<4>(ctx, n, e, sc, out, s, used);
    case 8: return launch_predict<8>(ctx, n, e, sc, out, s, used);
    default:
      ctx->last_error = "member capacity beyond 256 is outside the supported domain";
      return BSG_BAD_INPUT;
  }
}

// Which configs a host scenario set uses (out-of-range indices are skipped).
std::vector<uint8_t> cfgs_used(const bsg_scenario* sc, int64_t n, int32_t ncfg) {
  std::vector<uint8_t> u(static_cast<size_t>(std::max(ncfg, 0)), 0);
  for (int64_t i = 0; i < n; ++i)
    if (sc[i].cfg >= 0 && sc[i].cfg < ncfg) u[sc[i].cfg] = 1;
  return u;
}

int32_t host_need(const bsg_scenario* sc, int64_t n, const std::vector<bsg_instance_cfg>& cfgs) {
  int32_t need = 1;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t c = sc[i].cfg;
    const int32_t maxb = (c >= 0 && c < static_cast<int32_t>(cfgs.size())) ? cfgs[c].max_batch_size : 1;
    const int32_t tot = sc[i].run_n + sc[i].wait_n + 1;
    need = std::max(need, std::max(sc[i].run_n, std::min(maxb, tot)));
  }
  return need;
}

// Every scenario's running / waiting slice must lie inside [0, n_entries): a
// bad offset would otherwise read past a column (silently wrong) or fault the
// device (a sticky error that ends the process's CUDA context).
bsg_status check_ranges(bsg_ctx* ctx, const bsg_scenario* sc, int64_t n, int64_t n_entries) {
  for (int64_t i = 0; i < n; ++i) {
    const bsg_scenario& x = sc[i];
    const bool bad_run = x.run_n > 0 && (x.run_off < 0 || static_cast<int64_t>(x.run_off) + x.run_n > n_entries);
    const bool bad_wait = x.wait_n > 0 && (x.wait_off < 0 || static_cast<int64_t>(x.wait_off) + x.wait_n > n_entries);
    if (bad_run || bad_wait) {
      ctx->last_error = "scenario " + std::to_string(i) + " references entries outside [0, n_entries)";
      return BSG_INVALID_ARGUMENT;
    }
  }
  return BSG_OK;
}

// Uploads host entry columns + scenarios into the context's device buffers.
bsg_status upload(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                  const bsg_scenario* sc, int64_t n, bsg_entries* dev) {
  {
    const bsg_status v = check_ranges(ctx, sc, n, n_entries);
    if (v != BSG_OK) return v;
  }
  const size_t eb = static_cast<size_t>(std::max<int64_t>(n_entries, 1)) * sizeof(int32_t);
  if (!ctx->prompt.ensure(eb) || !ctx->est.ensure(eb) || !ctx->prefill.ensure(eb) ||
      !ctx->decoded.ensure(eb) || !ctx->scen.ensure(n * sizeof(bsg_scenario)) ||
      !ctx->res.ensure(n * sizeof(bsg_result))) {
    ctx->last_error = "device allocation failed";
    return BSG_CUDA_ERROR;
  }
  cudaStream_t s = ctx->stream;
  if (n_entries > 0) {
    BSG_CUDA(ctx, cudaMemcpyAsync(ctx->prompt.p, entries->prompt, n_entries * 4, cudaMemcpyHostToDevice, s));
    BSG_CUDA(ctx, cudaMemcpyAsync(ctx->est.p, entries->est, n_entries * 4, cudaMemcpyHostToDevice, s));
    BSG_CUDA(ctx, cudaMemcpyAsync(ctx->prefill.p, entries->prefill, n_entries * 4, cudaMemcpyHostToDevice, s));
    BSG_CUDA(ctx, cudaMemcpyAsync(ctx->decoded.p, entries->decoded, n_entries * 4, cudaMemcpyHostToDevice, s));
  }
  BSG_CUDA(ctx, cudaMemcpyAsync(ctx->scen.p, sc, n * sizeof(bsg_scenario), cudaMemcpyHostToDevice, s));
  dev->id = nullptr;
  dev->prompt = static_cast<const int32_t*>(ctx->prompt.p);
  dev->est = static_cast<const int32_t*>(ctx->est.p);
  dev->prefill = static_cast<const int32_t*>(ctx->prefill.p);
  dev->decoded = static_cast<const int32_t*>(ctx->decoded.p);
  return BSG_OK;
}

}  // namespace

namespace {
bsg_status dispatch_fused(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                          const bsg_scenario* scenarios, const int32_t* instance_ids,
                          int32_t n_inst, int32_t n_requests, const int32_t* lengths,
                          int32_t n_samples, int32_t objective, int32_t* chosen, int64_t* scores,
                          int64_t* sample_e2e, bsg_result* per_instance,
                          const uint64_t* request_ids, uint64_t seed, double mean_abs_rel_error,
                          int32_t* lengths_out, int64_t* dev_keys);
}  // namespace

extern "C" {

int bsg_abi_version(void) { return BSG_ABI_VERSION; }

double bsg_ticks_to_seconds(int64_t ticks) { return static_cast<double>(ticks) * 1e-9; }

bsg_status bsg_ctx_create(int device, bsg_ctx** out) {
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return BSG_CUDA_ERROR;
  if (device < 0 || device >= count) return BSG_INVALID_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return BSG_CUDA_ERROR;
  auto* ctx = new bsg_ctx();
  ctx->device = device;
  {  // keep stream-ordered scratch allocations cached in the device's pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return BSG_CUDA_ERROR;
  }
  for (int i = 0; i < bsg_ctx::kPipe; ++i) {
    if (cudaStreamCreateWithFlags(&ctx->pipe[i], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->pipe_done[i], cudaEventDisableTiming) != cudaSuccess) {
      delete ctx;
      return BSG_CUDA_ERROR;
    }
  }
  for (int i = 0; i < bsg_ctx::kPieces; ++i) {
    if (cudaEventCreateWithFlags(&ctx->piece_ev[i], cudaEventDisableTiming) != cudaSuccess) {
      delete ctx;
      return BSG_CUDA_ERROR;
    }
  }
  *out = ctx;
  return BSG_OK;
}

void bsg_ctx_destroy(bsg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  for (int i = 0; i < 3; ++i) {
    if (ctx->pipe[i]) {
      cudaStreamSynchronize(ctx->pipe[i]);
      cudaStreamDestroy(ctx->pipe[i]);
    }
    if (ctx->pipe_done[i]) cudaEventDestroy(ctx->pipe_done[i]);
  }
  for (int i = 0; i < bsg_ctx::kPieces; ++i) {
    if (ctx->piece_ev[i]) cudaEventDestroy(ctx->piece_ev[i]);
  }
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  delete ctx;
}

const char* bsg_last_error(const bsg_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

int64_t bsg_launch_count(const bsg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int64_t bsg_scenario_count(const bsg_ctx* ctx) { return ctx ? ctx->scenarios : 0; }

const char* bsg_last_launch(const bsg_ctx* ctx) { return ctx ? ctx->last_launch.c_str() : ""; }

}  // extern "C"

// validate_instance_config (types.cpp:47-61, same check order): BSG_BAD_CONFIG
// with the field code; then the supported integer domain (all
// token sums fit int32): BSG_BAD_INPUT.
bsg_status bsg_check_config(const bsg_instance_cfg& c, int32_t* field_code) {
  int32_t f = 0;
  if (c.total_blocks < 1) f = 1;
  else if (c.block_size < 1) f = 2;
  else if (c.max_batch_size < 1) f = 3;
  else if (c.chunk_budget < c.block_size) f = 4;
  else if (!(c.c0_s > 0)) f = 5;
  else if (c.prefill_s_per_token < 0) f = 6;
  else if (c.decode_s_per_seq < 0) f = 7;
  else if (c.context_s_per_token < 0) f = 8;
  *field_code = f;
  if (f) return BSG_BAD_CONFIG;
  if (static_cast<int64_t>(c.total_blocks) * c.block_size > (1LL << 30) || c.block_size > (1 << 20) ||
      c.chunk_budget > (1 << 30))
    return BSG_BAD_INPUT;
  return BSG_OK;
}

extern "C" {

bsg_status bsg_set_configs(bsg_ctx* ctx, const bsg_instance_cfg* cfgs, int32_t n,
                           int32_t* bad_index, int32_t* field_code) {
  if (!ctx || !cfgs || n <= 0) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  std::vector<DevCfg> dev(n);
  int32_t maxb = 0;
  for (int32_t i = 0; i < n; ++i) {
    const bsg_instance_cfg& c = cfgs[i];
    int32_t f = 0;
    const bsg_status v = bsg_check_config(c, &f);
    if (v != BSG_OK) {
      if (bad_index) *bad_index = i;
      if (field_code) *field_code = f;
      ctx->last_error = v == BSG_BAD_CONFIG ? "invalid config" : "config outside the supported integer domain";
      return v;
    }
    dev[i] = to_dev(c);
    maxb = std::max(maxb, c.max_batch_size);
  }
  if (!ctx->cfgs.ensure(n * sizeof(DevCfg))) return BSG_CUDA_ERROR;
  BSG_CUDA(ctx, cudaMemcpyAsync(ctx->cfgs.p, dev.data(), n * sizeof(DevCfg), cudaMemcpyHostToDevice,
                                ctx->stream));
  BSG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->host_cfgs.assign(cfgs, cfgs + n);
  ctx->dev_cfgs_host = dev;
  ctx->ncfg = n;
  ctx->max_batch_all = maxb;
  ctx->all_pow2 = true;
  for (int32_t i = 0; i < n; ++i) ctx->all_pow2 &= dev[i].div_magic == 0;
  return BSG_OK;
}

bsg_status bsg_predict_batch(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                             const bsg_scenario* scenarios, int64_t n, bsg_result* out) {
  if (!ctx || !entries || !scenarios || !out || n < 0) return BSG_INVALID_ARGUMENT;
  if (ctx->ncfg == 0) return BSG_INVALID_ARGUMENT;
  if (n == 0) return BSG_OK;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  const size_t eb = static_cast<size_t>(std::max<int64_t>(n_entries, 1)) * sizeof(int32_t);
  if (!ctx->prompt.ensure(eb) || !ctx->est.ensure(eb) || !ctx->prefill.ensure(eb) ||
      !ctx->decoded.ensure(eb) || !ctx->scen.ensure(n * sizeof(bsg_scenario)) ||
      !ctx->res.ensure(n * sizeof(bsg_result))) {
    ctx->last_error = "device allocation failed";
    return BSG_CUDA_ERROR;
  }
  bsg_entries dev{};
  dev.prompt = static_cast<const int32_t*>(ctx->prompt.p);
  dev.est = static_cast<const int32_t*>(ctx->est.p);
  dev.prefill = static_cast<const int32_t*>(ctx->prefill.p);
  dev.decoded = static_cast<const int32_t*>(ctx->decoded.p);
  auto* dsc = static_cast<bsg_scenario*>(ctx->scen.p);
  auto* dres = static_cast<bsg_result*>(ctx->res.p);
  // Chunked pipeline: chunk c (a contiguous scenario range) runs as soon as
  // the entry piece holding its last entry has landed, on its own stream, and
  // copies its results back while later pieces are still in flight. The
  // chunks shrink (weights BSG_PIPE_SPLIT, default 3:2:1): the last chunk's
  // kernel — the only one nothing overlaps — is short. Measured on cfg2
  // (tools/e2eprobe.py, one box, median of 40 calls): equal thirds 0.592 ms,
  // 3:2:1 0.557, 2:1 0.566, 4:3:2:1 0.569, 5:4:3:2:1 0.584 (each piece costs
  // four more copy calls), one chunk 0.698.
  std::vector<int64_t> bounds{0};
  {
    std::vector<double> wts;
    if (const char* env_split = std::getenv("BSG_PIPE_SPLIT")) {
      for (const char* q = env_split; *q;) {
        char* end = nullptr;
        const double v = std::strtod(q, &end);
        if (end == q) break;
        if (v > 0) wts.push_back(v);
        q = *end == ',' ? end + 1 : end;
      }
    }
    if (wts.empty()) wts = {3, 2, 1};
    if (static_cast<int>(wts.size()) > bsg_ctx::kPieces) wts.resize(bsg_ctx::kPieces);
    if (n < 16384) wts = {1};  // one wave or two: nothing to overlap
    double tot = 0;
    for (double v : wts) tot += v;
    double acc = 0;
    for (size_t c = 0; c + 1 < wts.size(); ++c) {
      acc += wts[c];
      bounds.push_back(std::min<int64_t>(n, static_cast<int64_t>(static_cast<double>(n) * acc / tot)));
    }
    bounds.push_back(n);
  }
  const int64_t nchunks = static_cast<int64_t>(bounds.size()) - 1;
  // BSG_PIPE_PROFILE=1 (diagnostics): host timestamps and per-chunk CUDA events to stderr
  const bool pipe_prof = std::getenv("BSG_PIPE_PROFILE") != nullptr;
  std::vector<cudaEvent_t> pev;
  std::vector<double> host_us;
  const auto h0 = std::chrono::steady_clock::now();
  auto hnow = [&]() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count(); };
  auto mark = [&](cudaStream_t st) {
    if (!pipe_prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    pev.push_back(e);
    host_us.push_back(hnow());
  };
  mark(ctx->pipe[0]);
  auto cols_h = std::array<const int32_t*, 4>{entries->prompt, entries->est, entries->prefill,
                                              entries->decoded};
  auto cols_d = std::array<int32_t*, 4>{static_cast<int32_t*>(ctx->prompt.p), static_cast<int32_t*>(ctx->est.p),
                                        static_cast<int32_t*>(ctx->prefill.p),
                                        static_cast<int32_t*>(ctx->decoded.p)};
  // The scenario rows and then the entry columns stream in pieces (one per
  // chunk) on pipe[0] from the start of the call — no host scan in front of the
  // first byte; scenario chunk c runs on its own stream pipe[1 + c % 6] once the
  // piece holding its last entry has landed, while the host scans the next
  // chunk (round 2: 0.60 ms vs 0.68 ms for per-chunk copies behind each chunk's
  // scan, BSG_PIPE=1).
  const char* env_pipe = std::getenv("BSG_PIPE");
  const bool v2 = !(env_pipe && std::atoi(env_pipe) == 1);
  const int np = static_cast<int>(nchunks);  // one entry piece per chunk, same fraction
  std::vector<int64_t> pe(np + 1);
  if (v2) {
    // the scenario rows first (1.9 MB at cfg2): every chunk needs its rows before its entries
    BSG_CUDA(ctx, cudaMemcpyAsync(dsc, scenarios, n * sizeof(bsg_scenario), cudaMemcpyHostToDevice,
                                  ctx->pipe[0]));
    for (int k = 0; k <= np; ++k) pe[k] = static_cast<int64_t>(static_cast<double>(n_entries) * bounds[k] / n);
    pe[np] = n_entries;
    for (int k = 0; k < np; ++k) {
      if (pe[k + 1] > pe[k])
        for (int q = 0; q < 4; ++q)
          BSG_CUDA(ctx, cudaMemcpyAsync(cols_d[q] + pe[k], cols_h[q] + pe[k], (pe[k + 1] - pe[k]) * 4,
                                        cudaMemcpyHostToDevice, ctx->pipe[0]));
      BSG_CUDA(ctx, cudaEventRecord(ctx->piece_ev[k], ctx->pipe[0]));
    }
    mark(ctx->pipe[0]);
  }
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t s0 = bounds[c], s1 = bounds[c + 1];
    if (s0 >= s1) continue;
    int64_t lo = INT64_MAX, hi = 0;
    int32_t need = 1;
    std::vector<uint8_t> used(static_cast<size_t>(ctx->ncfg), 0);
    for (int64_t i = s0; i < s1; ++i) {
      const bsg_scenario& x = scenarios[i];
      if (x.cfg >= 0 && x.cfg < ctx->ncfg) used[x.cfg] = 1;
      if (x.run_n > 0) {
        lo = std::min<int64_t>(lo, x.run_off);
        hi = std::max<int64_t>(hi, static_cast<int64_t>(x.run_off) + x.run_n);
      }
      if (x.wait_n > 0) {
        lo = std::min<int64_t>(lo, x.wait_off);
        hi = std::max<int64_t>(hi, static_cast<int64_t>(x.wait_off) + x.wait_n);
      }
      const int32_t cf = x.cfg;
      const int32_t maxb = (cf >= 0 && cf < ctx->ncfg) ? ctx->host_cfgs[cf].max_batch_size : 1;
      need = std::max(need, std::max(x.run_n, std::min(maxb, x.run_n + x.wait_n + 1)));
    }
    if (lo < 0 || hi > n_entries) {
      ctx->last_error = "scenario references entries outside [0, n_entries)";
      return BSG_INVALID_ARGUMENT;
    }
    cudaStream_t st = v2 ? ctx->pipe[1 + c % (bsg_ctx::kPipe - 1)] : ctx->pipe[c % 3];
    if (v2) {
      if (hi > lo) {  // the piece holding entry hi - 1 (pieces land in order)
        int k = 0;
        while (k + 1 < np && pe[k + 1] < hi) ++k;
        BSG_CUDA(ctx, cudaStreamWaitEvent(st, ctx->piece_ev[k], 0));
      }
    } else {
      if (c >= 3) BSG_CUDA(ctx, cudaStreamWaitEvent(st, ctx->pipe_done[c % 3], 0));
      if (hi > lo) {
        for (int q = 0; q < 4; ++q)
          BSG_CUDA(ctx, cudaMemcpyAsync(cols_d[q] + lo, cols_h[q] + lo, (hi - lo) * 4,
                                        cudaMemcpyHostToDevice, st));
      }
    }
    if (!v2)
      BSG_CUDA(ctx, cudaMemcpyAsync(dsc + s0, scenarios + s0, (s1 - s0) * sizeof(bsg_scenario),
                                    cudaMemcpyHostToDevice, st));
    else if (hi <= lo)  // no entries: still after the scenario rows
      BSG_CUDA(ctx, cudaStreamWaitEvent(st, ctx->piece_ev[0], 0));
    mark(st);  // H2D of chunk c done
    const int k = capacity_k(need);
    const bsg_status ls = launch_predict_k(ctx, k == 0 ? 8 : k, s1 - s0, dev, dsc + s0, dres + s0, st, &used);
    if (ls != BSG_OK) return ls;
    mark(st);  // kernels of chunk c done
    BSG_CUDA(ctx, cudaMemcpyAsync(out + s0, dres + s0, (s1 - s0) * sizeof(bsg_result),
                                  cudaMemcpyDeviceToHost, st));
    mark(st);  // D2H of chunk c done
    BSG_CUDA(ctx, cudaEventRecord(ctx->pipe_done[c % 3], st));
  }
  for (int i = 0; i < bsg_ctx::kPipe; ++i) BSG_CUDA(ctx, cudaStreamSynchronize(ctx->pipe[i]));
  if (pipe_prof && v2) {  // the piece copies' completion first, then the chunks
    std::rotate(pev.begin() + 1, pev.begin() + 2, pev.end());
    std::rotate(host_us.begin() + 1, host_us.begin() + 2, host_us.end());
  }
  if (pipe_prof) {
    std::string line = "pipe: host_end " + std::to_string(static_cast<int>(hnow())) + " us;";
    for (size_t i = 1; i < pev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pev[0], pev[i]);
      line += " [c" + std::to_string((i - 1) / 3) + (((i - 1) % 3) == 0 ? " h2d " : ((i - 1) % 3) == 1 ? " ker " : " d2h ") +
              std::to_string(static_cast<int>(ms * 1000)) + " enq@" + std::to_string(static_cast<int>(host_us[i])) + "]";
    }
    std::fprintf(stderr, "%s\n", line.c_str());
    for (cudaEvent_t e : pev) cudaEventDestroy(e);
  }
  return BSG_OK;
}

bsg_status bsg_predict_batch_device(bsg_ctx* ctx, const bsg_entries* dev_entries,
                                    const bsg_scenario* dev_scenarios, int64_t n,
                                    int32_t member_capacity, bsg_result* dev_out, void* stream) {
  if (!ctx || !dev_entries || !dev_scenarios || !dev_out || n < 0) return BSG_INVALID_ARGUMENT;
  if (ctx->ncfg == 0) return BSG_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const int32_t cap = member_capacity > 0 ? member_capacity : std::max(1, ctx->max_batch_all);
  int k = capacity_k(cap);
  if (k == 0) k = 8;
  return launch_predict_k(ctx, k, n, *dev_entries, dev_scenarios, dev_out, s, nullptr);
}

bsg_status bsg_trace(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                     const bsg_scenario* scenario, bsg_step_record* records, int64_t cap,
                     int64_t* n_steps, bsg_result* out) {
  if (!ctx || !entries || !scenario || !out || cap < 0) return BSG_INVALID_ARGUMENT;
  if (ctx->ncfg == 0) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  bsg_entries dev{};
  bsg_status st = upload(ctx, entries, n_entries, scenario, 1, &dev);
  if (st != BSG_OK) return st;
  if (!ctx->rec.ensure(std::max<int64_t>(cap, 1) * sizeof(bsg_step_record))) return BSG_CUDA_ERROR;
  BSG_CUDA(ctx, cudaMemsetAsync(ctx->rec.p, 0, std::max<int64_t>(cap, 1) * sizeof(bsg_step_record),
                                ctx->stream));
  const int k = capacity_k(host_need(scenario, 1, ctx->host_cfgs));
  auto* rec = static_cast<bsg_step_record*>(ctx->rec.p);
  auto* res = static_cast<bsg_result*>(ctx->res.p);
  auto* sc = static_cast<const bsg_scenario*>(ctx->scen.p);
  auto* cf = static_cast<const DevCfg*>(ctx->cfgs.p);
  // the window width under test: the kernels use 1 (wide / KV-pressure sets), 4
  // (32-member sets) and 8 (latency path, no cycle absorption); BSG_TRACE_J picks
  // which per-step trace to emit
  const char* tj = std::getenv("BSG_TRACE_J");
  const int wj = tj ? std::atoi(tj) : 1;
  // BSG_TRACE_CYC=0 traces the windows without admit/self-preempt cycle absorption
  // (the 32-member throughput kernels); default: with it (every other kernel)
  const char* tc = std::getenv("BSG_TRACE_CYC");
  const bool cyc = tc ? std::atoi(tc) != 0 : true;
#define BSG_TRACE_LAUNCH_C(KK, P2, WW)                                                           \
  {                                                                                              \
    if (cyc) trace_kernel<KK, P2, WW, true><<<1, 32, 0, ctx->stream>>>(cf, dev.prompt, dev.est, dev.prefill, dev.decoded, sc, res, rec, cap); \
    else trace_kernel<KK, P2, WW, false><<<1, 32, 0, ctx->stream>>>(cf, dev.prompt, dev.est, dev.prefill, dev.decoded, sc, res, rec, cap); \
  }
#define BSG_TRACE_LAUNCH(KK)                                                                     \
  {                                                                                              \
    if (wj == 8) {                                                                               \
      if (ctx->all_pow2) trace_kernel<KK, true, 8, false><<<1, 32, 0, ctx->stream>>>(cf, dev.prompt, dev.est, dev.prefill, dev.decoded, sc, res, rec, cap); \
      else trace_kernel<KK, false, 8, false><<<1, 32, 0, ctx->stream>>>(cf, dev.prompt, dev.est, dev.prefill, dev.decoded, sc, res, rec, cap); \
    } else if (wj == 4) {                                                                        \
      if (ctx->all_pow2) BSG_TRACE_LAUNCH_C(KK, true, 4) else BSG_TRACE_LAUNCH_C(KK, false, 4)   \
    } else {                                                                                     \
      if (ctx->all_pow2) BSG_TRACE_LAUNCH_C(KK, true, 1) else BSG_TRACE_LAUNCH_C(KK, false, 1)   \
    }                                                                                            \
  }
  switch (k) {
    case 1: BSG_TRACE_LAUNCH(1); break;
    case 2: BSG_TRACE_LAUNCH(2); break;
    case 4: BSG_TRACE_LAUNCH(4); break;
    case 8: BSG_TRACE_LAUNCH(8); break;
    default: ctx->last_error = "member capacity beyond 256"; return BSG_BAD_INPUT;
  }
#undef BSG_TRACE_LAUNCH
#undef BSG_TRACE_LAUNCH_C
  ctx->launches += 1;
  BSG_CUDA(ctx, cudaGetLastError());
  BSG_CUDA(ctx, cudaMemcpyAsync(out, res, sizeof(bsg_result), cudaMemcpyDeviceToHost, ctx->stream));
  BSG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *n_steps = out->steps;
  const int64_t got = std::min<int64_t>(cap, out->steps);
  if (got > 0) {
    BSG_CUDA(ctx, cudaMemcpy(records, rec, got * sizeof(bsg_step_record), cudaMemcpyDeviceToHost));
  }
  return BSG_OK;
}

bsg_status bsg_dispatch(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                        const bsg_scenario* scenarios, const int32_t* instance_ids,
                        int32_t n_inst, int32_t n_requests, int32_t objective, int32_t* chosen,
                        bsg_result* per_instance) {
  if (!ctx || !entries || !scenarios || !instance_ids || !chosen) return BSG_INVALID_ARGUMENT;
  if (n_inst <= 0) return BSG_NO_INSTANCES;  // scheduler.cpp:116
  if (n_requests <= 0) return BSG_OK;
  if (ctx->ncfg == 0) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  // A real fan-out evaluates ONE candidate on every instance: then the fused
  // single-copy path applies (the candidate's estimate is its one "sample").
  bool uniform = true;
  std::vector<int32_t> est(static_cast<size_t>(n_requests));
  for (int32_t r = 0; r < n_requests && uniform; ++r) {
    const bsg_scenario& a = scenarios[static_cast<int64_t>(r) * n_inst];
    est[r] = a.cand_est;
    for (int32_t i = 1; i < n_inst; ++i) {
      const bsg_scenario& b = scenarios[static_cast<int64_t>(r) * n_inst + i];
      if (b.cand_est != a.cand_est || b.cand_prompt != a.cand_prompt) uniform = false;
    }
  }
  if (uniform)
    return dispatch_fused(ctx, entries, n_entries, scenarios, instance_ids, n_inst, n_requests,
                          est.data(), 1, objective, chosen, nullptr, nullptr, per_instance, nullptr, 0,
                          0.0, nullptr, nullptr);
  cudaSetDevice(ctx->device);
  const int64_t n = static_cast<int64_t>(n_inst) * n_requests;
  bsg_entries dev{};
  bsg_status st = upload(ctx, entries, n_entries, scenarios, n, &dev);
  if (st != BSG_OK) return st;
  if (!ctx->ids.ensure(n * sizeof(int32_t)) || !ctx->chosen.ensure(n_requests * sizeof(int32_t)))
    return BSG_CUDA_ERROR;
  BSG_CUDA(ctx, cudaMemcpyAsync(ctx->ids.p, instance_ids, n * sizeof(int32_t),
                                cudaMemcpyHostToDevice, ctx->stream));
  const int k = capacity_k(host_need(scenarios, n, ctx->host_cfgs));
  auto* res = static_cast<bsg_result*>(ctx->res.p);
  const std::vector<uint8_t> used = cfgs_used(scenarios, n, ctx->ncfg);
  st = launch_predict_k(ctx, k == 0 ? 8 : k, n, dev, static_cast<const bsg_scenario*>(ctx->scen.p),
                        res, ctx->stream, &used);
  if (st != BSG_OK) return st;
  const int warps = 4;
  argmin_kernel<<<(n_requests + warps - 1) / warps, warps * 32, 0, ctx->stream>>>(
      res, static_cast<const int32_t*>(ctx->ids.p), n_inst, n_requests, objective,
      static_cast<int32_t*>(ctx->chosen.p));
  ctx->launches += 1;
  BSG_CUDA(ctx, cudaGetLastError());
  BSG_CUDA(ctx, cudaMemcpyAsync(chosen, ctx->chosen.p, n_requests * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, ctx->stream));
  if (per_instance) {
    BSG_CUDA(ctx, cudaMemcpyAsync(per_instance, res, n * sizeof(bsg_result),
                                  cudaMemcpyDeviceToHost, ctx->stream));
  }
  BSG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return BSG_OK;
}

}  // extern "C"

namespace {

// Fused what-if fan-out + argmin with one packed host->device copy: the
// latency path of bsg_dispatch (one "sample" = the candidate's estimate),
// bsg_dispatch_mc (samples given) and bsg_dispatch_mc_sampled (samples drawn
// on the device: request_ids != nullptr, lengths == nullptr). Caller holds ctx->mu.
bsg_status dispatch_fused(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                          const bsg_scenario* scenarios, const int32_t* instance_ids,
                          int32_t n_inst, int32_t n_requests, const int32_t* lengths,
                          int32_t n_samples, int32_t objective, int32_t* chosen, int64_t* scores,
                          int64_t* sample_e2e, bsg_result* per_instance,
                          const uint64_t* request_ids, uint64_t seed, double mean_abs_rel_error,
                          int32_t* lengths_out, int64_t* dev_keys) {
  cudaSetDevice(ctx->device);
  const int64_t n = static_cast<int64_t>(n_inst) * n_requests;
  const int64_t S = n_samples;
  const bool sample = request_ids != nullptr;
  {
    const bsg_status v = check_ranges(ctx, scenarios, n, n_entries);
    if (v != BSG_OK) return v;
  }
  if (dev_keys) {  // the packed key holds 16-bit instance ids
    for (int64_t i = 0; i < n; ++i)
      if (instance_ids[i] < 0 || instance_ids[i] >= 0xffff) {
        ctx->last_error = "instance ids must be in [0, 65535) for the packed cross-GPU key";
        return BSG_INVALID_ARGUMENT;
      }
  }
  // given samples: sort each request's, remembering the permutation for sample_e2e
  std::vector<int32_t> sorted, perm;
  if (!sample) {
    sorted.resize(static_cast<size_t>(n_requests * S));
    perm.resize(static_cast<size_t>(n_requests * S));
    for (int32_t r = 0; r < n_requests; ++r) {
      int32_t* pr = perm.data() + r * S;
      for (int32_t j = 0; j < S; ++j) pr[j] = j;
      const int32_t* lr = lengths + r * S;
      std::stable_sort(pr, pr + S, [&](int32_t a, int32_t b) { return lr[a] < lr[b]; });
      for (int32_t j = 0; j < S; ++j) sorted[r * S + j] = lr[pr[j]];
    }
  }
  // one packed host->device copy: 4 entry columns | scenarios | ids | sorted lengths or request ids
  const size_t ne = static_cast<size_t>(n_entries);
  auto r16 = [](size_t b) { return (b + 15) & ~size_t(15); };
  const size_t tail = sample ? static_cast<size_t>(n_requests) * 8 : sorted.size() * 4;
  const size_t bytes = 4 * r16(ne * 4) + r16(n * sizeof(bsg_scenario)) + r16(n * 4) + r16(tail);
  if (ctx->pinned_cap < bytes) {
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_cap = 0;
    BSG_CUDA(ctx, cudaHostAlloc(&ctx->pinned, bytes * 2, cudaHostAllocDefault));
    ctx->pinned_cap = bytes * 2;
  }
  if (!ctx->blob.ensure(bytes) || !ctx->scores.ensure(n * 8) || !ctx->res.ensure(n * sizeof(bsg_result)) ||
      !ctx->chosen.ensure(n_requests * 4) || !ctx->ids.ensure(4) ||
      (lengths_out && !ctx->samples.ensure(n_requests * S * 4))) {
    ctx->last_error = "device allocation failed";
    return BSG_CUDA_ERROR;
  }
  if (ctx->counters.cap < static_cast<size_t>(n_requests) * 4) {
    if (!ctx->counters.ensure(n_requests * 4)) return BSG_CUDA_ERROR;
    BSG_CUDA(ctx, cudaMemsetAsync(ctx->counters.p, 0, ctx->counters.cap, ctx->stream));
  }
  if (sample_e2e && !ctx->samples.ensure(n * S * 8)) return BSG_CUDA_ERROR;
  char* h = static_cast<char*>(ctx->pinned);
  size_t off = 0;
  auto put = [&](const void* src, size_t b) {
    std::memcpy(h + off, src, b);
    const size_t at = off;
    off += r16(b);
    return at;
  };
  const size_t o_p = put(entries->prompt, ne * 4), o_e = put(entries->est, ne * 4),
               o_f = put(entries->prefill, ne * 4), o_d = put(entries->decoded, ne * 4),
               o_s = put(scenarios, n * sizeof(bsg_scenario)), o_i = put(instance_ids, n * 4),
               o_l = sample ? put(request_ids, tail) : put(sorted.data(), tail);
  BSG_CUDA(ctx, cudaMemcpyAsync(ctx->blob.p, h, off, cudaMemcpyHostToDevice, ctx->stream));
  char* d = static_cast<char*>(ctx->blob.p);
  int32_t cap = 1;
  for (int64_t i = 0; i < n; ++i) {
    const bsg_scenario& sc = scenarios[i];
    const int32_t c = sc.cfg;
    const int32_t maxb = (c >= 0 && c < ctx->ncfg) ? ctx->host_cfgs[c].max_batch_size : 1;
    cap = std::max(cap, std::max(sc.run_n, std::min(maxb, sc.run_n + sc.wait_n + 1)));
  }
  int k = capacity_k(cap);
  if (k == 0) k = 8;
  const int64_t blocks = (n + kWarpsPerBlock - 1) / kWarpsPerBlock;
  auto* dp = reinterpret_cast<const int32_t*>(d + o_p);
  auto* de = reinterpret_cast<const int32_t*>(d + o_e);
  auto* df = reinterpret_cast<const int32_t*>(d + o_f);
  auto* dd = reinterpret_cast<const int32_t*>(d + o_d);
  auto* ds = reinterpret_cast<const bsg_scenario*>(d + o_s);
  auto* di = reinterpret_cast<const int32_t*>(d + o_i);
  auto* dl = reinterpret_cast<const int32_t*>(d + o_l);
  McSampling smp{sample ? reinterpret_cast<const uint64_t*>(d + o_l) : nullptr, seed,
                 mean_abs_rel_error * std::sqrt(3.14159265358979323846 / 2.0),
                 lengths_out ? static_cast<int32_t*>(ctx->samples.p) : nullptr};
  auto* dsc = static_cast<int64_t*>(ctx->scores.p);
  auto* dse = sample_e2e ? static_cast<int64_t*>(ctx->samples.p) : nullptr;
  auto* dres = static_cast<bsg_result*>(ctx->res.p);
  auto* dcnt = static_cast<unsigned*>(ctx->counters.p);
  auto* dch = static_cast<int32_t*>(ctx->chosen.p);
  auto* dcf = static_cast<const DevCfg*>(ctx->cfgs.p);
  const int32_t Sp = sample ? pow2_ceil(n_samples) : n_samples;
#define BSG_LAUNCH_MC2(KK, P2, SM)                                                              \
  {                                                                                             \
    const size_t sm = static_cast<size_t>(kWarpsPerBlock) * (smem_words(KK, BSG_WIN_J_LATENCY) + Sp) * 4; \
    if (sm > 48 * 1024)                                                                         \
      cudaFuncSetAttribute(dispatch_mc_kernel<KK, P2, SM>,                                      \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));  \
    dispatch_mc_kernel<KK, P2, SM><<<static_cast<unsigned>(blocks), kWarpsPerBlock * 32, sm,   \
                                     ctx->stream>>>(dcf, ctx->ncfg, dp, de, df, dd, ds, di,     \
                                                    n_inst, n_requests, dl, n_samples,          \
                                                    objective, dsc, dse, dres, dcnt, dch, smp,  \
                                                    dev_keys);                                  \
  }
#define BSG_LAUNCH_MC1(KK, P2)        \
  if (sample) {                       \
    BSG_LAUNCH_MC2(KK, P2, true)      \
  } else {                            \
    BSG_LAUNCH_MC2(KK, P2, false)     \
  }
#define BSG_LAUNCH_MC(KK)             \
  if (ctx->all_pow2) {                \
    BSG_LAUNCH_MC1(KK, true)          \
  } else {                            \
    BSG_LAUNCH_MC1(KK, false)         \
  }
  switch (k) {
    case 1: BSG_LAUNCH_MC(1); break;
    case 2: BSG_LAUNCH_MC(2); break;
    case 4: BSG_LAUNCH_MC(4); break;
    default: BSG_LAUNCH_MC(8); break;
  }
#undef BSG_LAUNCH_MC
#undef BSG_LAUNCH_MC1
#undef BSG_LAUNCH_MC2
  ctx->launches += 1;
  ctx->scenarios += n * S;
  ctx->last_launch = std::string("dispatch_mc_kernel<") + std::to_string(k) + "," +
                     (ctx->all_pow2 ? "true" : "false") + "," + (sample ? "true" : "false") + ">";
  BSG_CUDA(ctx, cudaGetLastError());
  BSG_CUDA(ctx, cudaMemcpyAsync(chosen, dch, n_requests * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (scores)
    BSG_CUDA(ctx, cudaMemcpyAsync(scores, dsc, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (per_instance)
    BSG_CUDA(ctx, cudaMemcpyAsync(per_instance, dres, n * sizeof(bsg_result), cudaMemcpyDeviceToHost,
                                  ctx->stream));
  if (lengths_out)
    BSG_CUDA(ctx, cudaMemcpyAsync(lengths_out, ctx->samples.p, n_requests * S * 4, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  std::vector<int64_t> tmp;
  if (sample_e2e) {
    tmp.resize(static_cast<size_t>(n * S));
    BSG_CUDA(ctx, cudaMemcpyAsync(tmp.data(), dse, n * S * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  BSG_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (sample_e2e) {
    for (int64_t q = 0; q < n; ++q) {
      const int32_t r = static_cast<int32_t>(q / n_inst);
      for (int32_t j = 0; j < S; ++j) sample_e2e[q * S + perm[r * S + j]] = tmp[q * S + j];
    }
  }
  return BSG_OK;
}

}  // namespace

extern "C" {

bsg_status bsg_dispatch_mc(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                           const bsg_scenario* scenarios, const int32_t* instance_ids,
                           int32_t n_inst, int32_t n_requests, const int32_t* lengths,
                           int32_t n_samples, int32_t objective, int32_t* chosen,
                           int64_t* scores, int64_t* sample_e2e, bsg_result* per_instance) {
  if (!ctx || !entries || !scenarios || !instance_ids || !lengths || !chosen)
    return BSG_INVALID_ARGUMENT;
  if (n_inst <= 0) return BSG_NO_INSTANCES;
  if (n_samples < 1 || n_samples > 1024) return BSG_INVALID_ARGUMENT;
  if (n_requests <= 0) return BSG_OK;
  if (ctx->ncfg == 0) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return dispatch_fused(ctx, entries, n_entries, scenarios, instance_ids, n_inst, n_requests,
                        lengths, n_samples, objective, chosen, scores, sample_e2e, per_instance, nullptr,
                        0, 0.0, nullptr, nullptr);
}

bsg_status bsg_dispatch_mc_sampled(bsg_ctx* ctx, const bsg_entries* entries, int64_t n_entries,
                                   const bsg_scenario* scenarios, const int32_t* instance_ids,
                                   int32_t n_inst, int32_t n_requests, const uint64_t* request_ids,
                                   int32_t n_samples, uint64_t seed, double mean_abs_rel_error,
                                   int32_t objective, int32_t* chosen, int64_t* scores,
                                   int32_t* lengths_out, bsg_result* per_instance, int64_t* dev_keys) {
  if (!ctx || !entries || !scenarios || !instance_ids || !request_ids || !chosen)
    return BSG_INVALID_ARGUMENT;
  if (n_inst <= 0) return BSG_NO_INSTANCES;
  if (n_samples < 1 || n_samples > 1024 || !(mean_abs_rel_error >= 0)) return BSG_INVALID_ARGUMENT;
  if (n_requests <= 0) return BSG_OK;
  if (ctx->ncfg == 0) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return dispatch_fused(ctx, entries, n_entries, scenarios, instance_ids, n_inst, n_requests, nullptr,
                        n_samples, objective, chosen, scores, nullptr, per_instance, request_ids, seed,
                        mean_abs_rel_error, lengths_out, dev_keys);
}

}  // extern "C"

#ifdef BSG_PROFILE_TIMELINE
// debug build only: copies the per-scenario (start, end, SM) timeline of the last predict pass
extern "C" int bsg_debug_timeline(uint64_t* host, int64_t n) {
  if (n > bsg::kTimelineCap) n = bsg::kTimelineCap;
  return cudaMemcpyFromSymbol(host, bsg::g_timeline, 3 * n * sizeof(uint64_t)) == cudaSuccess ? 0 : 1;
}
#endif

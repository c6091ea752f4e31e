// closed_loop.cu — K5: device-resident closed-loop replay.
//
// One thread block runs one whole closed loop — SimulationDriver
// (core/src/driver.cpp:134-289) with static provisioning, zero dispatch
// overhead and BlockPredictive dispatch — without returning to the host:
//
//   * live serving instances (Instance, core/src/backend.cpp:238-331) are kept
//     in HBM as SoA columns; instance i owns a running region R (max_batch
//     slots, admission order) and a waiting region A (victims are pushed at its
//     front, arrivals at its back), so every instance's status snapshot
//     (backend.cpp:351-373) is directly a (running, waiting) slice pair — the
//     what-if kernel reads it in place, no snapshot copy;
//   * every arrival's per-instance what-ifs (predict(), predictor.cpp:76-137)
//     run on the block's warps with the same simulate_scenario as K1, followed
//     by the BlockPredictive argmin (scheduler.cpp:138-150, lowest id on ties);
//   * the event loop (event_loop.cpp:28-57) exploits that instances only
//     interact through dispatch: between two arrival instants each warp
//     advances its own instances' steps independently (completions strictly
//     before the next arrival; at an arrival instant the arrivals go first —
//     their sequence numbers are lower — then that instant's completions, then
//     end_of_instant's begin_step for every idle instance with work,
//     driver.cpp:271-289).
//
// Outcomes (arrival/dispatch/first-token/finish ticks, instance, preemptions)
// are bit-identical to the host driver and to the reference's run_experiment.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <cstring>
#include <vector>

#include "bsg_ctx.cuh"
#include "mc_sampler.cuh"
#include "bsg_internal.h"

namespace bsg {

#ifndef BSG_CL_WARPS
#define BSG_CL_WARPS 8
#endif
#ifndef BSG_CL_MINB
#define BSG_CL_MINB 2
#endif
// warps per closed-loop block / resident blocks per SM (measured on the cfg5 grid:
// 8 x 2 beats 16 x 1, 4 x 4, 4 x 6 and 8 x 3; optimistic 32-slot what-ifs, which
// pay off in K1, double the cost here: live running lists reach max_batch)
constexpr int kClWarps = BSG_CL_WARPS;
constexpr int kClMaxInst = 256;
constexpr int64_t kNever = INT64_MAX;

struct ClRun {
  int32_t n_inst, objective, cfg, n_req;
  int64_t req_off;    // first request row
  int64_t arena_off;  // first arena entry
  // ProvisionPolicy (autoscaler.h:10-27); ticks are SimTime::from_seconds
  int32_t prov_kind, max_inst;
  double threshold_s;
  int64_t cold_start_ticks, cooldown_ticks;
  int32_t policy;            // bsg_policy (scheduler.h:16-23)
  int32_t immediate;         // dispatch_overhead_s == 0: admit at the decision
  uint64_t policy_seed;      // Random's SplitMix64 stream
  int64_t overhead_ticks;    // SimTime::from_seconds(dispatch_overhead_s)
};

// Live-state SoA columns.
struct Arena {
  int32_t *prompt, *est, *prefill, *decoded, *target, *rid, *chunk;
};

struct ClInst {
  int32_t n;           // running members R[0, n)
  int32_t whead;       // waiting = A[whead, wland)
  int32_t wtail;       // A[wland, wtail): dispatched, still in flight (overhead mode)
  int32_t free_blocks;
  int64_t t_done;      // completion time of the current step
  int32_t mid;         // mid-step
  int32_t wland;       // end of the landed waiting requests
  int32_t held;        // the status snapshot's sum of blocks_needed(stored) over running
  int32_t pad;         //   (backend.cpp:357-365), kept by live_begin / live_finish
};

// Instance i of a run: R at base, A at base + maxb (A's first maxb slots are
// the room for victims pushed in front of the first arrival).
__device__ __forceinline__ int64_t inst_stride(int32_t maxb, int32_t n_req) {
  return 2 * static_cast<int64_t>(maxb) + n_req;
}

// begin_step (backend.cpp:238-296) of a live instance; warp-wide. Returns a
// bsg_status (EMPTY_PLAN / DEADLOCK propagate like the reference's throws).
template <int K, bool POW2>
__device__ int32_t live_begin(const DevCfg& cfg, const Arena& ar, int64_t Rb, int64_t Ab,
                              ClInst& st, int64_t now, bsg_request_outcome* outs,
                              unsigned long long* preempts) {
  constexpr int CAP = 32 * K;
  const int lane = lane_id();
  const int32_t n = st.n, whead = st.whead, wtail = st.wland;
  int32_t free_blocks = st.free_blocks;
  const int32_t maxb = cfg.max_batch_size;
  const bool chunked = cfg.local_policy == BSG_CHUNKED_PREFILL;
  const bool waiting_nonempty = whead < wtail;
  int32_t prompt[K], prefill[K], decoded[K], est[K], target[K], rid[K];
  bool ready[K], nonready[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t p = lane * K + k;
    prompt[k] = 1;
    prefill[k] = decoded[k] = est[k] = target[k] = rid[k] = 0;
    if (p < n) {
      const int64_t g = Rb + p;
      prompt[k] = ar.prompt[g];
      prefill[k] = ar.prefill[g];
      decoded[k] = ar.decoded[g];
      est[k] = ar.est[g];
      target[k] = ar.target[g];
      rid[k] = ar.rid[g];
    }
    ready[k] = p < n && prefill[k] == prompt[k];
    nonready[k] = p < n && prefill[k] != prompt[k];
  }
  const int32_t D = count<K>(ready);
  bool any_local = false;
#pragma unroll
  for (int k = 0; k < K; ++k) any_local |= nonready[k];
  const bool any_nonready = __any_sync(kFull, any_local);
  int32_t chunk[K];
  bool dec[K];
  int32_t budget = 0;
  bool prefill_step = false;
  if (chunked) {  // plan_chunked_prefill (backend.cpp:113-149)
    int32_t b0 = cfg.chunk_budget - D;
    if (b0 < 0) b0 = 0;
    budget = b0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      chunk[k] = 0;
      dec[k] = ready[k];
    }
    if (any_nonready) {
      int32_t rem[K], S[K];
#pragma unroll
      for (int k = 0; k < K; ++k) rem[k] = nonready[k] ? prompt[k] - prefill[k] : 0;
      const int32_t tot = excl_scan<K>(rem, S);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int32_t c = b0 - S[k];
        c = c < 0 ? 0 : c;
        chunk[k] = nonready[k] ? (c < rem[k] ? c : rem[k]) : 0;
      }
      budget = b0 - tot;
      if (budget < 0) budget = 0;
    }
  } else {  // plan_prefill_priority (backend.cpp:151-182)
    prefill_step = waiting_nonempty || any_nonready;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      chunk[k] = (prefill_step && nonready[k]) ? prompt[k] - prefill[k] : 0;
      dec[k] = !prefill_step && ready[k];
    }
  }
  int32_t delta[K], stored[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {  // make_item (backend.cpp:94-111)
    stored[k] = prefill[k] + decoded[k];
    int32_t ns = stored[k];
    if (dec[k]) {
      ns = stored[k] + 1;
    } else if (chunk[k] > 0) {
      const int32_t np = prefill[k] + chunk[k];
      ns = np + decoded[k] + (np == prompt[k] ? 1 : 0);
    }
    delta[k] = (dec[k] || chunk[k] > 0) ? bnt<POW2>(ns, cfg) - bnt<POW2>(stored[k], cfg) : 0;
  }
  const int32_t run_delta = warp_sum<K>(delta);
  // waiting admissions: FCFS prefix of A (backend.cpp:132-148 / 158-175)
  int32_t a = 0;
  if (waiting_nonempty && n < maxb && (chunked ? budget > 0 : true)) {
    const int32_t pf = free_blocks - run_delta;
    bool valid[K];
    int32_t wprompt[K], fdelta[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t p = lane * K + k;
      valid[k] = p >= n && p < maxb && (p - n) < (wtail - whead);
      if (p >= n) {
        if (valid[k]) {
          const int64_t g = Ab + whead + (p - n);
          prompt[k] = ar.prompt[g];
          est[k] = ar.est[g];
          target[k] = ar.target[g];
          rid[k] = ar.rid[g];
        }
        prefill[k] = 0;
        decoded[k] = 0;
        stored[k] = 0;
      }
      wprompt[k] = valid[k] ? prompt[k] : 0;
      fdelta[k] = valid[k] ? bnt<POW2>(prompt[k] + 1, cfg) : 0;
    }
    int32_t P[K], DX[K];
    excl_scan<K>(wprompt, P);
    excl_scan<K>(fdelta, DX);
    bool stop[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t p = lane * K + k;
      bool ok = valid[k];
      int32_t c = prompt[k];
      if (chunked) {
        const int32_t bj = budget - P[k];
        ok = ok && bj > 0;
        c = prompt[k] < bj ? prompt[k] : bj;
      }
      const int32_t dj = bnt<POW2>(c + (c == prompt[k] ? 1 : 0), cfg);
      ok = ok && dj <= pf - DX[k];
      if (ok && p >= n) {
        chunk[k] = c;
        delta[k] = dj;
      }
      stop[k] = p >= n && !ok;
    }
    a = first_pos<K>(stop, CAP) - n;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t p = lane * K + k;
      if (p >= n + a) {
        chunk[k] = 0;
        delta[k] = 0;
      }
    }
  }
  if (!chunked && prefill_step && !any_nonready && a == 0) {  // backend.cpp:176-181
    prefill_step = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      dec[k] = ready[k];
      delta[k] = ready[k] ? bnt<POW2>(stored[k] + 1, cfg) - bnt<POW2>(stored[k], cfg) : 0;
    }
  }
  if (n == 0 && a == 0) return BSG_EMPTY_PLAN;  // backend.cpp:245
  const int32_t n_adm = n + a;
  // allocation with newest-member preemption: e* = max{e : F(e) >= 0}
  // (backend.cpp:263-288; derivation in scenario_sim.cuh / DESIGN.md)
  const int32_t tot_delta = warp_sum<K>(delta);
  int32_t e_star = n_adm;
  if (tot_delta > free_blocks) {
    int32_t ho[K], hinc[K], dinc[K], fe[K];
    bool badp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) ho[k] = (lane * K + k) < n ? bnt<POW2>(stored[k], cfg) : 0;
    const int32_t htot = excl_scan<K>(ho, hinc);
    excl_scan<K>(delta, dinc);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t p = lane * K + k;
      fe[k] = free_blocks + (htot - hinc[k] - ho[k]) - (dinc[k] + delta[k]);
      badp[k] = p < n_adm && fe[k] < 0;
    }
    e_star = first_pos<K>(badp, n_adm);
    if (e_star == 0) return BSG_DEADLOCK;  // backend.cpp:274-277
    free_blocks = read_pos<K>(fe, e_star - 1);
  } else {
    free_blocks -= tot_delta;
  }
  const int32_t v = n_adm - e_star;  // victims, oldest first
  const int32_t new_whead = whead + a - v;
  __syncwarp();  // every lane has read its A entries before victims overwrite A's front
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t p = lane * K + k;
    if (p >= n && p < e_star) {  // admitted and kept: into R
      const int64_t g = Rb + p;
      ar.prompt[g] = prompt[k];
      ar.est[g] = est[k];
      ar.prefill[g] = 0;
      ar.decoded[g] = 0;
      ar.target[g] = target[k];
      ar.rid[g] = rid[k];
    }
    if (p >= e_star && p < n_adm) {  // victim: recompute, to the waiting front (preempt, 221-232)
      const int64_t g = Ab + new_whead + (p - e_star);
      ar.prompt[g] = prompt[k];
      ar.est[g] = est[k];
      ar.prefill[g] = 0;
      ar.decoded[g] = 0;
      ar.target[g] = target[k];
      ar.rid[g] = rid[k];
      outs[rid[k]].preempt_count += 1;
    }
  }
  if (v > 0 && lane == 0 && preempts) atomicAdd(preempts, static_cast<unsigned long long>(v));
  // price the surviving plan (to_batch_plan 194-209, batch_latency 10-14)
  bool ds[K], ps[K];
  int32_t ctx[K], pt[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t p = lane * K + k;
    ds[k] = p < e_star && dec[k];
    ps[k] = p < e_star && chunk[k] > 0;
    ctx[k] = ds[k] ? stored[k] : 0;
    pt[k] = ps[k] ? chunk[k] : 0;
    if (p < e_star) ar.chunk[Rb + p] = ds[k] ? -1 : (ps[k] ? chunk[k] : 0);
  }
  const int32_t n_dec = count<K>(ds);
  const int64_t dur = step_ticks(cfg, warp_sum<K>(pt), n_dec, warp_sum<K>(ctx));
  int32_t hs[K];  // the surviving members' blocks at their pre-step stored tokens
#pragma unroll
  for (int k = 0; k < K; ++k) hs[k] = (lane * K + k) < e_star ? bnt<POW2>(stored[k], cfg) : 0;
  const int32_t held = warp_sum<K>(hs);
  // every lane writes the (warp-uniform) new state: no lane ever reads a value
  // another lane stored, so the state may live in registers, shared or global
  __syncwarp();
  st.held = held;
  st.n = e_star;
  st.whead = new_whead;
  st.free_blocks = free_blocks;
  st.mid = 1;
  st.t_done = now + dur;
  __syncwarp();
  return BSG_OK;
}

// finish_step (backend.cpp:298-331) + the driver's outcome bookkeeping
// (handle_batch_complete, driver.cpp:233-251); warp-wide.
template <int K, bool POW2>
__device__ void live_finish(const DevCfg& cfg, const Arena& ar, int64_t Rb, ClInst& st,
                            int64_t now, bsg_request_outcome* outs, double relief_threshold_s,
                            int64_t relief_after, unsigned long long* relief_min) {
  const int lane = lane_id();
  const int32_t n = st.n;
  int32_t prompt[K], prefill[K], decoded[K], est[K], target[K], rid[K], keep[K], dst[K], freed[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t p = lane * K + k;
    keep[k] = 0;
    freed[k] = 0;
    if (p < n) {
      const int64_t g = Rb + p;
      prompt[k] = ar.prompt[g];
      prefill[k] = ar.prefill[g];
      decoded[k] = ar.decoded[g];
      est[k] = ar.est[g];
      target[k] = ar.target[g];
      rid[k] = ar.rid[g];
      const int32_t c = ar.chunk[g];
      const int32_t prev = decoded[k];
      if (c < 0) {
        decoded[k] += 1;
      } else if (c > 0) {
        prefill[k] += c;
        if (prefill[k] == prompt[k]) decoded[k] += 1;
      }
      const bool item = c != 0;
      if (item && prev == 0 && decoded[k] >= 1 && outs[rid[k]].first_token_ticks < 0)
        outs[rid[k]].first_token_ticks = now;
      const bool done = item && decoded[k] >= target[k];
      if (done) {
        outs[rid[k]].finish_ticks = now;
        freed[k] = bnt<POW2>(prefill[k] + decoded[k], cfg);
        // relief provisioning signal: realized e2e (handle_batch_complete,
        // driver.cpp:245-248); only the earliest eligible trigger matters
        if (relief_min && now >= relief_after &&
            static_cast<double>(now - outs[rid[k]].arrival_ticks) * 1e-9 >= relief_threshold_s)
          atomicMin(relief_min, static_cast<unsigned long long>(now));
      }
      keep[k] = done ? 0 : 1;
    }
  }
  const int32_t kept = excl_scan<K>(keep, dst);
  const int32_t rel = warp_sum<K>(freed);
  int32_t hk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) hk[k] = keep[k] ? bnt<POW2>(prefill[k] + decoded[k], cfg) : 0;
  const int32_t held = warp_sum<K>(hk);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < K; ++k) {  // stable erase of completed members (backend.cpp:319-322)
    if (keep[k]) {
      const int64_t g = Rb + dst[k];
      ar.prompt[g] = prompt[k];
      ar.prefill[g] = prefill[k];
      ar.decoded[g] = decoded[k];
      ar.est[g] = est[k];
      ar.target[g] = target[k];
      ar.rid[g] = rid[k];
    }
  }
  __syncwarp();
  const int32_t nf = st.free_blocks + rel;  // warp-uniform state update, every lane
  __syncwarp();
  st.n = kept;
  st.held = held;
  st.free_blocks = nf;
  st.mid = 0;
  __syncwarp();
}

template <int K>
struct ClShared {
  ClInst inst[kClMaxInst];
  bsg_result res[kClMaxInst];
  int32_t scratch[kClWarps][smem_words(K, BSG_WIN_J_CLOSED)];
  int64_t pend[kClMaxInst];     // provision-complete times, non-decreasing
  unsigned long long preempts;
  unsigned long long end_ticks;
  unsigned long long cand_min;  // relief: earliest eligible trigger of an interval
  int64_t last_prov;            // Autoscaler::last_provision_ (-1: none)
  int64_t cur;                  // relief: the trigger instant being replayed
  int32_t cnt;                  // relief: qualifying completions at `cur`
  int32_t n_pend, pend_head;    // provisions triggered / completed
  int32_t active;               // instances dispatchable (instances_.size())
  int32_t next;
  int32_t err;
  // metric pipeline (aggregate, metrics.cpp:21-124, and the per-dispatch
  // free-block balance, driver.cpp:142-157)
  int32_t snap_free[kClMaxInst];
  // heuristic dispatch (pick_heuristic, scheduler.cpp:68-113)
  double hscore[kClMaxInst];
  int32_t qpm[kClMaxInst];      // dispatches of the last 60 s per instance (QpmTracker)
  int32_t qhead;                // oldest request still inside the QPM window
  int32_t chosen;
  int32_t idle_rep;             // lowest idle instance (its what-if serves every idle one)
  unsigned long long rng;       // Random's SplitMix64 state (rand.h:11-56)
  unsigned long long rr;        // RoundRobin's cursor
  double fm_sum, fv_sum;
  int32_t n_points;
  int32_t hist[256];
  unsigned long long sel_prefix;
  long long sel_k;
  long long cnt_fin;
  unsigned long long min_arr, max_fin;
};

__device__ __forceinline__ bool finished(const bsg_request_outcome& o) {
  return o.finish_ticks >= 0 && o.dispatch_ticks >= 0 && o.first_token_ticks >= 0;
}
__device__ __forceinline__ int64_t ttft_ticks(const bsg_request_outcome& o) {
  return o.first_token_ticks - o.dispatch_ticks;
}
__device__ __forceinline__ int64_t e2e_ticks(const bsg_request_outcome& o) {
  return o.finish_ticks - o.arrival_ticks;
}

// k-th smallest (0-based) TTFT (which = 0) or e2e (which = 1) tick count over
// the finished requests: block-wide radix select, 8 passes of 8-bit digits.
// SimTime::seconds is monotone in ticks, so this is the nearest-rank
// percentile of the reference's sorted doubles (metrics.cpp:11-19).
template <int K>
__device__ int64_t block_select(ClShared<K>& S, const bsg_request_outcome* outs, int32_t N, int which,
                                long long k) {
  if (threadIdx.x == 0) {
    S.sel_prefix = 0;
    S.sel_k = k;
  }
  unsigned long long mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) S.hist[b] = 0;
    __syncthreads();
    const unsigned long long prefix = S.sel_prefix;
    for (int32_t q = threadIdx.x; q < N; q += blockDim.x) {
      const bsg_request_outcome o = outs[q];
      if (!finished(o)) continue;
      const unsigned long long key = static_cast<unsigned long long>(which ? e2e_ticks(o) : ttft_ticks(o));
      if ((key & mask) == prefix) atomicAdd(&S.hist[(key >> shift) & 255], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long kk = S.sel_k;
      int d = 0;
      for (; d < 255 && kk >= S.hist[d]; ++d) kk -= S.hist[d];
      S.sel_k = kk;
      S.sel_prefix = prefix | (static_cast<unsigned long long>(d) << shift);
    }
    mask |= 0xffull << shift;
    __syncthreads();
  }
  const int64_t v = static_cast<int64_t>(S.sel_prefix);
  __syncthreads();  // every thread has read the result before the next selection resets it
  return v;
}

// percentile_nearest_rank's rank (metrics.cpp:14-17), 0-based
__device__ __forceinline__ long long nearest_rank0(double p, long long n) {
  long long rank = static_cast<long long>(ceil(__dmul_rn(p / 100.0, static_cast<double>(n))));
  if (rank < 1) rank = 1;
  if (rank > n) rank = n;
  return rank - 1;
}

// aggregate (metrics.cpp:21-124) of one finished run, on its block.
template <int K>
__device__ void block_report(ClShared<K>& S, const bsg_request_outcome* outs, int32_t N,
                             const bsg_replay_summary& sm, bsg_run_report* rep) {
  if (threadIdx.x == 0) {
    S.cnt_fin = 0;
    S.min_arr = ~0ull;
    S.max_fin = 0;
  }
  __syncthreads();
  long long fin = 0;
  unsigned long long mn = ~0ull, mx = 0;
  for (int32_t q = threadIdx.x; q < N; q += blockDim.x) {
    const bsg_request_outcome o = outs[q];
    mn = min(mn, static_cast<unsigned long long>(o.arrival_ticks));
    if (finished(o)) {
      ++fin;
      mx = max(mx, static_cast<unsigned long long>(o.finish_ticks));
    }
  }
  atomicAdd(reinterpret_cast<unsigned long long*>(&S.cnt_fin), static_cast<unsigned long long>(fin));
  atomicMin(&S.min_arr, mn);
  atomicMax(&S.max_fin, mx);
  __syncthreads();
  const long long n_fin = S.cnt_fin;
  bsg_run_report r{};
  if (n_fin > 0) {
    const int64_t t50 = block_select(S, outs, N, 0, nearest_rank0(50.0, n_fin));
    const int64_t t99 = block_select(S, outs, N, 0, nearest_rank0(99.0, n_fin));
    const int64_t e50 = block_select(S, outs, N, 1, nearest_rank0(50.0, n_fin));
    const int64_t e99 = block_select(S, outs, N, 1, nearest_rank0(99.0, n_fin));
    r.p50_ttft_s = static_cast<double>(t50) * 1e-9;
    r.p99_ttft_s = static_cast<double>(t99) * 1e-9;
    r.p50_e2e_s = static_cast<double>(e50) * 1e-9;
    r.p99_e2e_s = static_cast<double>(e99) * 1e-9;
  }
  if (threadIdx.x != 0) return;
  // means: summed in request order, as the reference does
  double st = 0, se = 0, so = 0;
  for (int32_t q = 0; q < N; ++q) {
    const bsg_request_outcome o = outs[q];
    if (!finished(o)) continue;
    st = __dadd_rn(st, static_cast<double>(ttft_ticks(o)) * 1e-9);
    se = __dadd_rn(se, static_cast<double>(e2e_ticks(o)) * 1e-9);
    so = __dadd_rn(so, static_cast<double>(o.dispatch_ticks - o.arrival_ticks) * 1e-9);
  }
  r.finished_requests = static_cast<int32_t>(n_fin);
  r.censored_requests = N - static_cast<int32_t>(n_fin);
  if (n_fin > 0) {
    r.mean_ttft_s = st / static_cast<double>(n_fin);
    r.mean_e2e_s = se / static_cast<double>(n_fin);
    r.mean_overhead_s = so / static_cast<double>(n_fin);
    const int64_t first = static_cast<int64_t>(S.min_arr), last = static_cast<int64_t>(S.max_fin);
    if (N > 0 && last > first)
      r.throughput_rps = static_cast<double>(n_fin) / (static_cast<double>(last - first) * 1e-9);
  }
  r.total_preemptions = sm.total_preemptions;
  r.instances_provisioned = sm.instances_provisioned;
  r.final_instance_count = sm.final_instance_count;
  if (S.n_points > 0) {
    r.free_blocks_mean_avg = S.fm_sum / static_cast<double>(S.n_points);
    r.free_blocks_var_avg = S.fv_sum / static_cast<double>(S.n_points);
  }
  *rep = r;
}

// Autoscaler::evaluate (autoscaler.cpp:36-52) for a signal of the run's kind:
// on a trigger, the instance's ProvisionComplete is due cold_start later
// (maybe_provision, driver.cpp:253-261). Caller: one thread.
template <int K>
__device__ __forceinline__ void autoscale(ClShared<K>& S, const ClRun& run, int32_t initial, double latency_s,
                                          int64_t now) {
  if (latency_s < run.threshold_s) return;
  if (S.last_prov >= 0 && now - S.last_prov < run.cooldown_ticks) return;
  if (initial + S.n_pend >= run.max_inst) return;  // active + pending (invariant under completion)
  S.last_prov = now;
  S.pend[S.n_pend++] = now + run.cold_start_ticks;
}

// Wide member lists (K >= 4: max_batch_size > 64) hold 4-8 members per lane in
// registers; at 2 blocks per SM (128 registers) they spilled 150-1800 B per
// thread, so they get one block per SM and the full register file.
__host__ __device__ constexpr int cl_min_blocks(int K) { return K >= 4 ? 1 : BSG_CL_MINB; }

template <int K, bool POW2>
__global__ void __launch_bounds__(kClWarps * 32, cl_min_blocks(K))
    closed_loop_kernel(const DevCfg* __restrict__ cfgs, const ClRun* __restrict__ runs,
                       const int32_t* __restrict__ rq_prompt, const int32_t* __restrict__ rq_output,
                       const int32_t* __restrict__ rq_est, const int64_t* __restrict__ rq_arrival,
                       Arena ar, bsg_request_outcome* __restrict__ outcomes,
                       bsg_replay_summary* __restrict__ summaries, int32_t* __restrict__ status,
                       bsg_run_report* __restrict__ reports) {
#ifdef BSG_CL_TIMING
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  extern __shared__ __align__(16) unsigned char cl_smem[];
  ClShared<K>& S = *reinterpret_cast<ClShared<K>*>(cl_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ClRun run = runs[blockIdx.x];
  const DevCfg cfg = cfgs[run.cfg];
  // live instances price steps with batch_latency itself (driver.cpp:274 calls
  // begin_step() without a latency function); only predict() uses the cache
  DevCfg live_cfg = cfg;
  live_cfg.cache_mode = BSG_CACHE_OFF;
  const int32_t I0 = run.n_inst, N = run.n_req, maxb = cfg.max_batch_size;
  const int32_t IMAX = run.prov_kind == 0 ? I0 : run.max_inst;  // instance slots
  const int64_t stride = inst_stride(maxb, N);
  bsg_request_outcome* outs = outcomes + run.req_off;
  const int64_t* arrival = rq_arrival + run.req_off;
  if (IMAX > kClMaxInst || maxb > 32 * K) {  // the host validates; never reached
    if (threadIdx.x == 0) status[blockIdx.x] = BSG_BAD_INPUT;
    return;
  }
  for (int i = threadIdx.x; i < IMAX; i += blockDim.x) {
    ClInst& s = S.inst[i];
    s.n = 0;
    s.whead = maxb;
    s.wtail = maxb;
    s.wland = maxb;
    s.held = 0;
    s.free_blocks = cfg.total_blocks;
    s.t_done = 0;
    s.mid = 0;
  }
  if (threadIdx.x == 0) {
    S.preempts = 0;
    S.end_ticks = 0;
    S.err = BSG_OK;
    S.last_prov = -1;
    S.n_pend = 0;
    S.pend_head = 0;
    S.active = I0;
    S.cand_min = ~0ull;
    S.fm_sum = 0;
    S.fv_sum = 0;
    S.n_points = 0;
    S.qhead = 0;
    S.rng = run.policy_seed;
    S.rr = 0;
  }
  for (int i = threadIdx.x; i < IMAX; i += blockDim.x) S.qpm[i] = 0;
  __syncthreads();
  const bool relief = run.prov_kind == 2;
  int64_t last_done = 0;  // this warp's latest processed completion
  int64_t relief_after = 0;  // relief: earliest trigger time the cooldown allows
  // close the instant tc (its completions, then end_of_instant's begin_step) and
  // advance through every completion strictly before t
  // overhead mode: the next in-flight request of instance s lands at its
  // arrival + overhead (kDispatch, driver.cpp:216-231); landings of one
  // instance are in dispatch order
  auto next_land = [&](const ClInst& s, int64_t Ab, int32_t wl) -> int64_t {
    if (wl >= s.wtail) return kNever;
    return arrival[__ldcg(&ar.rid[Ab + wl])] + run.overhead_ticks;
  };
  // every landing at `now`: the new landed end is computed in registers and
  // stored warp-uniformly (no lane reads a value another lane is writing)
  auto land_at = [&](ClInst& s, int64_t Ab, int64_t now) {
    int32_t wl = s.wland;
    while (next_land(s, Ab, wl) == now) ++wl;
    __syncwarp();
    s.wland = wl;
    __syncwarp();
  };
  // close the instant tc (its completions and landings — events at tc after
  // that instant's arrivals — then end_of_instant's begin_step) and advance
  // through every event strictly before t. A landing and a completion of the
  // same instance at one instant commute (finish_step does not read waiting_).
  auto advance = [&](int32_t i, int64_t tc, int64_t t) -> int32_t {
    ClInst& s = S.inst[i];
    const int64_t Rb = run.arena_off + i * stride;
    const int64_t Ab = Rb + maxb;
    if (tc >= 0) {
      if (s.mid && s.t_done == tc) {
        live_finish<K, POW2>(cfg, ar, Rb, s, tc, outs, run.threshold_s, relief_after,
                             relief ? &S.cand_min : nullptr);
        last_done = max(last_done, tc);
      }
      land_at(s, Ab, tc);
      if (!s.mid && (s.n > 0 || s.whead < s.wland)) {
        const int32_t e = live_begin<K, POW2>(live_cfg, ar, Rb, Ab, s, tc, outs, &S.preempts);
        if (e != BSG_OK) return e;
      }
    }
    for (;;) {
      const int64_t tl = next_land(s, Ab, s.wland);
      const int64_t td = s.mid ? s.t_done : kNever;
      const int64_t now = min(tl, td);
      if (now >= t) break;
      if (td == now) {
        live_finish<K, POW2>(cfg, ar, Rb, s, now, outs, run.threshold_s, relief_after,
                             relief ? &S.cand_min : nullptr);
      }
      land_at(s, Ab, now);
      last_done = max(last_done, now);
      if (!s.mid && (s.n > 0 || s.whead < s.wland)) {
        const int32_t e = live_begin<K, POW2>(live_cfg, ar, Rb, Ab, s, now, outs, &S.preempts);
        if (e != BSG_OK) return e;
      }
    }
    return BSG_OK;
  };
  auto fail = [&](int32_t e) {
    if (lane == 0) atomicCAS(&S.err, BSG_OK, e);
  };
  // Relief provisioning over the completions of the interval just advanced:
  // instances evolve independently of the autoscaler between arrivals, so the
  // triggers are replayed afterwards in time order. Each qualifying completion
  // is one signal (driver.cpp:245-248): the earliest one at or after
  // last_provision + cooldown triggers; with cooldown 0 every qualifying
  // completion of that instant triggers too (up to max_instances).
  auto relief_round = [&](int64_t t_end) {
    for (;;) {
      if (threadIdx.x == 0) {
        const unsigned long long c = S.cand_min;
        S.cand_min = ~0ull;
        S.cur = static_cast<int64_t>(c);
        S.cnt = 0;
        S.next = (c != ~0ull && static_cast<int64_t>(c) < t_end && I0 + S.n_pend < run.max_inst) ? 1 : 0;
      }
      __syncthreads();
      if (!S.next) break;
      const int64_t c = S.cur;
      auto qualifies = [&](int32_t q) {
        return static_cast<double>(outs[q].finish_ticks - outs[q].arrival_ticks) * 1e-9 >= run.threshold_s;
      };
      if (run.cooldown_ticks == 0)
        for (int32_t q = threadIdx.x; q < N; q += blockDim.x)
          if (outs[q].finish_ticks == c && qualifies(q)) atomicAdd(&S.cnt, 1);
      __syncthreads();
      if (threadIdx.x == 0) {
        int32_t m = run.cooldown_ticks == 0 ? S.cnt : 1;
        for (; m > 0 && I0 + S.n_pend < run.max_inst; --m) {
          S.last_prov = c;
          S.pend[S.n_pend++] = c + run.cold_start_ticks;
        }
      }
      relief_after = c + (run.cooldown_ticks > 0 ? run.cooldown_ticks : 1);
      __syncthreads();
      for (int32_t q = threadIdx.x; q < N; q += blockDim.x) {  // the next eligible completion
        const int64_t f = outs[q].finish_ticks;
        if (f >= relief_after && f < t_end && qualifies(q))
          atomicMin(&S.cand_min, static_cast<unsigned long long>(f));
      }
      __syncthreads();
    }
    relief_after = S.last_prov >= 0 ? S.last_prov + run.cooldown_ticks : 0;
  };
  int64_t t_prev = -1;
#ifdef BSG_CL_TIMING
  unsigned long long ph_adv = 0, ph_wif = 0, ph_t = 0;  // debug: advance / what-if phase ns
  auto gtime = [] {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
  };
#endif
  for (int32_t k = 0; k < N; ++k) {
    const int64_t t = arrival[k];
#ifdef BSG_CL_TIMING
    if (threadIdx.x == 0) ph_t = gtime();
#endif
    if (t != t_prev) {
      const int32_t I = S.active;
      for (int32_t i = warp; i < I; i += kClWarps) {
        const int32_t e = advance(i, t_prev, t);
        if (e != BSG_OK) {
          fail(e);
          break;
        }
      }
      __syncthreads();
#ifdef BSG_CL_TIMING
      if (threadIdx.x == 0) {
        const unsigned long long g = gtime();
        ph_adv += g - ph_t;
        ph_t = g;
      }
#endif
      if (S.err != BSG_OK) break;
      if (relief) relief_round(t);
      // ProvisionComplete events before this instant (arrivals at an equal time go first)
      if (threadIdx.x == 0)
        while (S.pend_head < S.n_pend && S.pend[S.pend_head] < t) {
          S.end_ticks = max(S.end_ticks, static_cast<unsigned long long>(S.pend[S.pend_head]));
          ++S.pend_head;
          ++S.active;
        }
      __syncthreads();
    }
    const int32_t I = S.active;
    // ---- dispatch: per-instance what-ifs (predict_across) + argmin, or the
    // heuristic scores of pick_heuristic (scheduler.cpp:68-113) ----
    const bool bp = run.policy == BSG_POLICY_BLOCK_PREDICTIVE;
    // An idle instance's snapshot (no running, no waiting) is the same for every
    // idle instance of the run (one config): predict() on it depends only on the
    // candidate, so the lowest idle instance's what-if serves them all (exact —
    // the same simulation). Light-load points of a sweep are mostly idle
    // instances.
    auto idle = [&](int32_t i) { return S.inst[i].n == 0 && S.inst[i].whead == S.inst[i].wland; };
    if (threadIdx.x == 0) S.idle_rep = INT32_MAX;
    __syncthreads();
    if (bp)
      for (int32_t i = threadIdx.x; i < I; i += blockDim.x)
        if (idle(i)) atomicMin(&S.idle_rep, i);
    if (threadIdx.x == 0) {
      S.next = 0;
      if (run.policy == BSG_POLICY_MIN_QPM) {  // QpmTracker: dispatches strictly younger than 60 s
        const int64_t cutoff = t - 60000000000LL;
        while (S.qhead < k && arrival[S.qhead] <= cutoff) {
          S.qpm[outs[S.qhead].instance] -= 1;
          S.qhead += 1;
        }
      }
    }
    __syncthreads();
    const int32_t cp = rq_prompt[run.req_off + k], ce = rq_est[run.req_off + k];
    const bool need_stats = reports || run.policy == BSG_POLICY_INFAAS_PP ||
                            run.policy == BSG_POLICY_LLUMNIX_MINUS;
    for (;;) {
      int32_t i = 0;
      if (lane == 0) i = atomicAdd(&S.next, 1);
      i = __shfl_sync(kFull, i, 0);
      if (i >= I) break;
      const ClInst& s = S.inst[i];
      if (need_stats) {  // the snapshot's free blocks (backend.cpp:357-365): total - sum held(stored)
        const int32_t snap_free = cfg.total_blocks - s.held;
        if (lane == 0) S.snap_free[i] = snap_free;
        if (!bp) {
          // load_infaas / load_llumnix (scheduler.cpp:33-46) over the snapshot
          const double used = static_cast<double>(cfg.total_blocks - snap_free);
          const double bsz = static_cast<double>(max(s.n, 1));
          double score = 0;
          if (run.policy == BSG_POLICY_LLUMNIX_MINUS) {
            long long pm = 0;  // blocks_needed(prompt - prefill_progress) over waiting
            for (int32_t q = s.whead + lane; q < s.wland; q += 32) {
              const int64_t g = run.arena_off + i * stride + maxb + q;
              pm += bnt<POW2>(__ldcg(&ar.prompt[g]) - __ldcg(&ar.prefill[g]), cfg);
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) pm += __shfl_xor_sync(kFull, pm, d);
            score = __ddiv_rn(__dadd_rn(used, static_cast<double>(pm)), bsz);
          } else if (run.policy == BSG_POLICY_INFAAS_PP) {
            score = __ddiv_rn(used, bsz);
          }
          if (lane == 0) S.hscore[i] = score;
        }
      }
      if (!bp || (i != S.idle_rep && idle(i))) continue;
      bsg_scenario sc;
      sc.run_off = static_cast<int32_t>(run.arena_off + i * stride);
      sc.run_n = s.n;
      sc.wait_off = static_cast<int32_t>(run.arena_off + i * stride + maxb + s.whead);
      sc.wait_n = s.wland - s.whead;
      sc.cand_prompt = cp;
      sc.cand_est = ce;
      sc.cfg = run.cfg;
      sc.reserved = 0;
      simulate_scenario<K, false, false, POW2, false, false, BSG_WIN_J_CLOSED, BSG_CYC_CLOSED>(
          cfg, ar.prompt, ar.est, ar.prefill, ar.decoded, sc, S.scratch[warp], &S.res[i],
          TraceSink{nullptr, 0});
    }
    __syncthreads();
#ifdef BSG_CL_TIMING
    if (threadIdx.x == 0) {
      const unsigned long long g = gtime();
      ph_wif += g - ph_t;
    }
#endif
    if (bp && S.idle_rep < I) {
      const int32_t r0 = S.idle_rep;
      for (int32_t i = threadIdx.x; i < I; i += blockDim.x)
        if (i != r0 && idle(i)) S.res[i] = S.res[r0];
      __syncthreads();
    }
    if (!bp) {
      if (threadIdx.x == 0) {
        int32_t c = 0;
        if (run.policy == BSG_POLICY_RANDOM) {  // ids[rng.below(n)] over sorted ids
          const unsigned long long n = static_cast<unsigned long long>(I);
          const unsigned long long limit = ~0ull - ~0ull % n;
          unsigned long long r;
          do {
            unsigned long long z = (S.rng += 0x9e3779b97f4a7c15ull);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            r = z ^ (z >> 31);
          } while (r >= limit);
          c = static_cast<int32_t>(r % n);
        } else if (run.policy == BSG_POLICY_ROUND_ROBIN) {
          c = static_cast<int32_t>(S.rr++ % static_cast<unsigned long long>(I));
        } else {  // lowest score, lowest id on ties (instances in id order)
          double best = 0;
          for (int32_t q = 0; q < I; ++q) {
            const double v = run.policy == BSG_POLICY_MIN_QPM ? static_cast<double>(S.qpm[q]) : S.hscore[q];
            if (q == 0 || v < best) {
              best = v;
              c = q;
            }
          }
        }
        S.chosen = c;
      }
      __syncthreads();
      // heuristics carry no prediction: preempt provisioning asks for the chosen
      // instance's (driver.cpp:202-209)
      if (run.prov_kind == 1 && warp == 0) {
        const int32_t i = S.chosen;
        const ClInst& s = S.inst[i];
        bsg_scenario sc;
        sc.run_off = static_cast<int32_t>(run.arena_off + i * stride);
        sc.run_n = s.n;
        sc.wait_off = static_cast<int32_t>(run.arena_off + i * stride + maxb + s.whead);
        sc.wait_n = s.wland - s.whead;
        sc.cand_prompt = cp;
        sc.cand_est = ce;
        sc.cfg = run.cfg;
        sc.reserved = 0;
        simulate_scenario<K, false, false, POW2, false, false, BSG_WIN_J_CLOSED, BSG_CYC_CLOSED>(
            cfg, ar.prompt, ar.est, ar.prefill, ar.decoded, sc, S.scratch[0], &S.res[i],
            TraceSink{nullptr, 0});
      }
      __syncthreads();
    }
    if (warp == 0) {
      int32_t best_i = 0, bad = BSG_OK;
      if (bp) {  // BlockPredictive argmin (scheduler.cpp:138-150)
        int64_t best_v = INT64_MAX;
        best_i = INT32_MAX;
        for (int32_t i = lane; i < I; i += 32) {
          const bsg_result& r = S.res[i];
          if (r.status != BSG_OK && bad == BSG_OK) bad = r.status;
          const int64_t v = run.objective == 1 ? r.ttft_ticks : r.e2e_ticks;
          if (v < best_v || (v == best_v && i < best_i)) {
            best_v = v;
            best_i = i;
          }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
          const int64_t ov = __shfl_xor_sync(kFull, best_v, d);
          const int32_t oi = __shfl_xor_sync(kFull, best_i, d);
          if (ov < best_v || (ov == best_v && oi < best_i)) {
            best_v = ov;
            best_i = oi;
          }
        }
        bad = static_cast<int32_t>(__reduce_max_sync(kFull, static_cast<uint32_t>(bad)));
      } else {
        best_i = S.chosen;
        if (run.prov_kind == 1 && S.res[best_i].status != BSG_OK) bad = S.res[best_i].status;
      }
      if (bad != BSG_OK) {
        fail(bad);  // PredictionError propagates out of the run (predictor.cpp:132-136)
      } else if (lane == 0) {  // the chosen instance receives the arrival
        if (reports) {  // memory-balance sample of this dispatch (driver.cpp:142-157)
          double mean = 0;
          for (int32_t q = 0; q < I; ++q) mean = __dadd_rn(mean, static_cast<double>(S.snap_free[q]));
          mean /= static_cast<double>(I);
          double var = 0;
          for (int32_t q = 0; q < I; ++q) {
            const double d = __dsub_rn(static_cast<double>(S.snap_free[q]), mean);
            var = __dadd_rn(var, __dmul_rn(d, d));
          }
          var /= static_cast<double>(I);
          S.fm_sum = __dadd_rn(S.fm_sum, mean);
          S.fv_sum = __dadd_rn(S.fv_sum, var);
          S.n_points += 1;
        }
        if (run.policy == BSG_POLICY_MIN_QPM) S.qpm[best_i] += 1;  // record_dispatch
        if (run.prov_kind == 1)  // preempt provisioning on the predicted e2e (driver.cpp:197-211)
          autoscale<K>(S, run, I0, static_cast<double>(S.res[best_i].e2e_ticks) * 1e-9, t);
        // append at the waiting tail; with overhead it lands later (driver.cpp:213-231)
        ClInst& s = S.inst[best_i];
        const int64_t g = run.arena_off + best_i * stride + maxb + s.wtail;
        ar.prompt[g] = cp;
        ar.est[g] = ce;
        ar.prefill[g] = 0;
        ar.decoded[g] = 0;
        ar.target[g] = rq_output[run.req_off + k];
        ar.rid[g] = k;
        s.wtail += 1;
        if (run.immediate) s.wland = s.wtail;
        outs[k].dispatch_ticks = run.immediate ? t : t + run.overhead_ticks;
        outs[k].instance = best_i;
      }
    }
    __syncthreads();
    if (S.err != BSG_OK) break;
    t_prev = t;
  }
  if (S.err == BSG_OK) {  // drain
    const int32_t I = S.active;
    for (int32_t i = warp; i < I; i += kClWarps) {
      const int32_t e = advance(i, t_prev, kNever);
      if (e != BSG_OK) {
        fail(e);
        break;
      }
    }
    __syncthreads();
    if (relief) relief_round(kNever);
    if (threadIdx.x == 0)  // the remaining ProvisionComplete events
      for (; S.pend_head < S.n_pend; ++S.pend_head, ++S.active)
        S.end_ticks = max(S.end_ticks, static_cast<unsigned long long>(S.pend[S.pend_head]));
  }
  if (lane == 0) atomicMax(&S.end_ticks, static_cast<unsigned long long>(max(last_done, t_prev)));
  __syncthreads();
  if (threadIdx.x == 0) {
    status[blockIdx.x] = S.err;
    bsg_replay_summary sm{};
    sm.total_preemptions = static_cast<int64_t>(S.preempts);
    sm.end_ticks = static_cast<int64_t>(S.end_ticks);
#ifdef BSG_CL_TIMING
    {  // debug: this block's wall time (ns) replaces the summary's end time
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      sm.end_ticks = static_cast<int64_t>(t_end - t_start);
    }
#endif
    sm.instances_provisioned = S.n_pend;
    sm.final_instance_count = S.active;
#ifdef BSG_CL_TIMING
    sm.total_preemptions = static_cast<int64_t>(ph_adv);                 // debug: advance ns
    sm.instances_provisioned = static_cast<int32_t>(ph_wif / 1000);      // debug: stats + what-if us
#endif
    summaries[blockIdx.x] = sm;
  }
  if (reports && S.err == BSG_OK) {
    __syncthreads();
    bsg_replay_summary sm{};
    sm.total_preemptions = static_cast<int64_t>(S.preempts);
    sm.instances_provisioned = S.n_pend;
    sm.final_instance_count = S.active;
    block_report<K>(S, outs, N, sm, &reports[blockIdx.x]);
  }
}

// ---- fleet: the live instances as a persistent device mirror ----------------
// SURVEY §8(f) row 2. A fleet keeps K5's arena (every instance's running and
// waiting lists) resident in HBM across calls; each bsg_fleet_dispatch is ONE
// launch with one warp per instance: the warp advances its instance to the
// arrival instant (the snapshot is updated in place — nothing is packed or
// copied), runs the what-if on it, and the last warp to finish takes the
// argmin and admits the request. The host sends only the candidate (and its
// Monte-Carlo lengths) and reads back the decision.
struct FleetDev {
  int64_t t_prev;        // last dispatch instant (-1: none)
  int32_t n_req;         // requests admitted so far
  int32_t done;          // warps finished in the current call
  int32_t chosen;
  int32_t status;
  int64_t end_ticks;
};

constexpr int kFleetWarps = 4;

// Per-call inputs of a fleet dispatch, staged in pinned memory and copied by the
// call's CUDA graph (so a dispatch is one graph launch).
struct FleetParams {
  int64_t now;
  int32_t prompt, est, output, S, objective, drain;
  int32_t sample, pad;  // sample: draw the S lengths on the device (K3) instead of lens
  uint64_t request_id, seed;
  double scale;         // mean_abs_rel_error * sqrt(pi / 2)
  int32_t lens[1024];   // sorted MC lengths, S of them (sample == 0)
};

template <int K, bool POW2, bool MC>
__global__ void __launch_bounds__(kFleetWarps * 32)
    fleet_dispatch_kernel(const DevCfg* __restrict__ cfgs, int32_t cfg_index, int32_t n_inst, int32_t n_cap,
                          Arena ar, ClInst* __restrict__ inst, FleetDev* __restrict__ fd,
                          bsg_request_outcome* __restrict__ outs, const FleetParams* __restrict__ P,
                          bsg_result* __restrict__ res, int64_t* __restrict__ scores) {
  const int64_t now = P->now;
  const int32_t prompt = P->prompt, est = P->est, output = P->output, S = P->S,
                objective = P->objective, drain = P->drain;
  const int32_t* sorted_len = P->lens;
  extern __shared__ __align__(16) int32_t fsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t i = blockIdx.x * kFleetWarps + warp;
  if (i >= n_inst) return;
  int32_t* smem = fsm + warp * (smem_words(K, BSG_WIN_J_LATENCY) + pow2_ceil(S));
  int32_t* len = smem + smem_words(K, BSG_WIN_J_LATENCY);
  const DevCfg cfg = cfgs[cfg_index];
  DevCfg live_cfg = cfg;
  live_cfg.cache_mode = BSG_CACHE_OFF;  // live steps use batch_latency itself
  const int32_t maxb = cfg.max_batch_size;
  const int64_t stride = inst_stride(maxb, n_cap);
  const int64_t Rb = static_cast<int64_t>(i) * stride, Ab = Rb + maxb;
  ClInst s = inst[i];  // warp-uniform working copy; written back before the hand-off
  const int64_t tc = __ldcg(&fd->t_prev);
  int32_t err = BSG_OK;
  int64_t last_done = 0;
  // close the previous instant, then every completion strictly before `now`
  if (tc >= 0 && tc != now) {
    if (s.mid && s.t_done == tc) {
      live_finish<K, POW2>(cfg, ar, Rb, s, tc, outs, 0.0, 0, nullptr);
      last_done = tc;
    }
    if (!s.mid && (s.n > 0 || s.whead < s.wtail))
      err = live_begin<K, POW2>(live_cfg, ar, Rb, Ab, s, tc, outs, nullptr);
  }
  while (err == BSG_OK && s.mid && s.t_done < now) {
    const int64_t t = s.t_done;
    live_finish<K, POW2>(cfg, ar, Rb, s, t, outs, 0.0, 0, nullptr);
    last_done = t;
    if (s.n > 0 || s.whead < s.wtail) err = live_begin<K, POW2>(live_cfg, ar, Rb, Ab, s, t, outs, nullptr);
  }
  if (last_done > 0 && lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&fd->end_ticks),
                                            static_cast<unsigned long long>(last_done));
  if (!drain && err == BSG_OK) {
    // the what-if on the live state, in place (predict(), predictor.cpp:76-137)
    bsg_scenario sc;
    sc.run_off = static_cast<int32_t>(Rb);
    sc.run_n = s.n;
    sc.wait_off = static_cast<int32_t>(Ab + s.whead);
    sc.wait_n = s.wtail - s.whead;
    sc.cand_prompt = prompt;
    sc.cand_est = est;
    sc.cfg = cfg_index;
    sc.reserved = 0;
    if constexpr (MC) {
      if (P->sample) {
        stage_mc_samples(len, est, P->request_id, S, P->seed, P->scale, nullptr);
      } else {
        for (int32_t j = lane; j < S; j += 32) len[j] = sorted_len[j];
        __syncwarp();
      }
      simulate_scenario<K, false, true, POW2, false, false, BSG_WIN_J_LATENCY, BSG_CYC_LATENCY>(cfg, ar.prompt, ar.est, ar.prefill, ar.decoded, sc,
                                                    smem, &res[i], TraceSink{nullptr, 0},
                                                    McArgs{len, S, nullptr, &scores[i], objective});
    } else {
      simulate_scenario<K, false, false, POW2, false, false, BSG_WIN_J_LATENCY, BSG_CYC_LATENCY>(
          cfg, ar.prompt, ar.est, ar.prefill, ar.decoded, sc, smem, &res[i], TraceSink{nullptr, 0});
      __syncwarp();
      if (lane == 0) {
        const bsg_result r = res[i];
        scores[i] = r.status != BSG_OK ? INT64_MAX : (objective == 1 ? r.ttft_ticks : r.e2e_ticks);
      }
    }
  } else if (lane == 0) {
    bsg_result r{};
    r.status = err;
    res[i] = r;
    scores[i] = INT64_MAX;
  }
  if (lane == 0) inst[i] = s;
  // the last warp to finish takes the argmin (scheduler.cpp:138-150) and admits
  __threadfence();
  int32_t prev = 0;
  if (lane == 0) prev = atomicAdd(&fd->done, 1);
  prev = __shfl_sync(kFull, prev, 0);
  if (prev != n_inst - 1) return;
  __threadfence();
  int64_t best_v = INT64_MAX;
  int32_t best_i = INT32_MAX, bad = BSG_OK;
  for (int32_t q = lane; q < n_inst; q += 32) {
    const int32_t stq = __ldcg(&res[q].status);
    if (stq != BSG_OK && bad == BSG_OK) bad = stq;
    const int64_t v = __ldcg(&scores[q]);
    if (v < best_v || (v == best_v && q < best_i)) {
      best_v = v;
      best_i = q;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const int64_t ov = __shfl_xor_sync(kFull, best_v, d);
    const int32_t oi = __shfl_xor_sync(kFull, best_i, d);
    if (ov < best_v || (ov == best_v && oi < best_i)) {
      best_v = ov;
      best_i = oi;
    }
  }
  bad = static_cast<int32_t>(__reduce_max_sync(kFull, static_cast<uint32_t>(bad)));
  if (lane != 0) return;
  fd->done = 0;
  if (drain) {
    fd->status = bad;
    return;
  }
  fd->t_prev = now;
  if (bad != BSG_OK || fd->n_req >= n_cap) {
    fd->status = bad != BSG_OK ? bad : BSG_INVALID_ARGUMENT;
    fd->chosen = -1;
    return;
  }
  ClInst& c = inst[best_i];
  const int32_t k = fd->n_req++;
  const int64_t g = static_cast<int64_t>(best_i) * stride + maxb + c.wtail;
  ar.prompt[g] = prompt;
  ar.est[g] = est;
  ar.prefill[g] = 0;
  ar.decoded[g] = 0;
  ar.target[g] = output;
  ar.rid[g] = k;
  c.wtail += 1;
  c.wland = c.wtail;
  bsg_request_outcome o;
  o.arrival_ticks = now;
  o.dispatch_ticks = now;
  o.first_token_ticks = -1;
  o.finish_ticks = -1;
  o.instance = best_i;
  o.preempt_count = 0;
  outs[k] = o;
  fd->chosen = best_i;
  fd->status = BSG_OK;
}

}  // namespace bsg

using namespace bsg;

namespace {

template <int K, bool POW2>
bsg_status launch_closed_loop(bsg_ctx* ctx, int32_t n_runs, const ClRun* runs,
                              const int32_t* p, const int32_t* o, const int32_t* e,
                              const int64_t* arr, const Arena& ar, bsg_request_outcome* outs,
                              bsg_replay_summary* sums, int32_t* st, bsg_run_report* rep) {
  const size_t sm = sizeof(ClShared<K>);
  cudaFuncSetAttribute(closed_loop_kernel<K, POW2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(sm));
  closed_loop_kernel<K, POW2><<<n_runs, kClWarps * 32, sm, ctx->stream>>>(
      static_cast<const DevCfg*>(ctx->cfgs.p), runs, p, o, e, arr, ar, outs, sums, st, rep);
  ctx->launches += 1;
  const cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BSG_OK : bsg_cuda_fail(ctx, err, "closed_loop_kernel launch");
}

}  // namespace

extern "C" bsg_status bsg_replay_device(bsg_ctx* ctx, const bsg_closed_loop_run* runs,
                                        int32_t n_runs, const int32_t* prompt,
                                        const int32_t* output, const int32_t* est,
                                        const int64_t* arrival_ticks, int64_t n_requests_total,
                                        bsg_request_outcome* outcomes,
                                        bsg_replay_summary* summaries, int32_t* run_status,
                                        bsg_run_report* reports) {
  if (!ctx || !runs || n_runs < 0 || !prompt || !output || !est || !arrival_ticks || !run_status)
    return BSG_INVALID_ARGUMENT;
  if (n_runs == 0) return BSG_OK;
  if (ctx->ncfg == 0) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  // host-side layout: arena offsets, validation (driver.cpp config checks)
  std::vector<ClRun> dr(static_cast<size_t>(n_runs));
  int64_t arena = 0;
  int32_t maxb_all = 1;
  bool pow2 = true;
  for (int32_t r = 0; r < n_runs; ++r) {
    const bsg_closed_loop_run& x = runs[r];
    if (x.cfg < 0 || x.cfg >= ctx->ncfg || x.n_instances < 1 || x.n_instances > kClMaxInst ||
        x.n_requests < 0 || x.req_off < 0 || x.req_off + x.n_requests > n_requests_total ||
        x.objective < 0 || x.objective > 1 || x.provision_kind < 0 || x.provision_kind > 2 ||
        (x.provision_kind != 0 && x.max_instances > kClMaxInst) || x.policy < BSG_POLICY_RANDOM ||
        x.policy > BSG_POLICY_BLOCK_PREDICTIVE) {
      ctx->last_error = "bad closed-loop run descriptor";
      return BSG_INVALID_ARGUMENT;
    }
    // validate_provision_policy (autoscaler.cpp:23-34), config.cpp:177-180
    if (!(x.threshold_s > 0) || x.cold_start_s < 0 || x.cooldown_s < 0 ||
        (x.provision_kind != 0 && x.max_instances < x.n_instances) ||
        !(x.dispatch_overhead_s >= 0))  // config.cpp:189-190
      return BSG_BAD_CONFIG;
    const int32_t slots = x.provision_kind == 0 ? x.n_instances : x.max_instances;
    const bsg_instance_cfg& c = ctx->host_cfgs[x.cfg];
    maxb_all = std::max(maxb_all, c.max_batch_size);
    pow2 &= ctx->dev_cfgs_host[x.cfg].div_magic == 0;
    for (int64_t q = x.req_off; q < x.req_off + x.n_requests; ++q) {
      // the workload must be servable (config.cpp:197-205)
      const int64_t need = (static_cast<int64_t>(prompt[q]) + output[q] + c.block_size - 1) / c.block_size;
      if (need > c.total_blocks) return BSG_TOO_LARGE_CANDIDATE;
      if (prompt[q] < 1 || prompt[q] > (1 << 22) || output[q] < 1 || output[q] > (1 << 24) ||
          est[q] < 0 || est[q] > (1 << 24) || (q > x.req_off && arrival_ticks[q] < arrival_ticks[q - 1])) {
        ctx->last_error = "closed-loop request outside the supported domain";
        return BSG_BAD_INPUT;
      }
    }
    dr[r] = ClRun{x.n_instances, x.objective, x.cfg, x.n_requests, x.req_off, arena,
                  x.provision_kind, x.provision_kind == 0 ? x.n_instances : x.max_instances,
                  x.threshold_s, std::llround(x.cold_start_s * 1e9), std::llround(x.cooldown_s * 1e9),
                  x.policy, x.dispatch_overhead_s == 0 ? 1 : 0, x.policy_seed,
                  std::llround(x.dispatch_overhead_s * 1e9)};
    arena += static_cast<int64_t>(slots) * (2 * static_cast<int64_t>(c.max_batch_size) + x.n_requests);
  }
  if (arena >= (int64_t{1} << 31)) {
    ctx->last_error = "closed-loop arena exceeds 2^31 entries; split the batch";
    return BSG_BAD_INPUT;
  }
  int k = 1;
  while (32 * k < maxb_all) k *= 2;
  if (k > 8) return BSG_BAD_INPUT;
  // device buffers (one allocation, freed at the end of the call)
  const int64_t nq = n_requests_total;
  const size_t b_runs = n_runs * sizeof(ClRun), b_req = nq * 4, b_arr = nq * 8,
               b_out = nq * sizeof(bsg_request_outcome), b_sum = n_runs * sizeof(bsg_replay_summary),
               b_st = n_runs * 4, b_col = static_cast<size_t>(std::max<int64_t>(arena, 1)) * 4,
               b_rep = reports ? n_runs * sizeof(bsg_run_report) : 0;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t total = up(b_runs) + 3 * up(b_req) + up(b_arr) + up(b_out) + up(b_sum) + up(b_st) +
                       7 * up(b_col) + up(b_rep);
  char* base = nullptr;
  cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&base), total, ctx->stream);
  if (ce != cudaSuccess) return bsg_cuda_fail(ctx, ce, "cudaMallocAsync(closed-loop)");
  size_t off = 0;
  auto take = [&](size_t b) {
    char* p = base + off;
    off += up(b);
    return p;
  };
  auto* d_runs = reinterpret_cast<ClRun*>(take(b_runs));
  auto* d_p = reinterpret_cast<int32_t*>(take(b_req));
  auto* d_o = reinterpret_cast<int32_t*>(take(b_req));
  auto* d_e = reinterpret_cast<int32_t*>(take(b_req));
  auto* d_a = reinterpret_cast<int64_t*>(take(b_arr));
  auto* d_out = reinterpret_cast<bsg_request_outcome*>(take(b_out));
  auto* d_sum = reinterpret_cast<bsg_replay_summary*>(take(b_sum));
  auto* d_st = reinterpret_cast<int32_t*>(take(b_st));
  auto* d_rep = reports ? reinterpret_cast<bsg_run_report*>(take(b_rep)) : nullptr;
  Arena ar{};
  int32_t** cols[7] = {&ar.prompt, &ar.est, &ar.prefill, &ar.decoded, &ar.target, &ar.rid, &ar.chunk};
  for (auto* c : cols) *c = reinterpret_cast<int32_t*>(take(b_col));
  // outcomes start as the driver's Request records: arrival set, the rest unset
  std::vector<bsg_request_outcome> init(static_cast<size_t>(nq));
  for (int64_t q = 0; q < nq; ++q) init[q] = bsg_request_outcome{arrival_ticks[q], -1, -1, -1, -1, 0};
  cudaStream_t s = ctx->stream;
  bsg_status st = BSG_OK;
#define BSG_CL_CHECK(call)                                  \
  do {                                                      \
    cudaError_t _e = (call);                                \
    if (_e != cudaSuccess && st == BSG_OK) st = bsg_cuda_fail(ctx, _e, #call); \
  } while (0)
  BSG_CL_CHECK(cudaMemcpyAsync(d_runs, dr.data(), b_runs, cudaMemcpyHostToDevice, s));
  BSG_CL_CHECK(cudaMemcpyAsync(d_p, prompt, b_req, cudaMemcpyHostToDevice, s));
  BSG_CL_CHECK(cudaMemcpyAsync(d_o, output, b_req, cudaMemcpyHostToDevice, s));
  BSG_CL_CHECK(cudaMemcpyAsync(d_e, est, b_req, cudaMemcpyHostToDevice, s));
  BSG_CL_CHECK(cudaMemcpyAsync(d_a, arrival_ticks, b_arr, cudaMemcpyHostToDevice, s));
  BSG_CL_CHECK(cudaMemcpyAsync(d_out, init.data(), b_out, cudaMemcpyHostToDevice, s));
  if (st == BSG_OK) {
    switch (k * 2 + (pow2 ? 1 : 0)) {
      case 2: st = launch_closed_loop<1, false>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
      case 3: st = launch_closed_loop<1, true>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
      case 4: st = launch_closed_loop<2, false>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
      case 5: st = launch_closed_loop<2, true>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
      case 8: st = launch_closed_loop<4, false>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
      case 9: st = launch_closed_loop<4, true>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
      case 16: st = launch_closed_loop<8, false>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
      default: st = launch_closed_loop<8, true>(ctx, n_runs, d_runs, d_p, d_o, d_e, d_a, ar, d_out, d_sum, d_st, d_rep); break;
    }
  }
  if (st == BSG_OK) {
    if (outcomes) BSG_CL_CHECK(cudaMemcpyAsync(outcomes, d_out, b_out, cudaMemcpyDeviceToHost, s));
    if (reports) BSG_CL_CHECK(cudaMemcpyAsync(reports, d_rep, b_rep, cudaMemcpyDeviceToHost, s));
    if (summaries) BSG_CL_CHECK(cudaMemcpyAsync(summaries, d_sum, b_sum, cudaMemcpyDeviceToHost, s));
    BSG_CL_CHECK(cudaMemcpyAsync(run_status, d_st, b_st, cudaMemcpyDeviceToHost, s));
  }
  BSG_CL_CHECK(cudaFreeAsync(base, s));
  BSG_CL_CHECK(cudaStreamSynchronize(s));
#undef BSG_CL_CHECK
  if (st == BSG_OK) {
    int64_t whatifs = 0;
    for (int32_t r = 0; r < n_runs; ++r) whatifs += static_cast<int64_t>(runs[r].n_instances) * runs[r].n_requests;
    ctx->scenarios += whatifs;
  }
  return st;
}

// ---- fleet host side ------------------------------------------------------------
struct bsg_fleet {
  bsg_ctx* ctx;
  int32_t cfg, n_inst, n_cap, k;
  bool pow2;
  char* base = nullptr;  // device allocation
  Arena ar{};
  ClInst* inst = nullptr;
  FleetDev* fd = nullptr;
  bsg_request_outcome* outs = nullptr;
  bsg_result* res = nullptr;
  int64_t* scores = nullptr;
  FleetParams* dparams = nullptr;  // device copy of the call's inputs
  FleetParams* hparams = nullptr;  // pinned staging of the call's inputs
  void* pinned = nullptr;          // pinned (chosen, status) + scores out
  int64_t last_now = -1;
  // one instantiated graph (params H2D -> kernel -> decision D2H) per sample count
  std::map<int32_t, cudaGraphExec_t> graphs;
};

namespace {

// Enqueues the fleet kernel on the context stream; inputs come from f->dparams.
template <int K, bool POW2, bool MC>
cudaError_t launch_fleet(bsg_fleet* f, int32_t S) {
  const size_t sm = static_cast<size_t>(kFleetWarps) * (smem_words(K, BSG_WIN_J_LATENCY) + pow2_ceil(S)) * 4;
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(fleet_dispatch_kernel<K, POW2, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm));
  const int blocks = (f->n_inst + kFleetWarps - 1) / kFleetWarps;
  fleet_dispatch_kernel<K, POW2, MC><<<blocks, kFleetWarps * 32, sm, f->ctx->stream>>>(
      static_cast<const DevCfg*>(f->ctx->cfgs.p), f->cfg, f->n_inst, f->n_cap, f->ar, f->inst, f->fd,
      f->outs, f->dparams, f->res, f->scores);
  return cudaGetLastError();
}

cudaError_t launch_fleet_any(bsg_fleet* f, int32_t S, bool mc) {
#define BSG_FLEET_CASE(KK)                                                                           \
  case KK:                                                                                           \
    if (mc) return f->pow2 ? launch_fleet<KK, true, true>(f, S) : launch_fleet<KK, false, true>(f, S); \
    return f->pow2 ? launch_fleet<KK, true, false>(f, S) : launch_fleet<KK, false, false>(f, S);
  switch (f->k) {
    BSG_FLEET_CASE(1)
    BSG_FLEET_CASE(2)
    BSG_FLEET_CASE(4)
    default:
      BSG_FLEET_CASE(8)
  }
#undef BSG_FLEET_CASE
}

// The dispatch sequence: params H2D, the kernel, the decision (+ scores) D2H.
cudaError_t enqueue_dispatch(bsg_fleet* f, int32_t S, bool mc) {
  cudaStream_t s = f->ctx->stream;
  auto* hout = reinterpret_cast<int32_t*>(f->pinned);
  auto* hsc = reinterpret_cast<int64_t*>(static_cast<char*>(f->pinned) + 64);
  cudaError_t e = cudaMemcpyAsync(f->dparams, f->hparams, offsetof(FleetParams, lens) + S * 4,
                                  cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_fleet_any(f, S, mc);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hout, &f->fd->chosen, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hsc, f->scores, f->n_inst * 8, cudaMemcpyDeviceToHost, s);
  return e;
}

}  // namespace

extern "C" bsg_status bsg_fleet_create(bsg_ctx* ctx, int32_t cfg, int32_t n_instances,
                                       int32_t max_requests, bsg_fleet** out) {
  if (!ctx || !out || n_instances < 1 || max_requests < 1) return BSG_INVALID_ARGUMENT;
  *out = nullptr;
  if (cfg < 0 || cfg >= ctx->ncfg) return BSG_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  const bsg_instance_cfg& c = ctx->host_cfgs[cfg];
  int k = 1;
  while (32 * k < c.max_batch_size) k *= 2;
  if (k > 8) return BSG_BAD_INPUT;
  const int64_t entries = static_cast<int64_t>(n_instances) * (2 * static_cast<int64_t>(c.max_batch_size) + max_requests);
  if (entries >= (int64_t{1} << 31)) return BSG_BAD_INPUT;
  auto* f = new bsg_fleet();
  f->ctx = ctx;
  f->cfg = cfg;
  f->n_inst = n_instances;
  f->n_cap = max_requests;
  f->k = k;
  f->pow2 = ctx->dev_cfgs_host[cfg].div_magic == 0;
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t b_col = up(static_cast<size_t>(entries) * 4), b_inst = up(n_instances * sizeof(ClInst)),
               b_fd = up(sizeof(FleetDev)), b_out = up(static_cast<size_t>(max_requests) * sizeof(bsg_request_outcome)),
               b_res = up(n_instances * sizeof(bsg_result)), b_sc = up(n_instances * 8),
               b_len = up(sizeof(FleetParams));
  const size_t total = 7 * b_col + b_inst + b_fd + b_out + b_res + b_sc + b_len;
  if (cudaMalloc(&f->base, total) != cudaSuccess) {
    cudaGetLastError();
    delete f;
    ctx->last_error = "fleet allocation failed";
    return BSG_CUDA_ERROR;
  }
  char* p = f->base;
  int32_t** cols[7] = {&f->ar.prompt, &f->ar.est, &f->ar.prefill, &f->ar.decoded, &f->ar.target, &f->ar.rid, &f->ar.chunk};
  for (auto* col : cols) {
    *col = reinterpret_cast<int32_t*>(p);
    p += b_col;
  }
  f->inst = reinterpret_cast<ClInst*>(p);
  p += b_inst;
  f->fd = reinterpret_cast<FleetDev*>(p);
  p += b_fd;
  f->outs = reinterpret_cast<bsg_request_outcome*>(p);
  p += b_out;
  f->res = reinterpret_cast<bsg_result*>(p);
  p += b_res;
  f->scores = reinterpret_cast<int64_t*>(p);
  p += b_sc;
  f->dparams = reinterpret_cast<FleetParams*>(p);
  std::vector<ClInst> init(static_cast<size_t>(n_instances));
  for (auto& x : init) x = ClInst{0, c.max_batch_size, c.max_batch_size, c.total_blocks, 0, 0, c.max_batch_size, 0, 0};
  FleetDev fd0{-1, 0, 0, -1, BSG_OK, 0};
  bool ok = cudaHostAlloc(&f->pinned, 64 + static_cast<size_t>(n_instances) * 8, cudaHostAllocDefault) == cudaSuccess;
  ok = ok && cudaHostAlloc(reinterpret_cast<void**>(&f->hparams), sizeof(FleetParams), cudaHostAllocDefault) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(f->inst, init.data(), n_instances * sizeof(ClInst), cudaMemcpyHostToDevice, ctx->stream) == cudaSuccess;
  ok = ok && cudaMemcpyAsync(f->fd, &fd0, sizeof(fd0), cudaMemcpyHostToDevice, ctx->stream) == cudaSuccess;
  ok = ok && cudaStreamSynchronize(ctx->stream) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    if (f->pinned) cudaFreeHost(f->pinned);
    if (f->hparams) cudaFreeHost(f->hparams);
    cudaFree(f->base);
    delete f;
    ctx->last_error = "fleet initialisation failed";
    return BSG_CUDA_ERROR;
  }
  *out = f;
  return BSG_OK;
}

extern "C" void bsg_fleet_destroy(bsg_fleet* f) {
  if (!f) return;
  cudaSetDevice(f->ctx->device);
  cudaStreamSynchronize(f->ctx->stream);
  for (auto& g : f->graphs) cudaGraphExecDestroy(g.second);
  if (f->pinned) cudaFreeHost(f->pinned);
  if (f->hparams) cudaFreeHost(f->hparams);
  cudaFree(f->base);
  delete f;
}

namespace {

// One fleet dispatch: given sorted-on-host lengths (lengths != nullptr), device-
// drawn samples (sample), or the estimate alone.
bsg_status fleet_dispatch(bsg_fleet* f, int64_t now_ticks, int32_t prompt, int32_t est, int32_t output,
                          const int32_t* lengths, bool sample, uint64_t request_id, uint64_t seed,
                          double mean_abs_rel_error, int32_t n_samples, int32_t objective, int32_t* chosen,
                          int64_t* scores) {
  if (!f || !chosen || now_ticks < 0 || objective < 0 || objective > 1) return BSG_INVALID_ARGUMENT;
  if (now_ticks < f->last_now) return BSG_INVALID_ARGUMENT;  // arrivals in time order
  if (prompt < 1 || prompt > (1 << 22) || est < 0 || est > (1 << 24) || output < 1 || output > (1 << 24))
    return BSG_BAD_INPUT;
  if (sample && !(mean_abs_rel_error >= 0)) return BSG_INVALID_ARGUMENT;
  const bool mc = lengths != nullptr || sample;
  if (mc && (n_samples < 1 || n_samples > 1024)) return BSG_INVALID_ARGUMENT;
  bsg_ctx* ctx = f->ctx;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  // the workload must be servable (config.cpp:197-205)
  const bsg_instance_cfg& c = ctx->host_cfgs[f->cfg];
  if ((static_cast<int64_t>(prompt) + output + c.block_size - 1) / c.block_size > c.total_blocks)
    return BSG_TOO_LARGE_CANDIDATE;
  auto* hout = reinterpret_cast<int32_t*>(f->pinned);
  auto* hsc = reinterpret_cast<int64_t*>(static_cast<char*>(f->pinned) + 64);
  cudaStream_t s = ctx->stream;
  const int32_t S = mc ? n_samples : 0;
  FleetParams& P = *f->hparams;
  P.now = now_ticks;
  P.prompt = prompt;
  P.est = est;
  P.output = output;
  P.S = S;
  P.objective = objective;
  P.drain = 0;
  P.sample = sample ? 1 : 0;
  P.request_id = request_id;
  P.seed = seed;
  P.scale = mean_abs_rel_error * std::sqrt(3.14159265358979323846 / 2.0);
  if (lengths) {
    std::memcpy(P.lens, lengths, S * 4);
    std::sort(P.lens, P.lens + S);  // the kernel walks the samples in ascending order
  }
  // One CUDA graph per sample count (params H2D -> kernel -> decision D2H),
  // captured on first use: a dispatch is a single graph launch.
  static const bool no_graph = std::getenv("BSG_FLEET_NO_GRAPH") != nullptr;
  cudaError_t e = cudaSuccess;
  if (no_graph) {
    e = enqueue_dispatch(f, S, mc);
  } else {
    const int32_t gkey = mc ? (sample ? -S : S) : 0;  // the graph's H2D copies lens only when given
    auto it = f->graphs.find(gkey);
    if (it == f->graphs.end()) {
      cudaGraph_t g = nullptr;
      cudaGraphExec_t x = nullptr;
      e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        const cudaError_t qe = enqueue_dispatch(f, S, mc);
        e = cudaStreamEndCapture(s, &g);
        if (e == cudaSuccess) e = qe;
      }
      if (e == cudaSuccess) e = cudaGraphInstantiate(&x, g, 0);
      if (g) cudaGraphDestroy(g);
      if (e != cudaSuccess) return bsg_cuda_fail(ctx, e, "fleet graph capture");
      it = f->graphs.emplace(gkey, x).first;
    }
    e = cudaGraphLaunch(it->second, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return bsg_cuda_fail(ctx, e, "fleet dispatch");
  ctx->launches += 1;
  f->last_now = now_ticks;
  ctx->scenarios += static_cast<int64_t>(f->n_inst) * (mc ? S : 1);
  *chosen = hout[0];
  if (scores) std::memcpy(scores, hsc, f->n_inst * 8);
  if (hout[1] != BSG_OK) {
    ctx->last_error = "fleet dispatch failed (see status)";
    return static_cast<bsg_status>(hout[1]);
  }
  return BSG_OK;
}

}  // namespace

extern "C" bsg_status bsg_fleet_dispatch(bsg_fleet* f, int64_t now_ticks, int32_t prompt, int32_t est,
                                         int32_t output, const int32_t* lengths, int32_t n_samples,
                                         int32_t objective, int32_t* chosen, int64_t* scores) {
  return fleet_dispatch(f, now_ticks, prompt, est, output, lengths, false, 0, 0, 0.0, n_samples, objective,
                        chosen, scores);
}

extern "C" bsg_status bsg_fleet_dispatch_sampled(bsg_fleet* f, int64_t now_ticks, int32_t prompt, int32_t est,
                                                 int32_t output, uint64_t request_id, int32_t n_samples,
                                                 uint64_t seed, double mean_abs_rel_error, int32_t objective,
                                                 int32_t* chosen, int64_t* scores) {
  return fleet_dispatch(f, now_ticks, prompt, est, output, nullptr, true, request_id, seed,
                        mean_abs_rel_error, n_samples, objective, chosen, scores);
}

extern "C" bsg_status bsg_fleet_finish(bsg_fleet* f, bsg_request_outcome* outcomes, int32_t* n_requests,
                                       bsg_replay_summary* summary) {
  if (!f || !outcomes || !n_requests) return BSG_INVALID_ARGUMENT;
  bsg_ctx* ctx = f->ctx;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  FleetParams& P = *f->hparams;  // drain: run every remaining step
  P.now = INT64_MAX;
  P.prompt = P.est = P.output = 1;
  P.S = 0;
  P.objective = 0;
  P.drain = 1;
  cudaError_t e = cudaMemcpyAsync(f->dparams, f->hparams, offsetof(FleetParams, lens),
                                  cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_fleet_any(f, 0, false);
  ctx->launches += 1;
  FleetDev fd{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&fd, f->fd, sizeof(fd), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && fd.n_req > 0)
    e = cudaMemcpy(outcomes, f->outs, static_cast<size_t>(fd.n_req) * sizeof(bsg_request_outcome),
                   cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return bsg_cuda_fail(ctx, e, "fleet finish");
  *n_requests = fd.n_req;
  if (summary) {
    std::memset(summary, 0, sizeof(*summary));
    int64_t pre = 0;
    for (int32_t q = 0; q < fd.n_req; ++q) pre += outcomes[q].preempt_count;
    summary->total_preemptions = pre;
    summary->end_ticks = std::max(fd.end_ticks, fd.t_prev);
    summary->final_instance_count = f->n_inst;
  }
  return fd.status == BSG_OK ? BSG_OK : static_cast<bsg_status>(fd.status);
}

extern "C" bsg_status bsg_fleet_snapshot(bsg_fleet* f, int32_t instance, int32_t* run_n, int32_t* wait_n,
                                         int32_t* prompt, int32_t* est, int32_t* prefill,
                                         int32_t* decoded, int32_t cap) {
  if (!f || !run_n || !wait_n || instance < 0 || instance >= f->n_inst) return BSG_INVALID_ARGUMENT;
  bsg_ctx* ctx = f->ctx;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaSetDevice(ctx->device);
  ClInst st{};
  cudaError_t e = cudaMemcpy(&st, f->inst + instance, sizeof(st), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return bsg_cuda_fail(ctx, e, "fleet snapshot");
  *run_n = st.n;
  *wait_n = st.wtail - st.whead;
  if (st.n + *wait_n > cap) return BSG_OK;  // sizes only
  const int32_t maxb = ctx->host_cfgs[f->cfg].max_batch_size;
  const int64_t Rb = static_cast<int64_t>(instance) * (2 * static_cast<int64_t>(maxb) + f->n_cap);
  const int64_t Ab = Rb + maxb + st.whead;
  int32_t* dst[4] = {prompt, est, prefill, decoded};
  int32_t* src[4] = {f->ar.prompt, f->ar.est, f->ar.prefill, f->ar.decoded};
  for (int c = 0; c < 4 && e == cudaSuccess; ++c) {
    if (!dst[c]) continue;
    if (st.n > 0) e = cudaMemcpy(dst[c], src[c] + Rb, st.n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && *wait_n > 0) e = cudaMemcpy(dst[c] + st.n, src[c] + Ab, *wait_n * 4, cudaMemcpyDeviceToHost);
  }
  if (e != cudaSuccess) return bsg_cuda_fail(ctx, e, "fleet snapshot");
  return BSG_OK;
}

// scenario_sim.cuh — K1: warp-per-scenario what-if simulation (sm_100a).
//
// One warp replays one instance's continuous-batching engine forward from a
// snapshot with the candidate appended to the waiting tail, until the
// candidate completes: blocksim predict() (core/src/predictor.cpp:76-137)
// driving Instance::execute_step (core/src/backend.cpp:238-331).
//
// State layout (per warp, in registers): the "resident list" of up to 32*K
// members, position p held by lane p / K, register slot p % K (contiguous, so
// prefix scans are lane-local + one warp scan):
//   positions [0, n)  : running_ in admission order (backend.h:157)
//   positions [n, L)  : preemption victims = the FRONT of waiting_, head first
//   then, virtually   : snapshot.waiting[h..wait_n) (read-only, HBM/L2), then the
//                       candidate if it was never admitted.
// Because the victim of every preemption is the newest running member (the
// running tail) and victims go to the waiting FRONT, preemption is
// "n -= 1" and admission of a victim is "n += 1": both are boundary moves.
//
// Allocation with preemption (backend.cpp:263-288) is evaluated in parallel:
// with F(e) = free + sum_{v>=e} held_old[v] - sum_{items at pos<e} delta, which
// is non-increasing in e, the sequential victim loop ends with exactly
// e* = max{e : F(e) >= 0} survivors, and deadlocks iff e* == 0 (DESIGN.md §4
// derives this). One ballot finds e*.
//
// Floating point: batch_latency's unfused ((c0 + p*T) + d*D) + c*C in double
// (backend.cpp:10-14) with __dmul_rn/__dadd_rn (no contraction), then llround
// (time.h:20-22); elapsed is an int64 tick sum, so results are bit-exact.
#pragma once

#include <cstdint>

#include "../../include/blocksim_b200.h"

namespace bsg {

constexpr unsigned kFull = 0xffffffffu;
// Event-skipping window: WJ steps per lane, 32 * WJ steps per window — a
// template parameter of simulate_scenario, chosen per kernel (measured, see
// DESIGN.md): wide windows for decode-dominated throughput sets and for the
// latency path, narrow ones where events keep windows short.
#ifndef BSG_MAX_WIN_J
#define BSG_MAX_WIN_J 8
#endif
constexpr int kMaxWinJ = BSG_MAX_WIN_J;
#ifndef BSG_WIN_J_PREDICT
#define BSG_WIN_J_PREDICT 4   // K1, 32-member sets (cfg1/cfg2 shape)
#endif
#ifndef BSG_WIN_J_WIDE
#define BSG_WIN_J_WIDE 1      // K1 for wide / KV-pressure sets (and their optimistic pass)
#endif
#ifndef BSG_WIN_J_LATENCY
#define BSG_WIN_J_LATENCY 8   // per-request dispatch (dispatch_mc, fleet): one wave, the longest
#endif                        // simulation is the latency (cfg4 p99 113 -> 100 us vs 128-step windows)
#ifndef BSG_WIN_J_CLOSED
#define BSG_WIN_J_CLOSED 1    // K5 closed-loop what-ifs
#endif
// Admit / self-preempt cycle absorption in the windows (simulate_scenario's
// CYC) for the latency path (dispatch_mc, fleet) and the K5 closed loop; the
// throughput kernels choose per launch shape (bsg_capi.cu). Off by measurement:
// cfg4 p99 116 vs 123 us, cfg5 full grid 0.333 vs 0.355 s (their instances
// rarely thrash; the extra registers cost more than the cycles save).
#ifndef BSG_CYC_LATENCY
#define BSG_CYC_LATENCY 0
#endif
#ifndef BSG_CYC_CLOSED
#define BSG_CYC_CLOSED 0
#endif
// Drain pass (simulate_scenario): once nothing can be admitted any more, the
// steps up to the candidate's completion are priced in one pass (BSG_DRAIN=0:
// windows only, for A/B measurements).
#ifndef BSG_DRAIN
#define BSG_DRAIN 1
#endif
// Per-warp shared-memory words of simulate_scenario with window width WJ: the
// completion-compaction area (5 x 32K) / the window histograms and cycle arrays
// (4 x 32 x WJ), whichever is larger.
__host__ __device__ constexpr int smem_words(int K, int WJ = kMaxWinJ) {
  return (5 * 32 * K > 4 * 32 * WJ ? 5 * 32 * K : 4 * 32 * WJ);
}
constexpr int64_t kMaxSimulatedSteps = 50000000LL;  // predictor.cpp:11

// Device-side config: bsg_instance_cfg + precomputed block-size divisor.
struct DevCfg {
  int32_t total_blocks, block_size, max_batch_size, chunk_budget;
  int32_t local_policy, cache_mode, context_bucket;
  uint32_t div_magic;   // 0 => power of two
  int32_t div_shift;
  int32_t pad[3];
  double c0, cp, cd, cc;
};

// floor(n / block_size) for 0 <= n < 2^31 (Granlund-Montgomery, N = 31).
__device__ __forceinline__ int32_t div_bs(int32_t n, const DevCfg& c) {
  if (c.div_magic == 0) return n >> c.div_shift;
  return static_cast<int32_t>(__umulhi(static_cast<uint32_t>(n), c.div_magic) >> c.div_shift);
}
// blocks_needed (types.cpp:63-66): tokens <= 0 ? 0 : ceil(tokens / block_size).
__device__ __forceinline__ int32_t bn(int32_t t, const DevCfg& c) {
  return t <= 0 ? 0 : div_bs(t + c.block_size - 1, c);
}

// Compile-time specialisation for power-of-two block sizes (the common case):
// division and modulo become a shift and a mask.
template <bool POW2>
__device__ __forceinline__ int32_t divt(int32_t n, const DevCfg& c) {
  if constexpr (POW2) return n >> c.div_shift;
  else return div_bs(n, c);
}
template <bool POW2>
__device__ __forceinline__ int32_t modt(int32_t n, const DevCfg& c) {
  if constexpr (POW2) return n & (c.block_size - 1);
  else return n - div_bs(n, c) * c.block_size;
}
template <bool POW2>
__device__ __forceinline__ int32_t bnt(int32_t t, const DevCfg& c) {
  return t <= 0 ? 0 : divt<POW2>(t + c.block_size - 1, c);
}

// Sum of a per-lane non-negative int64 over the warp: two 32-bit redux.sync
// on 16-bit-split halves when every value is < 2^42, shuffles otherwise.
__device__ __forceinline__ int64_t warp_sum_i64(int64_t d) {
  if (!__any_sync(kFull, d >= (int64_t{1} << 42))) {
    const uint32_t lo = __reduce_add_sync(kFull, static_cast<uint32_t>(d & 0xffff));
    const uint32_t hi = __reduce_add_sync(kFull, static_cast<uint32_t>(d >> 16));
    return (static_cast<int64_t>(hi) << 16) + lo;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(kFull, d, o);
  return d;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Inclusive warp scan: 5 x (shfl.up with its in-range predicate + predicated
// add) — no lane-index compares on the dependent chain.
__device__ __forceinline__ int32_t warp_incl_scan(int32_t x) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    asm("{\n\t.reg .s32 r;\n\t.reg .pred p;\n\t"
        "shfl.sync.up.b32 r|p, %0, %1, 0, -1;\n\t"
        "@p add.s32 %0, %0, r;\n\t}"
        : "+r"(x)
        : "r"(d));
  }
  return x;
}

// Inclusive warp scan of a 64-bit value (e.g. two packed 32-bit counters whose
// low-half sums never carry).
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t x) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    asm("{\n\t.reg .b32 lo, hi;\n\t.reg .b64 y;\n\t.reg .pred p;\n\t"
        "mov.b64 {lo, hi}, %0;\n\t"
        "shfl.sync.up.b32 lo|p, lo, %1, 0, -1;\n\t"
        "shfl.sync.up.b32 hi, hi, %1, 0, -1;\n\t"
        "mov.b64 y, {lo, hi};\n\t"
        "@p add.u64 %0, %0, y;\n\t}"
        : "+l"(x)
        : "r"(d));
  }
  return x;
}

// Exclusive prefix over positions (lane-contiguous layout); returns the total.
template <int K>
__device__ __forceinline__ int32_t excl_scan(const int32_t (&in)[K], int32_t (&out)[K]) {
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    out[k] = s;
    s += in[k];
  }
  const int32_t incl = warp_incl_scan(s);
  const int32_t base = incl - s;
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] += base;
  // the total off the scan's dependent chain
  return static_cast<int32_t>(__reduce_add_sync(kFull, static_cast<uint32_t>(s)));
}

template <int K>
__device__ __forceinline__ int32_t warp_sum(const int32_t (&in)[K]) {
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += in[k];
  return static_cast<int32_t>(__reduce_add_sync(kFull, static_cast<uint32_t>(s)));
}

// Position of the first set flag (or `none`).
template <int K>
__device__ __forceinline__ int32_t first_pos(const bool (&f)[K], int32_t none) {
  int32_t local = none;
#pragma unroll
  for (int k = K - 1; k >= 0; --k)
    if (f[k]) local = lane_id() * K + k;
  return static_cast<int32_t>(__reduce_min_sync(kFull, static_cast<uint32_t>(local)));
}

template <int K>
__device__ __forceinline__ int32_t count(const bool (&f)[K]) {
  int32_t c = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) c += __popc(__ballot_sync(kFull, f[k]));
  return c;
}

// Reads position p's value of a per-lane register array (warp-uniform p).
template <int K>
__device__ __forceinline__ int32_t read_pos(const int32_t (&v)[K], int32_t p) {
  int32_t mine = 0;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (k == p % K) mine = v[k];
  return __shfl_sync(kFull, mine, p / K);
}

// The member "org" word: bit 31 = ever_scheduled (backend.h:124),
// bits 0..30 = origin + 1 (origin: running i -> i, waiting j -> run_n + j,
// candidate -> -1).
__device__ __forceinline__ int32_t org_origin(int32_t w) { return (w & 0x7fffffff) - 1; }
__device__ __forceinline__ bool org_ever(int32_t w) { return (w >> 31) & 1; }
constexpr int32_t kEverBit = static_cast<int32_t>(0x80000000u);
constexpr int32_t kCandOrg = 0;  // origin -1 -> org 0 (never scheduled)

__device__ __forceinline__ uint64_t hash_term(uint32_t tag, uint32_t k, int32_t origin, int32_t v) {
  return bsg_hash_term(tag, k, origin, v);
}

// latency (backend.cpp:10-14; bucketed context predictor.cpp:29-32) -> ticks (time.h:20-22)
__device__ __forceinline__ int64_t step_ticks(const DevCfg& c, int32_t prefill_tokens,
                                              int32_t n_decode, int32_t context) {
  int64_t ctx = context;
  if (c.cache_mode == BSG_CACHE_BUCKETED) {
    const int64_t b = c.context_bucket < 1 ? 1 : c.context_bucket;
    ctx = (ctx + b / 2) / b * b;
  }
  double x = __dadd_rn(c.c0, __dmul_rn(c.cp, static_cast<double>(prefill_tokens)));
  x = __dadd_rn(x, __dmul_rn(c.cd, static_cast<double>(n_decode)));
  x = __dadd_rn(x, __dmul_rn(c.cc, static_cast<double>(ctx)));
  return llround(__dmul_rn(x, 1e9));
}

struct TraceSink {
  bsg_step_record* rec;
  int64_t cap;
};

// Monte-Carlo length samples of the candidate. The samples
// are sorted ascending; the simulation runs once with target = len[S-1] and
// sample j's e2e is the elapsed time at the end of the first step in which the
// candidate's decoded count reaches len[j] (the candidate's target influences
// nothing before its own completion, so this equals running predict() with
// target len[j]; prefix sharing is exact).
struct McArgs {
  const int32_t* len;   // sorted sample lengths (shared memory), S >= 1
  int32_t S;
  int64_t* sample_e2e;  // optional, sorted order
  int64_t* score;       // sum_j e2e_j (or S * ttft for the ttft objective)
  int32_t objective;
};

// Simulates one scenario with the calling warp. All lanes return the same
// result; lane 0 writes it.
// Snapshot loads: read-only-cache loads (__ldg) when the entries are immutable
// for the kernel's lifetime (K1 and the dispatch kernels); coherent L2 loads
// when other warps of the same kernel write them (the device-resident closed
// loop, closed_loop.cu).
template <bool LDG>
__device__ __forceinline__ int32_t ld_entry(const int32_t* p) {
  if constexpr (LDG) return __ldg(p);
  else return __ldcg(p);
}

// Internal status of an optimistic (OPT) narrow simulation whose resident list
// would outgrow its 32K member slots: the caller re-runs it with a wider K.
constexpr int32_t kStatusRetryWider = 100;

template <int K, bool TRACE, bool MC = false, bool POW2 = false, bool LDG = true, bool OPT = false,
          int WJ = 1, bool CYC = true>
__device__ void simulate_scenario(const DevCfg& cfg, const int32_t* __restrict__ g_prompt,
                                  const int32_t* __restrict__ g_est,
                                  const int32_t* __restrict__ g_prefill,
                                  const int32_t* __restrict__ g_decoded, const bsg_scenario sc,
                                  // smem_words(K, WJ) int32 per warp. Not __restrict__: lanes
                                  // exchange values through it across __syncwarp(), which
                                  // a restrict-qualified pointer lets the compiler reorder
                                  // loads across (the barrier does not take the pointer)
                                  int32_t* smem,
                                  bsg_result* __restrict__ out, TraceSink trace,
                                  McArgs mc = McArgs{}) {
  constexpr int CAP = 32 * K;
  // candidate target: its estimate, or the largest MC sample
  const int32_t cand_target = MC ? mc.len[mc.S - 1] : sc.cand_est;
  int32_t cand_hi = 0;     // MC: highest decoded count the candidate has reached
  int32_t mc_ptr = 0;      // MC: samples already completed (sorted prefix)
  int64_t mc_sum = 0;      // MC: per-lane partial score
  const int lane = lane_id();
  bsg_result res{};

  // ---- load running entries: from_snapshot (backend.cpp:24-41) with
  // correct_lengths (predictor.cpp:65-74) applied to est -> target.
  int32_t prompt[K], target[K], prefill[K], decoded[K], org[K];
  const int32_t run_n = sc.run_n;
  bool bad = false;
  int32_t held[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int32_t p = lane * K + k;
    prompt[k] = 1;
    target[k] = 0;
    prefill[k] = 0;
    decoded[k] = 0;
    org[k] = 0;
    held[k] = 0;
    if (p < run_n) {
      const int32_t g = sc.run_off + p;
      prompt[k] = ld_entry<LDG>(g_prompt + g);
      const int32_t est = ld_entry<LDG>(g_est + g);
      prefill[k] = ld_entry<LDG>(g_prefill + g);
      decoded[k] = ld_entry<LDG>(g_decoded + g);
      target[k] = decoded[k] >= est ? decoded[k] + 10 : est;
      org[k] = (p + 1) | kEverBit;
      bad |= prompt[k] < 1 || prompt[k] > (1 << 22) || prefill[k] < 0 || prefill[k] > prompt[k] ||
             decoded[k] < 0 || decoded[k] > (1 << 22) || est > (1 << 24);
      held[k] = bnt<POW2>(prefill[k] + decoded[k], cfg);
    }
  }
  if (__any_sync(kFull, bad) || run_n > CAP) {
    res.status = (OPT && run_n > CAP) ? kStatusRetryWider : BSG_BAD_INPUT;
    if (lane == 0) *out = res;
    return;
  }
  int32_t free_blocks = cfg.total_blocks - warp_sum<K>(held);
  if (free_blocks < 0) {  // backend.cpp:42-44
    res.status = BSG_TOO_LARGE_RUNNING;
    if (lane == 0) *out = res;
    return;
  }
  // waiting entries: validated eagerly (one coalesced pass; the simulation then
  // reads them lazily, only when the waiting head is examined)
  {
    bool badw = false;
    for (int32_t j = lane; j < sc.wait_n; j += 32) {
      const int32_t g = sc.wait_off + j;
      const int32_t pr = ld_entry<LDG>(g_prompt + g);
      const int32_t est = ld_entry<LDG>(g_est + g);
      const int32_t dec = ld_entry<LDG>(g_decoded + g);
      const int32_t tg = dec >= est ? dec + 10 : est;
      badw |= pr < 1 || pr > (1 << 22) || tg > (1 << 24) + 10;
    }
    if (__any_sync(kFull, badw)) {
      res.status = BSG_BAD_INPUT;
      if (lane == 0) *out = res;
      return;
    }
  }
  // the candidate's admit check (backend.cpp:76-83):
  {
    const int64_t need = (static_cast<int64_t>(sc.cand_prompt) + cand_target + cfg.block_size - 1) /
                         cfg.block_size;
    if (sc.cand_prompt < 1 || sc.cand_prompt > (1 << 22) || cand_target < 0 ||
        cand_target > (1 << 24)) {
      res.status = BSG_BAD_INPUT;
      if (lane == 0) *out = res;
      return;
    }
    if (need > cfg.total_blocks) {
      res.status = BSG_TOO_LARGE_CANDIDATE;
      res.detail = static_cast<int32_t>(need);
      if (lane == 0) *out = res;
      return;
    }
  }

  int32_t n = run_n;   // running count
  int32_t L = run_n;   // running + victim stack
  int32_t h = 0;       // next unread snapshot.waiting index
  bool cand_tail = true;
  int64_t elapsed = 0, steps = 0;
  bool qd_set = false, ttft_set = false;
  const int32_t wait_n = sc.wait_n;
  const bool chunked = cfg.local_policy == BSG_CHUNKED_PREFILL;
  const int32_t maxb = cfg.max_batch_size;
#ifdef BSG_PROFILE_DRAIN
  int32_t prof_dr_ok = 0, prof_dr_fail = 0;
#endif
#ifdef BSG_PROFILE_ITERS
  int64_t prof_gen = 0, prof_win = 0, prof_adm = 0, prof_pre = 0, prof_prf = 0;
#endif

  for (;;) {
    const bool waiting_nonempty = (L > n) || (h < wait_n) || cand_tail;
    if (n == 0 && !waiting_nonempty) {  // predictor.cpp:102-104
      res.status = BSG_VANISHED;
      break;
    }
    // ---------------- plan (backend.cpp:113-182) ----------------
    bool ready[K], nonready[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t p = lane * K + k;
      ready[k] = p < n && prefill[k] == prompt[k];
      nonready[k] = p < n && prefill[k] != prompt[k];
    }
    const int32_t D = count<K>(ready);
    bool any_local = false;
#pragma unroll
    for (int k = 0; k < K; ++k) any_local |= nonready[k];
    const bool any_nonready = __any_sync(kFull, any_local);
    int32_t chunk[K];
    bool decode_item[K];
    int32_t budget = 0;  // budget left for waiting admissions (chunked prefill)
    bool prefill_step = false;  // prefill-priority pure-prefill step
    if (chunked) {
      int32_t b0 = cfg.chunk_budget - D;  // one budget token per decode (backend.cpp:116-121)
      if (b0 < 0) b0 = 0;
      budget = b0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        chunk[k] = 0;
        decode_item[k] = ready[k];
      }
      if (any_nonready) {  // running partial prefills in order, break at budget 0 (122-130)
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
    } else {
      prefill_step = waiting_nonempty || any_nonready;  // backend.cpp:152-155
#pragma unroll
      for (int k = 0; k < K; ++k) {
        chunk[k] = (prefill_step && nonready[k]) ? prompt[k] - prefill[k] : 0;
        decode_item[k] = !prefill_step && ready[k];
      }
    }
    // deltas of running items (make_item, backend.cpp:94-111) — computed only
    // when a waiting head is examined or a general step runs: a pure-decode
    // window derives its block demand itself
    int32_t delta[K], stored[K];
#pragma unroll
    for (int k = 0; k < K; ++k) stored[k] = prefill[k] + decoded[k];
    bool delta_ready = false;
    auto running_deltas = [&]() {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        int32_t ns = stored[k];
        if (decode_item[k]) {
          ns = stored[k] + 1;
        } else if (chunk[k] > 0) {
          const int32_t np = prefill[k] + chunk[k];
          ns = np + decoded[k] + (np == prompt[k] ? 1 : 0);
        }
        delta[k] = (decode_item[k] || chunk[k] > 0) ? bnt<POW2>(ns, cfg) - bnt<POW2>(stored[k], cfg) : 0;
      }
      delta_ready = true;
    };

    // ---------------- waiting admissions ----------------
    int32_t a = 0;  // admitted waiting heads
    int32_t run_delta = 0;
    // this step admits a preemption victim's first chunk (< its prompt) and
    // nothing else: the first step of an admit / self-preempt cycle the window
    // below may absorb
    bool cyc0 = false;
    int32_t cyc_hp = 0;  // its prompt
    bool try_admit = waiting_nonempty && n < maxb && (chunked ? budget > 0 : true);
    if (try_admit) {
      running_deltas();
      run_delta = warp_sum<K>(delta);
    }
    if (try_admit) {
      // Fast reject: admission is a prefix of the waiting queue, so when the
      // head's first chunk does not fit projected_free (backend.cpp:141-142)
      // nothing is admitted — decided from one entry instead of materialising
      // the queue (KV-pressure sets spend most steps here).
      int32_t hp;
      if (L > n) hp = read_pos<K>(prompt, n);  // victims: the waiting front
      else if (h < wait_n) hp = ld_entry<LDG>(g_prompt + sc.wait_off + h);
      else hp = sc.cand_prompt;
      const int32_t hc = chunked ? (hp < budget ? hp : budget) : hp;
      if (bnt<POW2>(hc + (hc == hp ? 1 : 0), cfg) > free_blocks - run_delta) {
        try_admit = false;
      } else if (chunked && hp >= budget && n < CAP) {  // (n == CAP: the general path decides)
        // Single admission: the head fits and its first chunk takes the whole
        // remaining budget, so the loop stops right after it (backend.cpp:136):
        // admit exactly the head without materialising the queue.
        try_admit = false;
        a = 1;
        cyc0 = CYC && L > n && hp > budget;
        cyc_hp = hp;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int32_t p = lane * K + k;
          if (p == n) {
            if (p >= L) {
              if (h < wait_n) {
                const int32_t g = sc.wait_off + h;
                prompt[k] = hp;
                const int32_t est = ld_entry<LDG>(g_est + g);
                const int32_t dec = ld_entry<LDG>(g_decoded + g);
                target[k] = dec >= est ? dec + 10 : est;  // correct_lengths on waiting too
                org[k] = run_n + h + 1;
              } else {
                prompt[k] = sc.cand_prompt;
                target[k] = cand_target;
                org[k] = kCandOrg;
              }
              prefill[k] = 0;
              decoded[k] = 0;
            }
            chunk[k] = hc;
            delta[k] = bnt<POW2>(hc + (hc == hp ? 1 : 0), cfg);
          }
        }
      }
    }
    if (try_admit) {
      const int32_t pf = free_blocks - run_delta;  // projected_free (backend.cpp:131-133 / 158-164)
      // Materialise waiting heads at positions [L, CAP): snapshot.waiting[h..], then candidate.
      bool valid[K];
      int32_t wprompt[K], fdelta[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        valid[k] = p >= n && p < maxb;
        if (p >= L) {
          const int32_t j = h + (p - L);
          if (j < wait_n) {
            const int32_t g = sc.wait_off + j;
            prompt[k] = ld_entry<LDG>(g_prompt + g);
            const int32_t est = ld_entry<LDG>(g_est + g);
            const int32_t dec = ld_entry<LDG>(g_decoded + g);
            target[k] = dec >= est ? dec + 10 : est;  // correct_lengths on waiting too
            org[k] = run_n + j + 1;
          } else if (j == wait_n && cand_tail) {
            prompt[k] = sc.cand_prompt;
            target[k] = cand_target;
            org[k] = kCandOrg;
          } else {
            valid[k] = false;
          }
          prefill[k] = 0;
          decoded[k] = 0;
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
        if (ok) chunk[k] = c;
        stop[k] = p >= n && !ok;
        if (ok) delta[k] = dj;
      }
      const int32_t first_stop = first_pos<K>(stop, CAP);
      a = first_stop - n;
      if constexpr (OPT) {
        // every slot admitted while the batch cap allows more and more waiting
        // entries exist: the wider kernel must decide (resident list > 32K)
        if (first_stop == CAP && CAP < maxb &&
            (L - n) + (wait_n - h) + (cand_tail ? 1 : 0) > a) {
          res.status = kStatusRetryWider;
          break;
        }
      }
      // entries that were not admitted keep chunk 0 / delta 0
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        if (p >= n && p >= n + a) {
          chunk[k] = 0;
          delta[k] = 0;
        }
      }
    }
    if (!chunked && prefill_step && !any_nonready && a == 0) {
      // nothing to prefill fits: fall back to decoding all ready (backend.cpp:176-181)
      prefill_step = false;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        decode_item[k] = ready[k];
        const int32_t ns = stored[k] + 1;
        delta[k] = ready[k] ? bnt<POW2>(ns, cfg) - bnt<POW2>(stored[k], cfg) : 0;
      }
      delta_ready = true;
    }
    if (n == 0 && a == 0) {  // backend.cpp:245
      res.status = BSG_EMPTY_PLAN;
      break;
    }
    bool first_tok[K], done[K], dec_s[K], pre_s[K];
    int32_t freed[K];
    bool cand_first = false, cand_done = false;

    // ---------------- event skipping: pure-decode window ----------------
    // This step is pure decode with no admission. Member p (r_p = target -
    // decoded - 1) decodes in window steps t <= r_p and completes at the end of
    // step r_p; nothing else changes membership until (a) a step whose block
    // demand exceeds free (preemption), (b) the first step at which the waiting
    // head would be admitted (completions free blocks, budget and batch slots),
    // (c) the running set empties, or (d) the candidate completes (inclusive).
    // Lane l evaluates steps t = l*J + j of a kWin = 32*J step window:
    // D(t) = #alive, context C(t) = sum(stored)+t*D(t), demand
    // dem(t) = #{alive p : (stored_p + t) % block_size == 0}, free before the
    // step A(t) = free - sum_{s<t} dem(s) + sum_{s<t} freed(s) — from four
    // per-step shared-memory histograms and lane-contiguous warp scans.
    int32_t T = 0;
    static_assert(WJ >= 1 && WJ <= kMaxWinJ, "window width");
    int64_t win_pre[WJ];
    int64_t win_base = 0;
    bool win = (a == 0 || cyc0) && D == n && n > 0 && !prefill_step;
    if constexpr (CYC) {
      // Exact pre-checks of the window's first steps, so that a window which
      // would retire nothing is never set up (KV-pressure sets otherwise pay a
      // window per general step): a plain window stops at step 0 iff its decode
      // demand needs a victim; a cycle window is cut before its A1 step when
      // step 1 shows the cycle cannot close (the head would finish its prefill,
      // or more than the head would be evicted) — the tests the window applies.
      if (win) {
        bool d0[K], c0[K], d1[K];
        int32_t fr0[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const bool alive = lane * K + k < n;
          d0[k] = alive && modt<POW2>(stored[k], cfg) == 0;
          c0[k] = alive && target[k] - decoded[k] == 1;
          d1[k] = alive && !c0[k] && modt<POW2>(stored[k] + 1, cfg) == 0;
          fr0[k] = c0[k] ? bnt<POW2>(stored[k] + 1, cfg) : 0;
        }
        const int32_t dem0 = count<K>(d0);
        if (!cyc0) {
          win = dem0 <= free_blocks;
        } else {
          const int32_t nc0 = count<K>(c0);
          const int32_t D1 = n - nc0;
          const int32_t A1 = free_blocks - dem0 + (nc0 > 0 ? warp_sum<K>(fr0) : 0);
          const int32_t dem1 = count<K>(d1);
          const int32_t cA = cfg.chunk_budget - n;
          const int32_t hA = bnt<POW2>(cA, cfg);
          const int32_t bud1 = cfg.chunk_budget - D1;
          const int32_t rem = cyc_hp - cA;
          const int32_t ch = rem < bud1 ? rem : bud1;
          const int32_t dB = bnt<POW2>(cA + ch + (ch == rem ? 1 : 0), cfg) - hA;
          // step 1 evicts the head alone (a two-step cycle), or the head's next
          // chunk fits without finishing its prefill (a longer cycle may follow)
          const bool evict = dem1 + dB > A1 - hA;
          win = !(D1 == 0 || bud1 <= 0 || (evict && dem1 > A1) || (!evict && ch == rem));
        }
      }
    }
#ifdef BSG_PROFILE_T0
    bool prof_entered = false;
#endif
    // ---------------- drain: the rest of the run in one pass ----------------
    // Nothing is waiting (no victim, the snapshot's queue consumed, the
    // candidate admitted) and every running member decodes: no admission can
    // happen any more, so the steps up to the candidate's completion are pure
    // decode and only completions change the batch — unless the decode block
    // demand runs out of free blocks. If the members' total demand up to the
    // candidate's completion fits in the free blocks now (releases only add),
    // no step preempts, and the run ends at step T = r_cand + 1 with
    //   D(t) = #{p : r_p >= t},  C(t) = sum_{p : r_p >= t} (stored_p + t),
    // the window's formulas (below) without its 32*WJ-step cap. Members are
    // ranked by r_p into shared memory; lane l prices steps
    // [T*l/32, T*(l+1)/32), walking the completions in order. (Reference:
    // backend.cpp:113-182 with an empty waiting_ is a decode-all plan;
    // 263-288 allocates without eviction while demand <= free.)
    bool drained = false;
    if constexpr (BSG_DRAIN) {
      if (win && !cyc0 && L == n && h >= wait_n && !cand_tail) {
        int32_t rk[K], rc = 0x7fffffff;
        int64_t dem = 0;
        const int32_t rcl = [&] {
          int32_t m = 0x7fffffff;
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (lane * K + k < n && org[k] == (kCandOrg | kEverBit)) m = target[k] - decoded[k] - 1;
          return m;
        }();
        rc = static_cast<int32_t>(__reduce_min_sync(kFull, static_cast<uint32_t>(rcl)));
        const int64_t lim = kMaxSimulatedSteps + 1 - steps;
        const int32_t Td = rc + 1;  // steps to the candidate's completion (inclusive)
        if (rc != 0x7fffffff && Td <= lim) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            rk[k] = lane * K + k < n ? target[k] - decoded[k] - 1 : 0x7fffffff;
            if (lane * K + k < n) {
              const int32_t rl = rk[k] < Td - 1 ? rk[k] : Td - 1;
              dem += bnt<POW2>(stored[k] + rl + 1, cfg) - bnt<POW2>(stored[k], cfg);
            }
          }
          dem = warp_sum_i64(dem);
          bool fits = dem <= free_blocks;
          // 32-member lists: (r, stored) bitonic-sorted across the lanes, ascending r
          int32_t key = rk[0], val = stored[0];
          bool sorted = false;
          auto sort_members = [&]() {
#pragma unroll
            for (int kb = 2; kb <= 32; kb <<= 1) {
#pragma unroll
              for (int j = kb >> 1; j > 0; j >>= 1) {
                const int32_t ko = __shfl_xor_sync(kFull, key, j);
                const int32_t vo = __shfl_xor_sync(kFull, val, j);
                const bool keep_min = ((lane & j) == 0) == ((lane & kb) == 0);
                if (keep_min ? ko < key : ko > key) {
                  key = ko;
                  val = vo;
                }
              }
            }
            sorted = true;
          };
          if constexpr (K == 1 && !OPT) {  // (KV-pressure sets: the bound rarely holds, cfg3 +3 %)
            if (!fits) {
              // With the releases: step t needs free + R(t) >= Dc(t) (cumulative
              // demand vs the blocks of members completed before t). R grows only
              // at completions, so checking t = r_(k) at each distinct r suffices;
              // there Dc(t) <= (full demand of members sorted up to k) + (members
              // after k) * ceil((t + 1) / block_size) — one block per block_size
              // steps at most — and R(t) is the exclusive prefix of releases.
              int64_t rel = lane < n && rk[0] < Td - 1 ? bnt<POW2>(stored[0] + rk[0] + 1, cfg) : 0;
              rel = warp_sum_i64(rel);
              if (dem <= free_blocks + rel) {
                sort_members();
                const bool alive = lane < n;
                const int32_t tk = key < Td - 1 ? key : Td - 1;
                const int32_t dfull = alive ? bnt<POW2>(val + tk + 1, cfg) - bnt<POW2>(val, cfg) : 0;
                const int32_t fr = alive && key < Td - 1 ? bnt<POW2>(val + key + 1, cfg) : 0;
                const uint64_t pk = static_cast<uint32_t>(dfull) | (static_cast<uint64_t>(static_cast<uint32_t>(fr)) << 32);
                const uint64_t incl = warp_incl_scan_u64(pk);  // halves < 2^31 each: no carry
                const int64_t P = static_cast<int64_t>(static_cast<uint32_t>(incl));
                const int64_t R = static_cast<int64_t>(incl >> 32) - fr;
                const int32_t kprev = __shfl_up_sync(kFull, key, 1);
                const bool start = alive && (lane == 0 || kprev < key);
                const int64_t bound = P + static_cast<int64_t>(n - lane - 1) * divt<POW2>(tk + cfg.block_size, cfg);
                fits = __all_sync(kFull, !start || free_blocks + R >= bound);
              }
            }
          }
#ifdef BSG_PROFILE_DRAIN
          // debug: drain attempts that pass / fail the demand check (tools/drainprobe.py)
          if (fits) prof_dr_ok += 1;
          else prof_dr_fail += 1;
#endif
          if (fits) {
            drained = true;
            T = Td;
            int32_t* s_r = smem;
            int32_t* s_s = smem + CAP;
            int32_t* s_p = smem + 2 * CAP;
            __syncwarp();
            if constexpr (K == 1) {
              if (!sorted) sort_members();
              if (lane < n) {
                s_r[lane] = key;
                s_s[lane] = val;
              }
            } else {
              // rank members by (r, position) and store (r, stored) in that order
              int32_t rank[K];
#pragma unroll
              for (int k = 0; k < K; ++k) rank[k] = 0;
              for (int src = 0; src < 32; ++src) {
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
                  const int32_t rq = __shfl_sync(kFull, rk[kk], src);
                  const int32_t q = src * K + kk;
#pragma unroll
                  for (int k = 0; k < K; ++k)
                    rank[k] += (rq < rk[k] || (rq == rk[k] && q < lane * K + k)) ? 1 : 0;
                }
              }
#pragma unroll
              for (int k = 0; k < K; ++k) {
                if (lane * K + k < n) {
                  s_r[rank[k]] = rk[k];
                  s_s[rank[k]] = stored[k];
                }
              }
            }
            __syncwarp();
            int32_t sv[K], sp[K];
#pragma unroll
            for (int k = 0; k < K; ++k) sv[k] = lane * K + k < n ? s_s[lane * K + k] : 0;
            const int32_t s_tot = excl_scan<K>(sv, sp);
#pragma unroll
            for (int k = 0; k < K; ++k) s_p[lane * K + k] = sp[k];
            __syncwarp();
            const int32_t t0 = static_cast<int32_t>((static_cast<int64_t>(Td) * lane) >> 5);
            const int32_t t1 = static_cast<int32_t>((static_cast<int64_t>(Td) * (lane + 1)) >> 5);
            int32_t lo = 0, hi = n;  // idx = #{members with r < t0}
            while (lo < hi) {
              const int32_t mid = (lo + hi) >> 1;
              if (s_r[mid] < t0) lo = mid + 1;
              else hi = mid;
            }
            int32_t idx = lo;
            int32_t S = idx < n ? s_tot - s_p[idx] : 0;  // stored tokens of the members alive at t
            int32_t nxt = idx < n ? s_r[idx] : 0x7fffffff;
            // step_ticks(cfg, 0, D, C) split at its D term (same operations, same order)
            auto xd_of = [&](int32_t D) {
              const double x = __dadd_rn(cfg.c0, __dmul_rn(cfg.cp, 0.0));
              return __dadd_rn(x, __dmul_rn(cfg.cd, static_cast<double>(D)));
            };
            double xd = xd_of(n - idx);
            int64_t sum = 0, msum = 0;
            // MC: sample j (sorted) ends at step L_j - dec0 - 1; this lane's
            // samples are those ending in [t0, t1), recorded at their step with
            // the lane-local prefix, rebased after the walk
            const int32_t dec0 = cand_target - 1 - rc;  // the candidate's decoded count now
            int32_t jp = 0, j0 = 0;
            int64_t part = 0;
            if constexpr (MC) {
              int32_t a0 = mc_ptr, b0 = mc.S;
              while (a0 < b0) {
                const int32_t mid = (a0 + b0) >> 1;
                if (mc.len[mid] - dec0 - 1 < t0) a0 = mid + 1;
                else b0 = mid;
              }
              jp = j0 = a0;
            }
            for (int32_t t = t0; t < t1; ++t) {
              if (nxt < t) {
                do {
                  S -= s_s[idx];
                  ++idx;
                  nxt = idx < n ? s_r[idx] : 0x7fffffff;
                } while (nxt < t);
                xd = xd_of(n - idx);
              }
              const int32_t D = n - idx;
              int64_t ctx = S + t * D;
              if (cfg.cache_mode == BSG_CACHE_BUCKETED) {
                const int64_t b = cfg.context_bucket < 1 ? 1 : cfg.context_bucket;
                ctx = (ctx + b / 2) / b * b;
              }
              const double x = __dadd_rn(xd, __dmul_rn(cfg.cc, static_cast<double>(ctx)));
              sum += llround(__dmul_rn(x, 1e9));
              msum += D + 1;
              if constexpr (MC) {
                while (jp < mc.S && mc.len[jp] - dec0 - 1 == t) {
                  part += sum;
                  if (mc.sample_e2e) mc.sample_e2e[jp] = sum;
                  ++jp;
                }
              }
            }
            if constexpr (MC) {
              // elapsed before this lane's first step: exclusive scan of the lane sums
              int64_t pre = sum;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(kFull, pre, o);
                if (lane >= o) pre += y;
              }
              const int64_t base = elapsed + (pre - sum);
              mc_sum += part + static_cast<int64_t>(jp - j0) * base;
              if (mc.sample_e2e)
                for (int32_t j = j0; j < jp; ++j) mc.sample_e2e[j] += base;
              mc_ptr = mc.S;  // the candidate completes in this pass: every sample is done
              cand_hi = cand_target;
            }
            if constexpr (TRACE) {
              // per-step records (bsg_trace), as the window writes them
              int32_t fcur = free_blocks;
              for (int32_t t = 0; t < T && steps + t < trace.cap; ++t) {
                int32_t al[K], ral[K], cp[K], rcp[K], z[K], rz[K], cx[K], dm[K], fr[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                  const bool in = lane * K + k < n;
                  al[k] = in && rk[k] >= t ? 1 : 0;
                  cp[k] = in && rk[k] == t ? 1 : 0;
                  z[k] = in && t == 0 && decoded[k] == 0 ? 1 : 0;
                  cx[k] = al[k] ? stored[k] + t : 0;
                  dm[k] = al[k] && modt<POW2>(stored[k] + t, cfg) == 0 ? 1 : 0;
                  fr[k] = cp[k] ? bnt<POW2>(stored[k] + t + 1, cfg) : 0;
                }
                const int32_t nd = excl_scan<K>(al, ral);
                const int32_t ncp = excl_scan<K>(cp, rcp);
                excl_scan<K>(z, rz);
                uint64_t hplan = 0, hev = 0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                  const int32_t o = org_origin(org[k]);
                  if (al[k]) hplan += hash_term(BSG_TAG_PLAN, ral[k], o, 0);
                  if (z[k]) hev += hash_term(BSG_TAG_FIRST, rz[k], o, 0);
                  if (cp[k]) hev += hash_term(BSG_TAG_COMPLETED, rcp[k], o, 0);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                  hplan += __shfl_xor_sync(kFull, hplan, o);
                  hev += __shfl_xor_sync(kFull, hev, o);
                }
                const int32_t ct = warp_sum<K>(cx);
                fcur += warp_sum<K>(fr) - warp_sum<K>(dm);
                if (lane == 0) {
                  bsg_step_record& rec = trace.rec[steps + t];
                  rec.duration_ticks = step_ticks(cfg, 0, nd, ct);
                  rec.context_tokens = ct;
                  rec.n_decode = nd;
                  rec.prefill_tokens = 0;
                  rec.n_prefill = 0;
                  rec.n_preempted = 0;
                  rec.n_completed = ncp;
                  rec.free_blocks_after = fcur;
                  rec.plan_hash = hplan;
                  rec.event_hash = hev;
                }
              }
              __syncwarp();
            }
            elapsed += warp_sum_i64(sum);
            steps += T;
            res.member_steps += warp_sum_i64(msum);
            free_blocks -= static_cast<int32_t>(dem);
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const int32_t p = lane * K + k;
              dec_s[k] = p < n;
              pre_s[k] = false;
              first_tok[k] = false;
              if (p < n) decoded[k] += rk[k] < T ? rk[k] + 1 : T;
              done[k] = p < n && decoded[k] >= target[k];
              freed[k] = done[k] ? bnt<POW2>(prefill[k] + decoded[k], cfg) : 0;
              if (org[k] == (kCandOrg | kEverBit)) cand_done |= done[k];
            }
            __syncwarp();
          }
        }
      }
    }
    if (win && !drained) {
#ifdef BSG_PROFILE_T0
      prof_entered = true;
#endif
#ifdef BSG_PROFILE_WENTRY
      ++prof_pre;  // debug: window entries (reported in the preempt counter's slot)
#endif
      constexpr int J = WJ, W = 32 * WJ;
      int32_t* h_cnt = smem;          // members completing at the end of step s
      int32_t* h_sst = smem + W;      // their stored tokens at window start
      int32_t* h_dem = smem + 2 * W;  // block demand of step t
      int32_t* h_frd = smem + 3 * W;  // blocks released at the end of step s
      __syncwarp();  // the previous iteration's reads of this scratch are complete
#pragma unroll
      for (int i = 0; i < 4 * J; ++i) smem[i * 32 + lane] = 0;
      __syncwarp();
      const int32_t bs = cfg.block_size;
      int32_t lc = 0x7fffffff;  // candidate's r (if running)
      int32_t st_run[K], rr[K], fd[K];
      const unsigned lanes_lt = (1u << lane) - 1u;
      const bool strided = J > 1 && (bs >= W || bs % J == 0);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        st_run[k] = 0;
        rr[k] = -1;
        fd[k] = W;
        if (p < n) {
          const int32_t r = target[k] - decoded[k] - 1;
          const int32_t sp = stored[k];
          st_run[k] = sp;
          rr[k] = r;
          if (org[k] == (kCandOrg | kEverBit)) lc = r;
          if (r < W) {  // completes inside the window (few members): histogram by step
            atomicAdd(&h_cnt[r], 1);
            atomicAdd(&h_sst[r], sp);
            atomicAdd(&h_frd[r], bnt<POW2>(sp + r + 1, cfg));
          }
          const int32_t m = modt<POW2>(sp, cfg);
          fd[k] = m == 0 ? 0 : bs - m;  // first step whose decode opens a new block
          if constexpr (J == 1) {  // 32-step window: at most ceil(32 / bs) demand steps
            const int32_t rmax = r < W - 1 ? r : W - 1;
            for (int32_t t = fd[k]; t <= rmax; t += bs) atomicAdd(&h_dem[t], 1);
          }
        }
        if constexpr (J > 1) {
          // Block demand: member p demands at steps fd, fd + bs, ... <= r_p.
          // Histograms with match_any (one writer per distinct key — per-step
          // shared atomics over a 64-128 step window cost more than the window
          // saves). Strided layout (bs a multiple of J): histogram the LAST
          // demand step in the window; dem(t) is then the suffix sum along
          // t, t+bs, t+2bs, ... (shuffles below) and completions need no
          // correction. Otherwise: histogram the first demand step,
          // dem(t) = R[t mod bs], minus completed members (loop below).
          int32_t key = -1;
          if (rr[k] >= 0 && fd[k] < W) {
            if (strided) {
              const int32_t rmax = rr[k] < W - 1 ? rr[k] : W - 1;
              if (fd[k] <= rmax) key = fd[k] + divt<POW2>(rmax - fd[k], cfg) * bs;
            } else {
              key = fd[k];
            }
          }
          const unsigned peers = __match_any_sync(kFull, key >= 0 ? key : -1 - lane);
          if (key >= 0 && (peers & lanes_lt) == 0) h_dem[key] += __popc(peers);
          __syncwarp();
        }
      }
      __syncwarp();
      // lane-contiguous step layout: this lane's steps are t0 + j
      const int32_t t0 = lane * J;
      int32_t c_cnt[J], c_sst[J], c_dem[J], c_frd[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int32_t t = t0 + j;
        c_cnt[j] = h_cnt[t];
        c_sst[j] = h_sst[t];
        c_dem[j] = h_dem[(J > 1 && !strided) ? modt<POW2>(t, cfg) : t];
        c_frd[j] = h_frd[t];
      }
      if (strided) {  // suffix sums along each residue class: strides bs, 2bs, 4bs, ...
        for (int32_t st = bs; st < W; st <<= 1) {
          const int32_t dl = st / J;  // lanes per stride (bs is a multiple of J)
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const int32_t v = __shfl_down_sync(kFull, c_dem[j], dl);
            if (t0 + j + st < W) c_dem[j] += v;
          }
        }
      }
      // members completing before the window's last step stop demanding after r
#pragma unroll
      for (int k = 0; k < (J > 1 ? K : 0); ++k) {
        if (strided) break;
        for (unsigned cm = __ballot_sync(kFull, rr[k] >= 0 && rr[k] < W - 1 && fd[k] < W); cm;
             cm &= cm - 1) {
          const int src = __ffs(cm) - 1;
          const int32_t rp = __shfl_sync(kFull, rr[k], src);
          const int32_t fp = __shfl_sync(kFull, fd[k], src);
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const int32_t t = t0 + j;
            if (t > rp && t >= fp && modt<POW2>(t - fp, cfg) == 0) c_dem[j] -= 1;
          }
        }
      }
      const int32_t s_tot = warp_sum<K>(st_run);
      // two scans instead of four: (cnt | dem << 16) — both <= 256 per step and
      // <= 256 * kWin in total — and (sst | frd << 32) — sums of held tokens and
      // blocks, < 2^31 by the integer domain, so the low half never carries.
      int32_t cnt_x[J], sst_x[J], dem_x[J], frd_x[J];
      {
        int32_t cd_in[J], cd_x[J];
        uint64_t sf_lane = 0;
        uint64_t sf_x[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          cd_in[j] = c_cnt[j] | (c_dem[j] << 16);
          sf_x[j] = sf_lane;
          sf_lane += static_cast<uint32_t>(c_sst[j]) | (static_cast<uint64_t>(c_frd[j]) << 32);
        }
        excl_scan<J>(cd_in, cd_x);
        const uint64_t sf_base = warp_incl_scan_u64(sf_lane) - sf_lane;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          cnt_x[j] = cd_x[j] & 0xffff;
          dem_x[j] = static_cast<int32_t>(static_cast<uint32_t>(cd_x[j]) >> 16);
          const uint64_t v = sf_x[j] + sf_base;
          sst_x[j] = static_cast<int32_t>(static_cast<uint32_t>(v));
          frd_x[j] = static_cast<int32_t>(v >> 32);
        }
      }
      int32_t hp = 0;  // waiting head's prompt
      if (waiting_nonempty) {
        if (L > n) hp = read_pos<K>(prompt, n);  // victims: the waiting front
        else if (h < wait_n) hp = ld_entry<LDG>(g_prompt + sc.wait_off + h);
        else hp = sc.cand_prompt;
      }
      // Admit / self-preempt cycles (chunked prefill under KV pressure). When
      // the waiting head is a preemption victim (prefill = decoded = 0) whose
      // first chunk c1 = budget < prompt fits, step A1 admits it with that chunk
      // (the budget is then exhausted: a single admission, backend.cpp:135-147);
      // in the following steps A2, A3, ... its next full-budget chunks fit, until
      // at step B its next chunk does not, and the newest member — the head
      // itself — is evicted (263-288) and returns to the waiting front exactly
      // as before A1. While it runs, the head holds bn(progress) blocks, and B
      // refunds them, so after B the free count is what pure-decode steps would
      // leave, and A(t) below stays exact outside cycles. Per step t the window
      // computes where a cycle starting at t would end (e(t), a lane-parallel
      // walk over its steps), then follows the chain of cycles from step 0
      // (next event: a fitting step starts a cycle, a stop ends the window). A
      // cycle whose head would finish its prefill, or whose B would evict more
      // than the head, or that runs past the window, ends the window before it.
      const bool cyc_head = CYC && chunked && L > n;
      int32_t Dt[J], Ct[J], At[J], bud[J];
      bool fits[J], fa[J];
      int32_t rs_lane = -1;  // lane-local inclusive max of cycle-run starts
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int32_t t = t0 + j;
        Dt[j] = n - cnt_x[j];                          // alive in step t
        Ct[j] = (s_tot - sst_x[j]) + t * Dt[j];        // context of step t
        At[j] = free_blocks - dem_x[j] + frd_x[j];     // free before step t (no A at t-1)
        bud[j] = cfg.chunk_budget - Dt[j];
        // would the waiting head be admitted at step t? (backend.cpp:132-148 / 158-175)
        bool f = false;
        if (t == 0) {
          f = a > 0;
        } else if (waiting_nonempty && Dt[j] > 0) {
          if (chunked) {
            const int32_t c = hp < bud[j] ? hp : bud[j];
            f = bud[j] > 0 && Dt[j] < maxb && bnt<POW2>(c + (c == hp ? 1 : 0), cfg) <= At[j] - c_dem[j];
          } else {
            f = Dt[j] < maxb && bnt<POW2>(hp + 1, cfg) <= At[j];
          }
        }
        fits[j] = f;
        fa[j] = f && cyc_head && hp > bud[j];
      }
      int32_t first_stop = W;
      bool isA[J], isB[J];
      int32_t hprog[J];  // head's prefill progress before step t (cycle steps)
#pragma unroll
      for (int j = 0; j < J; ++j) {
        isA[j] = false;
        isB[j] = false;
        hprog[j] = 0;
      }
      bool any_fa = false;
#pragma unroll
      for (int j = 0; j < J; ++j) any_fa |= fa[j];
      if (CYC && __any_sync(kFull, any_fa)) {
        // per-step values in shared memory (the histograms are in registers now)
        int32_t* s_D = smem;
        int32_t* s_bud = smem + W;
        int32_t* s_At = smem + 2 * W;
        int32_t* s_dem = smem + 3 * W;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < J; ++j) {
          s_D[t0 + j] = Dt[j];
          s_bud[t0 + j] = bud[j];
          s_At[t0 + j] = At[j];
          s_dem[t0 + j] = c_dem[j];
        }
        __syncwarp();
        // e(t): the B step of a cycle whose A1 is step t (-1: cut before t)
        int32_t e[J], P[J];
        bool open[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          e[j] = -1;
          P[j] = bud[j];
          open[j] = fa[j];
        }
        for (int32_t d = 1;; ++d) {
          bool any_open = false;
#pragma unroll
          for (int j = 0; j < J; ++j) {
            if (open[j]) {
              const int32_t st = t0 + j + d;
              if (st >= W) {
                open[j] = false;
              } else {
                const int32_t Ds = s_D[st], bs_ = s_bud[st], As = s_At[st], cd = s_dem[st];
                const int32_t rem = hp - P[j];
                const int32_t ch = rem < bs_ ? rem : bs_;
                const int32_t hA = bnt<POW2>(P[j], cfg);
                const int32_t dl = bnt<POW2>(P[j] + ch + (ch == rem ? 1 : 0), cfg) - hA;
                if (Ds == 0 || bs_ <= 0) {
                  open[j] = false;
                } else if (cd + dl > As - hA) {  // F(n+1) < 0: the head is evicted
                  open[j] = false;
                  if (cd <= As) e[j] = st;       // F(n) >= 0: and nobody else
                } else if (ch == rem) {          // it would finish its prefill
                  open[j] = false;
                } else {
                  P[j] += ch;
                }
              }
              any_open |= open[j];
            }
          }
          if (!__any_sync(kFull, any_open)) break;
        }
        // next event at or after t: a fitting step (cycle start or cut) or a stop
        int32_t ev[J];
        {
          int32_t nx = W;
#pragma unroll
          for (int j = J - 1; j >= 0; --j) {
            const bool pstop = Dt[j] == 0 || c_dem[j] > At[j] || (fits[j] && !fa[j]);
            if (fa[j] || pstop) nx = t0 + j;
            ev[j] = nx;
          }
          // suffix-min over lanes: lane l gets min over lanes > l of their first event
          int32_t sfx = nx;  // this lane's first event
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_down_sync(kFull, sfx, o);
            if (lane + o < 32) sfx = min(sfx, y);
          }
          int32_t after = __shfl_down_sync(kFull, sfx, 1);
          if (lane == 31) after = W;
#pragma unroll
          for (int j = 0; j < J; ++j) ev[j] = min(ev[j], after);
        }
        int32_t* s_e = s_D;     // reused: e(t) of fitting steps, -1 otherwise
        int32_t* s_ev = s_bud;  // next event
        int32_t* s_cs = s_At;   // 1 = a cycle starts here
        __syncwarp();
#pragma unroll
        for (int j = 0; j < J; ++j) {
          s_e[t0 + j] = fa[j] ? e[j] : -1;
          s_ev[t0 + j] = ev[j];
          s_cs[t0 + j] = 0;
        }
        __syncwarp();
        // the chain of cycles from step 0 (warp-uniform walk over broadcast reads)
        int32_t cur = 0;
        for (;;) {
          const int32_t pos = cur < W ? s_ev[cur] : W;
          if (pos >= W) break;
          const int32_t eb = s_e[pos];
          if (eb < 0) {
            first_stop = pos;
            break;
          }
          if (lane == 0) s_cs[pos] = 1;
          cur = eb + 1;
        }
        __syncwarp();
        // each step's cycle: the latest start at or before it (prefix max)
        int32_t rs[J];
        {
          int32_t m = -1;
#pragma unroll
          for (int j = 0; j < J; ++j) {
            if (s_cs[t0 + j]) m = t0 + j;
            rs[j] = m;
          }
          int32_t pm = m;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, pm, o);
            if (lane >= o) pm = max(pm, y);
          }
          int32_t before = __shfl_up_sync(kFull, pm, 1);
          if (lane == 0) before = -1;
#pragma unroll
          for (int j = 0; j < J; ++j) rs[j] = max(rs[j], before);
        }
        // head progress: exclusive prefix of chunks (= budgets) from the cycle start
        int32_t Sx[J];
        excl_scan<J>(bud, Sx);
        int32_t* s_S = s_dem;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < J; ++j) s_S[t0 + j] = Sx[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int32_t t = t0 + j;
          if (rs[j] >= 0 && t < first_stop) {
            const int32_t eb = s_e[rs[j]];
            if (t <= eb) {
              isB[j] = t == eb;
              isA[j] = t < eb;
              hprog[j] = Sx[j] - s_S[rs[j]];
            }
          }
        }
      } else {
#pragma unroll
        for (int j = J - 1; j >= 0; --j) {
          const bool stop = Dt[j] == 0 || c_dem[j] > At[j] || fits[j];
          if (stop) first_stop = t0 + j;
        }
        first_stop = static_cast<int32_t>(__reduce_min_sync(kFull, static_cast<uint32_t>(first_stop)));
      }
      T = first_stop;
      const int32_t t_cand = static_cast<int32_t>(__reduce_min_sync(kFull, static_cast<uint32_t>(lc)));
      if (t_cand < W - 1) T = min(T, t_cand + 1);
      const int64_t lim = kMaxSimulatedSteps + 1 - steps;
      if (lim < T) T = static_cast<int32_t>(lim);
      if (T > 0) {
        int64_t d[J];
        int64_t dsum = 0;
        int32_t msum = 0;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const bool in = t0 + j < T;
          d[j] = in ? step_ticks(cfg, isA[j] ? bud[j] : 0, Dt[j], Ct[j]) : 0;
          dsum += d[j];
          msum += in ? Dt[j] + 1 + (isA[j] ? 1 : 0) : 0;
        }
        const int64_t sum = warp_sum_i64(dsum);
        if constexpr (MC) {
          // inclusive prefix of step durations: elapsed at the end of window step t
          int64_t pre = dsum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, pre, o);
            if (lane >= o) pre += y;
          }
          int64_t acc = pre - dsum;
#pragma unroll
          for (int j = 0; j < J; ++j) {
            acc += d[j];
            win_pre[j] = acc;
          }
          win_base = elapsed;
        }
        // free after the window's allocations (releases are added below with the
        // completed members' holdings)
        int32_t dem_i[J];
#pragma unroll
        for (int j = 0; j < J; ++j) dem_i[j] = dem_x[j] + c_dem[j];
        const int32_t dem_T = read_pos<J>(dem_i, T - 1);
        if constexpr (TRACE) {
          int32_t rr[K];
#pragma unroll
          for (int k = 0; k < K; ++k) rr[k] = (lane * K + k) < n ? target[k] - decoded[k] - 1 : -1;
          int32_t fafter[J], kind[J];  // free after step t; 1 = A step, 2 = B step
#pragma unroll
          for (int j = 0; j < J; ++j) {
            fafter[j] = free_blocks - dem_i[j] + frd_x[j] + c_frd[j] -
                        (isA[j] ? bnt<POW2>(hprog[j] + bud[j], cfg) : 0);
            kind[j] = isA[j] ? 1 : (isB[j] ? 2 : 0);
          }
          const int32_t head_o = cyc_head ? org_origin(read_pos<K>(org, n)) : 0;
          for (int32_t t = 0; t < T; ++t) {
            int32_t al[K], ral[K], cp[K], rcp[K], z[K], rz[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
              al[k] = rr[k] >= t ? 1 : 0;
              cp[k] = rr[k] == t ? 1 : 0;
              z[k] = (t == 0 && rr[k] >= 0 && decoded[k] == 0) ? 1 : 0;
            }
            excl_scan<K>(al, ral);
            const int32_t ncp = excl_scan<K>(cp, rcp);
            excl_scan<K>(z, rz);
            uint64_t hplan = 0, hev = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const int32_t o = org_origin(org[k]);
              if (al[k]) hplan += hash_term(BSG_TAG_PLAN, ral[k], o, 0);
              if (z[k]) hev += hash_term(BSG_TAG_FIRST, rz[k], o, 0);
              if (cp[k]) hev += hash_term(BSG_TAG_COMPLETED, rcp[k], o, 0);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              hplan += __shfl_xor_sync(kFull, hplan, o);
              hev += __shfl_xor_sync(kFull, hev, o);
            }
            int64_t dl = 0;
#pragma unroll
            for (int j = 0; j < J; ++j)
              if (j == t % J) dl = d[j];
            const int64_t dt = __shfl_sync(kFull, dl, t / J);
            const int32_t ct = read_pos<J>(Ct, t);
            const int32_t nd = read_pos<J>(Dt, t);
            const int32_t fat = read_pos<J>(fafter, t);
            const int32_t kt = read_pos<J>(kind, t);
            const int32_t ca = read_pos<J>(bud, t);
            if (kt == 1) hplan += hash_term(BSG_TAG_PLAN + 16u, 0, head_o, ca);
            if (kt == 2) hev += hash_term(BSG_TAG_PREEMPT, 0, head_o, 0);
            if (lane == 0 && steps + t < trace.cap) {
              bsg_step_record& rec = trace.rec[steps + t];
              rec.duration_ticks = dt;
              rec.context_tokens = ct;
              rec.n_decode = nd;
              rec.prefill_tokens = kt == 1 ? ca : 0;
              rec.n_prefill = kt == 1 ? 1 : 0;
#ifdef BSG_PROFILE_T0
              rec.n_prefill |= 1 << 20;  // debug: retired by a window
#endif
              rec.n_preempted = kt == 2 ? 1 : 0;
              rec.n_completed = ncp;
              rec.free_blocks_after = fat;
              rec.plan_hash = hplan;
              rec.event_hash = hev;
            }
          }
          __syncwarp();
        }
        elapsed += sum;
        steps += T;
        res.member_steps += static_cast<int64_t>(
            __reduce_add_sync(kFull, static_cast<uint32_t>(msum)));
        free_blocks -= dem_T;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int32_t p = lane * K + k;
          dec_s[k] = p < n;
          pre_s[k] = false;
          first_tok[k] = false;  // only possible at window step 0; never the candidate
          if (p < n) {
            const int32_t r = target[k] - decoded[k] - 1;
            decoded[k] += r < T ? r + 1 : T;
          }
          done[k] = p < n && decoded[k] >= target[k];
          freed[k] = done[k] ? bnt<POW2>(prefill[k] + decoded[k], cfg) : 0;
          if (org[k] == (kCandOrg | kEverBit)) cand_done |= done[k];
        }
      }
    }
#ifdef BSG_PROFILE_ITERS
    if (T == 0) ++prof_gen; else ++prof_win;
#ifdef BSG_PROFILE_T0
    // debug: general steps after a window that retired nothing (cycle entry / plain)
    if (T == 0 && prof_entered && a > 0) ++prof_adm;
    if (T == 0 && prof_entered && a == 0) ++prof_prf;
#else
    if (T == 0 && a > 0) ++prof_adm;
    if (T == 0 && any_nonready) ++prof_prf;
#endif
#endif
    if (T == 0 && !delta_ready) running_deltas();
    if (T == 0) {
    // ---------------- begin_step: admissions (backend.cpp:249-261) ----------------
    const int32_t n_adm = n + a;
    if (a > 0) {
      const int32_t from_tail = n_adm > L ? n_adm - L : 0;  // admitted beyond the victim stack
      const int32_t avail_w = wait_n - h;
      if (from_tail > avail_w) cand_tail = false;  // the candidate was admitted
      h += from_tail < avail_w ? from_tail : avail_w;
      if (n_adm > L) L = n_adm;
      bool started[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        started[k] = p >= n && p < n_adm && !org_ever(org[k]);
      }
      if constexpr (TRACE) {
        int32_t one[K], rk[K];
#pragma unroll
        for (int k = 0; k < K; ++k) one[k] = started[k] ? 1 : 0;
        excl_scan<K>(one, rk);
        uint64_t hs = 0;
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (started[k]) hs += hash_term(BSG_TAG_STARTED, rk[k], org_origin(org[k]), 0);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) hs += __shfl_xor_sync(kFull, hs, d);
        if (lane == 0 && steps < trace.cap) trace.rec[steps].event_hash = hs;
      }
      bool cand_started = false;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (started[k]) {
          if (org[k] == kCandOrg) cand_started = true;
          org[k] |= kEverBit;
        }
      }
      if (!qd_set && __any_sync(kFull, cand_started)) {
        res.qdelay_ticks = elapsed;  // predictor.cpp:111-115
        qd_set = true;
      }
    } else if constexpr (TRACE) {
      if (lane == 0 && steps < trace.cap) trace.rec[steps].event_hash = 0;
    }

    // ---------------- allocation + preemption (backend.cpp:263-288) ----------------
    const int32_t tot_delta = warp_sum<K>(delta);
    int32_t e_star = n_adm;
    if (tot_delta > free_blocks) {
      int32_t ho[K], hinc[K], dinc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        ho[k] = p < n ? bnt<POW2>(stored[k], cfg) : 0;
      }
      const int32_t htot = excl_scan<K>(ho, hinc);
      excl_scan<K>(delta, dinc);
      bool badp[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        // F(p+1) = free + (htot - incl_held(p)) - incl_delta(p)
        const int32_t f = free_blocks + (htot - hinc[k] - ho[k]) - (dinc[k] + delta[k]);
        badp[k] = p < n_adm && f < 0;
      }
      e_star = first_pos<K>(badp, n_adm);
      if (e_star == 0) {  // backend.cpp:274-277
        res.status = BSG_DEADLOCK;
        res.detail = org_origin(read_pos<K>(org, 0));
        break;
      }
      // F(e*) = free + sum_{v>=e*} held_old - sum_{p<e*} delta
      int32_t fe[K];
#pragma unroll
      for (int k = 0; k < K; ++k)
        fe[k] = free_blocks + (htot - hinc[k] - ho[k]) - (dinc[k] + delta[k]);
      free_blocks = read_pos<K>(fe, e_star - 1);
      if constexpr (TRACE) {
        uint64_t hp = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int32_t p = lane * K + k;
          if (p >= e_star && p < n_adm)
            hp += hash_term(BSG_TAG_PREEMPT, static_cast<uint32_t>(n_adm - 1 - p),
                            org_origin(org[k]), 0);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) hp += __shfl_xor_sync(kFull, hp, d);
        if (lane == 0 && steps < trace.cap) {
          trace.rec[steps].event_hash += hp;
          trace.rec[steps].n_preempted = n_adm - e_star;
        }
      }
      // victims: recompute semantics (preempt, backend.cpp:221-232)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        if (p >= e_star && p < n_adm) {
          prefill[k] = 0;
          decoded[k] = 0;
          chunk[k] = 0;
          decode_item[k] = false;
          delta[k] = 0;
        }
      }
    } else {
      free_blocks -= tot_delta;
      if constexpr (TRACE) {
        if (lane == 0 && steps < trace.cap) trace.rec[steps].n_preempted = 0;
      }
    }
#if defined(BSG_PROFILE_ITERS) && !defined(BSG_PROFILE_WENTRY)
    if (e_star < n_adm) ++prof_pre;
#endif
    n = e_star;

    // ---------------- price the surviving plan (to_batch_plan 194-209) ----------------
    int32_t ctx[K], pt[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t p = lane * K + k;
      dec_s[k] = p < n && decode_item[k];
      pre_s[k] = p < n && chunk[k] > 0;
      ctx[k] = dec_s[k] ? stored[k] : 0;
      pt[k] = pre_s[k] ? chunk[k] : 0;
    }
    const int32_t n_dec = count<K>(dec_s);
    res.member_steps += n_dec + count<K>(pre_s) + 1;
    const int32_t context = warp_sum<K>(ctx);
    const int32_t prefill_tokens = warp_sum<K>(pt);
    const int64_t dur = step_ticks(cfg, prefill_tokens, n_dec, context);
    elapsed += dur;
    steps += 1;
    if constexpr (TRACE) {
      int32_t od[K], rd[K], op[K], rp[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        od[k] = dec_s[k] ? 1 : 0;
        op[k] = pre_s[k] ? 1 : 0;
      }
      excl_scan<K>(od, rd);
      const int32_t n_pre = excl_scan<K>(op, rp);
      uint64_t hplan = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (dec_s[k]) hplan += hash_term(BSG_TAG_PLAN, rd[k], org_origin(org[k]), 0);
        if (pre_s[k]) hplan += hash_term(BSG_TAG_PLAN + 16u, rp[k], org_origin(org[k]), chunk[k]);
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) hplan += __shfl_xor_sync(kFull, hplan, d);
      if (lane == 0 && steps - 1 < trace.cap) {
        bsg_step_record& r = trace.rec[steps - 1];
        r.duration_ticks = dur;
        r.context_tokens = context;
        r.n_decode = n_dec;
        r.prefill_tokens = prefill_tokens;
        r.n_prefill = n_pre;
        r.plan_hash = hplan;
      }
    }

    // ---------------- finish_step (backend.cpp:298-331) ----------------
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t prev = decoded[k];
      if (dec_s[k]) {
        decoded[k] += 1;
      } else if (pre_s[k]) {
        prefill[k] += chunk[k];
        if (prefill[k] == prompt[k]) decoded[k] += 1;
      }
      const bool item = dec_s[k] || pre_s[k];
      first_tok[k] = item && prev == 0 && decoded[k] >= 1;
      done[k] = item && decoded[k] >= target[k];
      freed[k] = done[k] ? bnt<POW2>(prefill[k] + decoded[k], cfg) : 0;
      if (org[k] == (kCandOrg | kEverBit)) {
        cand_first |= first_tok[k];
        cand_done |= done[k];
      }
    }
    }  // general step (T == 0)
    if (TRACE && T == 0) {
      // item order: decodes (position order), then prefill items (position order)
      int32_t fd[K], fp[K], cd[K], cp[K], rfd[K], rfp[K], rcd[K], rcp[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        fd[k] = (first_tok[k] && dec_s[k]) ? 1 : 0;
        fp[k] = (first_tok[k] && pre_s[k]) ? 1 : 0;
        cd[k] = (done[k] && dec_s[k]) ? 1 : 0;
        cp[k] = (done[k] && pre_s[k]) ? 1 : 0;
      }
      const int32_t nfd = excl_scan<K>(fd, rfd);
      excl_scan<K>(fp, rfp);
      const int32_t ncd = excl_scan<K>(cd, rcd);
      const int32_t ncp = excl_scan<K>(cp, rcp);
      uint64_t he = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t o = org_origin(org[k]);
        if (fd[k]) he += hash_term(BSG_TAG_FIRST, rfd[k], o, 0);
        if (fp[k]) he += hash_term(BSG_TAG_FIRST, nfd + rfp[k], o, 0);
        if (cd[k]) he += hash_term(BSG_TAG_COMPLETED, rcd[k], o, 0);
        if (cp[k]) he += hash_term(BSG_TAG_COMPLETED, ncd + rcp[k], o, 0);
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) he += __shfl_xor_sync(kFull, he, d);
      if (lane == 0 && steps - 1 < trace.cap) {
        trace.rec[steps - 1].event_hash += he;
        trace.rec[steps - 1].n_completed = ncd + ncp;
      }
    }
    if (!ttft_set && __any_sync(kFull, cand_first)) {  // predictor.cpp:117-121
      res.ttft_ticks = elapsed;
      ttft_set = true;
    }
    if constexpr (MC) {
      // candidate's decoded count after this step / window (-1 when not running)
      int32_t cd = -1;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if ((lane * K + k) < n && org[k] == (kCandOrg | kEverBit)) cd = decoded[k];
      cd = static_cast<int32_t>(__reduce_max_sync(kFull, static_cast<uint32_t>(cd + 1))) - 1;
      if (cd > cand_hi) {
        const int32_t dec0 = cd - (T > 0 ? T : 1);  // decoded before this step / window
        for (;;) {
          const int32_t j = mc_ptr + lane;
          const int32_t lj = j < mc.S ? mc.len[j] : 0x7fffffff;
          const bool hit = lj <= cd;
          // step (within the window) at whose end decoded first reaches lj
          const int32_t tj = hit ? lj - dec0 - 1 : 0;
          int64_t at = elapsed;
          if (T > 0) {  // elapsed at the end of window step tj (held by lane tj / J, slot tj % J)
            const int32_t tw = tj & (32 * WJ - 1);
            int64_t v = 0;
#pragma unroll
            for (int j = 0; j < WJ; ++j) {
              const int64_t x = __shfl_sync(kFull, win_pre[j], tw / WJ);
              if (j == tw % WJ) v = x;
            }
            at = win_base + v;
          }
          if (hit) {
            mc_sum += at;
            if (mc.sample_e2e) mc.sample_e2e[j] = at;
          }
          const int32_t c = __popc(__ballot_sync(kFull, hit));
          mc_ptr += c;
          if (c < 32) break;
        }
        cand_hi = cd;
      }
    }
    const int32_t n_done = count<K>(done);
    if (n_done > 0) {
      free_blocks += warp_sum<K>(freed);
      // stable erase of completed members from running_ (backend.cpp:319-322):
      // compact positions [0, L) through shared memory.
      int32_t keep[K], dst[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        keep[k] = (p < L && !done[k]) ? 1 : 0;
      }
      excl_scan<K>(keep, dst);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (keep[k]) {
          int32_t* s = smem + dst[k];
          s[0 * CAP] = prompt[k];
          s[1 * CAP] = target[k];
          s[2 * CAP] = prefill[k];
          s[3 * CAP] = decoded[k];
          s[4 * CAP] = org[k];
        }
      }
      __syncwarp();
      n -= n_done;
      L -= n_done;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int32_t p = lane * K + k;
        if (p < L) {
          const int32_t* s = smem + p;
          prompt[k] = s[0 * CAP];
          target[k] = s[1 * CAP];
          prefill[k] = s[2 * CAP];
          decoded[k] = s[3 * CAP];
          org[k] = s[4 * CAP];
        }
      }
      __syncwarp();
    }
    if constexpr (TRACE) {
      if (lane == 0 && steps - 1 < trace.cap) trace.rec[steps - 1].free_blocks_after = free_blocks;
    }
    if (__any_sync(kFull, cand_done)) {  // predictor.cpp:122-124
      res.e2e_ticks = elapsed;
      if (!ttft_set) res.ttft_ticks = elapsed;  // predictor.cpp:130
      res.status = BSG_OK;
      break;
    }
    if (steps > kMaxSimulatedSteps) {  // predictor.cpp:125-127
      res.status = BSG_STEP_LIMIT;
      break;
    }
  }
  res.steps = steps;
#ifdef BSG_PROFILE_DRAIN
  res.detail = prof_dr_ok + 1000 * prof_dr_fail;
#endif
#ifdef BSG_PROFILE_ITERS
  // debug build only (tools/iterprobe.py): loop iterations by kind
  res.detail = static_cast<int32_t>(prof_gen);
  res.member_steps = prof_win;
  res.ttft_ticks = prof_adm;    // general steps that admit
  res.qdelay_ticks = prof_prf;  // general steps with a running partial prefill
  res.e2e_ticks = prof_pre;     // general steps that preempt
#endif
  if constexpr (MC) {
    int64_t tot = mc_sum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
    if (mc.objective == 1) tot = static_cast<int64_t>(mc.S) * res.ttft_ticks;
    if (lane == 0) *mc.score = res.status == BSG_OK ? tot : INT64_MAX;
  }
  if (lane == 0) *out = res;
}

}  // namespace bsg

/*
 * oracle/blocksim_oracle.c — CPU restatement of the reference's what-if
 * simulation (blocksim predict()), in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's
 * library, and only as the checker. The product path (paper_2508_03611_b200)
 * never links or calls it.
 *
 * Parity pinning: this restatement is checked (tests/test_oracle.py) against
 *   (1) the reference's own known-answer tests, restated in
 *       tests/golden/reference_kats.json (test_backend.cpp, test_predictor.cpp,
 *       test_core.cpp, test_driver.cpp:16-36, acceptance C11 fixtures), and
 *   (2) the reference itself, compiled from /root/reference by oracle/Makefile
 *       into oracle/_ref/libblocksim_ref.so, on seeded fuzz scenarios and on
 *       committed golden vectors (tests/golden/ JSON files, made by
 *       tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line (paths relative to
 * /root/reference/proj/core) whose behaviour it restates. The structure is a
 * deliberately naive, sequential transcription (slot pool, running vector,
 * waiting deque, per-step item list) so it reads against the reference line
 * by line; it is not fast and is not meant to be.
 */
#include "blocksim_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Slot — backend.h:113-126. */
typedef struct {
  int32_t prompt, target, prefill, decoded;
  int64_t held;
  uint64_t seq; /* admission_seq, nonzero while running */
  int32_t origin;
  int32_t ever; /* ever_scheduled */
} oslot;

/* PlanItem — backend.h:128-134. */
typedef struct {
  int32_t slot, chunk, new_stored;
  int64_t delta;
  int32_t preempted;
} oitem;

typedef struct {
  const bsg_instance_cfg* cfg;
  oslot* pool;
  int32_t npool;
  int32_t* running; /* slot indices, admission order */
  int32_t nrun;
  int32_t* wq; /* waiting deque as ring buffer */
  int32_t wcap, whead, wn;
  int64_t free_blocks;
  uint64_t next_seq;
  oitem* items;
  int32_t nitems;
  int32_t* done; /* finish_step's done_slots (backend.cpp:301) */
} oinst;

/* blocks_needed — types.cpp:63-66. */
static int64_t o_blocks_needed(int64_t tokens, int32_t block_size) {
  if (tokens <= 0) return 0;
  return (tokens + block_size - 1) / block_size;
}

/* batch_latency — backend.cpp:10-14; unfused double arithmetic, left to right. */
static double o_batch_latency(const bsg_instance_cfg* c, int64_t prefill_tokens, int64_t n_decode,
                              int64_t context) {
  return c->c0_s + c->prefill_s_per_token * (double)prefill_tokens +
         c->decode_s_per_seq * (double)n_decode + c->context_s_per_token * (double)context;
}

/* LatencyCache::lookup_or_compute — predictor.cpp:26-54. Off and exact modes
 * both return batch_latency(plan) (a hit returns exactly what a miss stored);
 * bucketed prices the bucket representative (predictor.cpp:29-32, 45-47). */
static double o_latency(const bsg_instance_cfg* c, int64_t prefill_tokens, int64_t n_decode,
                        int64_t context) {
  if (c->cache_mode == BSG_CACHE_BUCKETED) {
    int64_t b = c->context_bucket < 1 ? 1 : c->context_bucket; /* predictor.cpp:23-24 */
    context = (context + b / 2) / b * b;
  }
  return o_batch_latency(c, prefill_tokens, n_decode, context);
}

/* SimTime::from_seconds — time.h:20-22. */
static int64_t o_from_seconds(double s) { return (int64_t)llround(s * 1e9); }

static int32_t o_stored(const oslot* s) { return s->prefill + s->decoded; }
static int o_ready(const oslot* s) { return s->prefill == s->prompt; }

static void w_push_back(oinst* in, int32_t slot) {
  in->wq[(in->whead + in->wn) % in->wcap] = slot;
  in->wn++;
}
static void w_push_front(oinst* in, int32_t slot) {
  in->whead = (in->whead + in->wcap - 1) % in->wcap;
  in->wq[in->whead] = slot;
  in->wn++;
}
static int32_t w_at(const oinst* in, int32_t i) { return in->wq[(in->whead + i) % in->wcap]; }
static int32_t w_pop_front(oinst* in) {
  int32_t s = in->wq[in->whead];
  in->whead = (in->whead + 1) % in->wcap;
  in->wn--;
  return s;
}

/* make_item — backend.cpp:94-111. */
static oitem o_make_item(const oinst* in, int32_t slot, int32_t chunk) {
  const oslot* s = &in->pool[slot];
  oitem it;
  it.slot = slot;
  it.chunk = chunk;
  it.preempted = 0;
  int32_t old_stored = o_stored(s);
  if (chunk == 0) {
    it.new_stored = old_stored + 1;
  } else {
    int32_t new_prefill = s->prefill + chunk;
    it.new_stored = new_prefill + s->decoded + (new_prefill == s->prompt ? 1 : 0);
  }
  it.delta = o_blocks_needed(it.new_stored, in->cfg->block_size) -
             o_blocks_needed(old_stored, in->cfg->block_size);
  return it;
}

/* plan_chunked_prefill — backend.cpp:113-149. */
static int32_t o_plan_chunked(oinst* in) {
  int32_t admit = 0;
  int64_t budget = in->cfg->chunk_budget;
  for (int32_t i = 0; i < in->nrun; ++i) {
    int32_t slot = in->running[i];
    if (o_ready(&in->pool[slot])) {
      in->items[in->nitems++] = o_make_item(in, slot, 0);
      budget -= 1;
    }
  }
  if (budget < 0) budget = 0;
  for (int32_t i = 0; i < in->nrun; ++i) {
    if (budget == 0) break;
    int32_t slot = in->running[i];
    const oslot* s = &in->pool[slot];
    if (!o_ready(s)) {
      int64_t rem = (int64_t)s->prompt - s->prefill;
      int32_t chunk = (int32_t)(rem < budget ? rem : budget);
      in->items[in->nitems++] = o_make_item(in, slot, chunk);
      budget -= chunk;
    }
  }
  int64_t projected_free = in->free_blocks;
  for (int32_t k = 0; k < in->nitems; ++k) projected_free -= in->items[k].delta;
  int32_t members = in->nrun;
  for (int32_t j = 0; j < in->wn; ++j) {
    if (budget == 0 || members >= in->cfg->max_batch_size) break;
    int32_t slot = w_at(in, j);
    const oslot* s = &in->pool[slot];
    int64_t rem = (int64_t)s->prompt - s->prefill;
    int32_t chunk = (int32_t)(rem < budget ? rem : budget);
    oitem it = o_make_item(in, slot, chunk);
    if (it.delta > projected_free) break; /* head blocks the queue (backend.cpp:142) */
    in->items[in->nitems++] = it;
    budget -= chunk;
    projected_free -= it.delta;
    ++members;
    ++admit;
  }
  return admit;
}

/* plan_prefill_priority — backend.cpp:151-182. */
static int32_t o_plan_prefill_priority(oinst* in) {
  int32_t admit = 0;
  int prefill_needed = in->wn > 0;
  for (int32_t i = 0; i < in->nrun; ++i)
    if (!o_ready(&in->pool[in->running[i]])) prefill_needed = 1;
  if (prefill_needed) {
    int64_t projected_free = in->free_blocks;
    for (int32_t i = 0; i < in->nrun; ++i) {
      int32_t slot = in->running[i];
      const oslot* s = &in->pool[slot];
      if (!o_ready(s)) {
        oitem it = o_make_item(in, slot, s->prompt - s->prefill);
        projected_free -= it.delta;
        in->items[in->nitems++] = it;
      }
    }
    int32_t members = in->nrun;
    for (int32_t j = 0; j < in->wn; ++j) {
      if (members >= in->cfg->max_batch_size) break;
      int32_t slot = w_at(in, j);
      const oslot* s = &in->pool[slot];
      oitem it = o_make_item(in, slot, s->prompt - s->prefill);
      if (it.delta > projected_free) break;
      in->items[in->nitems++] = it;
      projected_free -= it.delta;
      ++members;
      ++admit;
    }
    if (in->nitems > 0) return admit; /* pure-prefill batch (backend.cpp:176) */
  }
  for (int32_t i = 0; i < in->nrun; ++i) {
    int32_t slot = in->running[i];
    if (o_ready(&in->pool[slot])) in->items[in->nitems++] = o_make_item(in, slot, 0);
  }
  return admit;
}

/* preempt — backend.cpp:221-232. */
static void o_preempt(oinst* in, int32_t slot) {
  int32_t w = 0;
  for (int32_t i = 0; i < in->nrun; ++i)
    if (in->running[i] != slot) in->running[w++] = in->running[i];
  in->nrun = w;
  oslot* s = &in->pool[slot];
  in->free_blocks += s->held;
  s->held = 0;
  s->prefill = 0;
  s->decoded = 0;
  s->seq = 0;
  w_push_front(in, slot);
}

typedef struct {
  int64_t duration;
  int64_t context;
  int32_t n_decode, prefill_tokens, n_prefill, n_preempted, n_completed;
  uint64_t plan_hash, event_hash;
  int cand_started, cand_first, cand_completed;
  int32_t error;      /* bsg_status */
  int32_t error_detail;
} ostep;

/* begin_step + finish_step (backend.cpp:238-331) fused as execute_step
 * (backend.cpp:338-349), pricing through o_latency. */
static void o_execute_step(oinst* in, int32_t cand_slot, ostep* st) {
  memset(st, 0, sizeof(*st));
  if (in->nrun == 0 && in->wn == 0) { /* backend.cpp:240 */
    st->error = BSG_EMPTY_PLAN;
    return;
  }
  in->nitems = 0;
  int32_t admit = in->cfg->local_policy == BSG_CHUNKED_PREFILL ? o_plan_chunked(in)
                                                               : o_plan_prefill_priority(in);
  if (in->nitems == 0) { /* backend.cpp:245 */
    st->error = BSG_EMPTY_PLAN;
    return;
  }
  uint32_t k_started = 0;
  /* admitted waiting heads join the running tail before allocation
   * (backend.cpp:249-261) */
  for (int32_t i = 0; i < admit; ++i) {
    int32_t slot = w_pop_front(in);
    oslot* s = &in->pool[slot];
    s->seq = in->next_seq++;
    if (!s->ever) {
      s->ever = 1;
      st->event_hash += bsg_hash_term(BSG_TAG_STARTED, k_started++, s->origin, 0);
      if (slot == cand_slot) st->cand_started = 1;
    }
    in->running[in->nrun++] = slot;
  }
  /* allocation with newest-member preemption (backend.cpp:263-288) */
  uint32_t k_pre = 0;
  for (int32_t k = 0; k < in->nitems; ++k) {
    oitem* item = &in->items[k];
    if (item->preempted) continue;
    while (item->delta > in->free_blocks) {
      int32_t victim = -1;
      uint64_t newest = 0;
      for (int32_t i = 0; i < in->nrun; ++i) {
        if (in->pool[in->running[i]].seq > newest) {
          newest = in->pool[in->running[i]].seq;
          victim = in->running[i];
        }
      }
      if (victim == item->slot && in->nrun == 1) { /* backend.cpp:274-277 */
        st->error = BSG_DEADLOCK;
        st->error_detail = in->pool[item->slot].origin;
        return;
      }
      st->event_hash += bsg_hash_term(BSG_TAG_PREEMPT, k_pre++, in->pool[victim].origin, 0);
      st->n_preempted++;
      for (int32_t q = 0; q < in->nitems; ++q)
        if (in->items[q].slot == victim) in->items[q].preempted = 1;
      o_preempt(in, victim);
      if (item->preempted) break;
    }
    if (item->preempted) continue;
    in->free_blocks -= item->delta;
    in->pool[item->slot].held += item->delta;
  }
  /* to_batch_plan — backend.cpp:194-209 (surviving items, pre-step stored) */
  uint32_t kd = 0, kp = 0;
  int64_t context = 0, total_prefill = 0;
  uint64_t hd = 0, hp = 0;
  for (int32_t k = 0; k < in->nitems; ++k) {
    const oitem* it = &in->items[k];
    if (it->preempted) continue;
    const oslot* s = &in->pool[it->slot];
    if (it->chunk == 0) {
      hd += bsg_hash_term(BSG_TAG_PLAN, kd++, s->origin, 0);
      context += o_stored(s);
    } else {
      hp += bsg_hash_term(BSG_TAG_PLAN + 16u, kp++, s->origin, it->chunk);
      total_prefill += it->chunk;
    }
  }
  st->n_decode = (int32_t)kd;
  st->n_prefill = (int32_t)kp;
  st->prefill_tokens = (int32_t)total_prefill;
  st->context = context;
  st->plan_hash = hd + hp;
  /* begin_step pricing: SimTime::from_seconds(latency_fn(plan)) backend.cpp:292 */
  st->duration = o_from_seconds(o_latency(in->cfg, total_prefill, kd, context));

  /* finish_step — backend.cpp:298-331 */
  uint32_t k_first = 0, k_done = 0;
  int32_t ndone = 0;
  for (int32_t k = 0; k < in->nitems; ++k) {
    const oitem* it = &in->items[k];
    if (it->preempted) continue;
    oslot* s = &in->pool[it->slot];
    int32_t prev_decoded = s->decoded;
    if (it->chunk > 0) {
      s->prefill += it->chunk;
      if (s->prefill == s->prompt) s->decoded += 1;
    } else {
      s->decoded += 1;
    }
    if (prev_decoded == 0 && s->decoded >= 1) {
      st->event_hash += bsg_hash_term(BSG_TAG_FIRST, k_first++, s->origin, 0);
      if (it->slot == cand_slot) st->cand_first = 1;
    }
    if (s->decoded >= s->target) {
      st->event_hash += bsg_hash_term(BSG_TAG_COMPLETED, k_done++, s->origin, 0);
      if (it->slot == cand_slot) st->cand_completed = 1;
      in->done[ndone++] = it->slot;
    }
  }
  for (int32_t d = 0; d < ndone; ++d) {
    int32_t slot = in->done[d];
    int32_t w = 0;
    for (int32_t i = 0; i < in->nrun; ++i)
      if (in->running[i] != slot) in->running[w++] = in->running[i];
    in->nrun = w;
    in->free_blocks += in->pool[slot].held;
    in->pool[slot].held = 0;
  }
  st->n_completed = ndone;
}

/* predict — predictor.cpp:76-137 (with correct_lengths predictor.cpp:65-74,
 * Instance::from_snapshot backend.cpp:20-56 and admit backend.cpp:74-92). */
int32_t oracle_predict(const bsg_instance_cfg* cfg, const bsg_entries* e,
                       const bsg_scenario* sc, bsg_result* out, bsg_step_record* trace,
                       int64_t trace_cap, int64_t* n_steps) {
  memset(out, 0, sizeof(*out));
  if (n_steps) *n_steps = 0;
  /* validate_instance_config — types.cpp:47-61 (Instance ctor, backend.cpp:16-18) */
  {
    int32_t f = oracle_validate_config(cfg);
    if (f) {
      out->status = BSG_BAD_CONFIG;
      out->detail = f;
      return out->status;
    }
  }
  oinst in;
  memset(&in, 0, sizeof(in));
  in.cfg = cfg;
  int32_t cap = sc->run_n + sc->wait_n + 1;
  in.pool = (oslot*)calloc((size_t)cap, sizeof(oslot));
  in.running = (int32_t*)calloc((size_t)cap, sizeof(int32_t));
  in.wcap = cap;
  in.wq = (int32_t*)calloc((size_t)cap, sizeof(int32_t));
  in.items = (oitem*)calloc((size_t)cap, sizeof(oitem));
  in.done = (int32_t*)calloc((size_t)cap, sizeof(int32_t));
  in.free_blocks = cfg->total_blocks;
  in.next_seq = 1;

  /* correct_lengths — predictor.cpp:65-74: decoded >= est => est = decoded + 10 */
#define CORRECTED(idx) \
  (e->decoded[idx] >= e->est[idx] ? e->decoded[idx] + 10 : e->est[idx])
  /* from_snapshot running — backend.cpp:24-41 */
  for (int32_t i = 0; i < sc->run_n; ++i) {
    int32_t idx = sc->run_off + i;
    oslot* s = &in.pool[in.npool];
    s->prompt = e->prompt[idx];
    s->target = CORRECTED(idx);
    s->prefill = e->prefill[idx];
    s->decoded = e->decoded[idx];
    s->held = o_blocks_needed(o_stored(s), cfg->block_size);
    s->seq = in.next_seq++;
    s->ever = 1;
    s->origin = i;
    in.free_blocks -= s->held;
    in.running[in.nrun++] = in.npool++;
  }
  int32_t status = BSG_OK;
  if (in.free_blocks < 0) { /* backend.cpp:42-44 */
    status = BSG_TOO_LARGE_RUNNING;
    goto done;
  }
  /* from_snapshot waiting — backend.cpp:45-54: progress restarts at zero */
  for (int32_t j = 0; j < sc->wait_n; ++j) {
    int32_t idx = sc->wait_off + j;
    oslot* s = &in.pool[in.npool];
    s->prompt = e->prompt[idx];
    s->target = CORRECTED(idx);
    s->origin = sc->run_n + j;
    w_push_back(&in, in.npool++);
  }
#undef CORRECTED
  /* admit the candidate at the waiting tail — backend.cpp:74-92 */
  if (o_blocks_needed((int64_t)sc->cand_prompt + sc->cand_est, cfg->block_size) >
      cfg->total_blocks) {
    status = BSG_TOO_LARGE_CANDIDATE;
    out->detail = (int32_t)o_blocks_needed((int64_t)sc->cand_prompt + sc->cand_est,
                                           cfg->block_size);
    goto done;
  }
  int32_t cand_slot = in.npool;
  {
    oslot* s = &in.pool[in.npool];
    s->prompt = sc->cand_prompt;
    s->target = sc->cand_est;
    s->origin = -1;
    w_push_back(&in, in.npool++);
  }
  /* forward loop — predictor.cpp:99-128 */
  {
    int64_t elapsed = 0, steps = 0;
    int qd_set = 0, ttft_set = 0;
    for (;;) {
      if (in.nrun == 0 && in.wn == 0) { /* predictor.cpp:102-104 */
        status = BSG_VANISHED;
        break;
      }
      int64_t step_start = elapsed;
      ostep st;
      o_execute_step(&in, cand_slot, &st);
      if (st.error) {
        status = st.error;
        out->detail = st.error_detail;
        break;
      }
      elapsed += st.duration;
      steps += 1;
      out->member_steps += st.n_decode + st.n_prefill + 1;
      if (trace && steps <= trace_cap) {
        bsg_step_record* r = &trace[steps - 1];
        r->duration_ticks = st.duration;
        r->context_tokens = st.context;
        r->n_decode = st.n_decode;
        r->prefill_tokens = st.prefill_tokens;
        r->n_prefill = st.n_prefill;
        r->n_preempted = st.n_preempted;
        r->n_completed = st.n_completed;
        r->free_blocks_after = (int32_t)in.free_blocks;
        r->plan_hash = st.plan_hash;
        r->event_hash = st.event_hash;
      }
      if (!qd_set && st.cand_started) {
        out->qdelay_ticks = step_start;
        qd_set = 1;
      }
      if (!ttft_set && st.cand_first) {
        out->ttft_ticks = elapsed;
        ttft_set = 1;
      }
      if (st.cand_completed) {
        out->e2e_ticks = elapsed;
        if (!ttft_set) out->ttft_ticks = elapsed; /* predictor.cpp:130 */
        break;
      }
      if (steps > ORACLE_MAX_STEPS) { /* predictor.cpp:125-127 */
        status = BSG_STEP_LIMIT;
        break;
      }
    }
    out->steps = steps;
    if (n_steps) *n_steps = steps;
  }
done:
  out->status = status;
  free(in.pool);
  free(in.running);
  free(in.wq);
  free(in.items);
  free(in.done);
  return status;
}

/* validate_instance_config — types.cpp:47-61. Returns the field code of the
 * first violated check, 0 when valid. */
int32_t oracle_validate_config(const bsg_instance_cfg* c) {
  if (c->total_blocks < 1) return 1;
  if (c->block_size < 1) return 2;
  if (c->max_batch_size < 1) return 3;
  if (c->chunk_budget < c->block_size) return 4;
  if (!(c->c0_s > 0)) return 5;
  if (c->prefill_s_per_token < 0) return 6;
  if (c->decode_s_per_seq < 0) return 7;
  if (c->context_s_per_token < 0) return 8;
  return 0;
}

void oracle_predict_batch(const bsg_instance_cfg* cfgs, const bsg_entries* e,
                          const bsg_scenario* sc, int64_t n, bsg_result* out) {
  for (int64_t i = 0; i < n; ++i)
    oracle_predict(&cfgs[sc[i].cfg], e, &sc[i], &out[i], NULL, 0, NULL);
}

double oracle_ticks_to_seconds(int64_t ticks) { return (double)ticks * 1e-9; /* time.h:25 */ }
int64_t oracle_llround_1e9(double s) { return o_from_seconds(s); }
int64_t oracle_blocks_needed(int64_t tokens, int32_t block_size) {
  return o_blocks_needed(tokens, block_size);
}
double oracle_batch_latency(const bsg_instance_cfg* c, int64_t prefill_tokens, int64_t n_decode,
                            int64_t context) {
  return o_batch_latency(c, prefill_tokens, n_decode, context);
}

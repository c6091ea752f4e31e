"""Seeded scenario generators for parity tests (test infrastructure).

fuzz_set() covers the edge inputs of SURVEY.md Appendix A.9: overrun decodes
(the +10 correction), waiting entries with non-zero progress (reset), running
entries mid-prefill, running sets exceeding memory (TOO_LARGE_RUNNING), tiny
total_blocks (preemption / deadlock), candidates exactly at capacity,
target 1, prefill_priority, bucketed cache, non-power-of-two block sizes.
"""
from __future__ import annotations

import numpy as np

from paper_2508_03611_b200 import abi


def fuzz_configs() -> np.ndarray:
    cfgs = [
        abi.make_config(),  # reference_config (test_backend.cpp:15-22)
        abi.make_config(local_policy=abi.PREFILL_PRIORITY),
        abi.make_config(cache_mode=abi.CACHE_BUCKETED, context_bucket=256),
        abi.make_config(cache_mode=abi.CACHE_EXACT),
        abi.make_config(total_blocks=64, block_size=8, max_batch_size=8, chunk_budget=64),
        abi.make_config(total_blocks=48, block_size=8, max_batch_size=6, chunk_budget=4096),
        abi.make_config(total_blocks=40, block_size=7, max_batch_size=12, chunk_budget=21,
                        local_policy=abi.PREFILL_PRIORITY),
        abi.make_config(total_blocks=30, block_size=5, max_batch_size=4, chunk_budget=5,
                        cache_mode=abi.CACHE_BUCKETED, context_bucket=3),
        abi.make_config(total_blocks=200, block_size=3, max_batch_size=64, chunk_budget=100),
        abi.make_config(total_blocks=20, block_size=1, max_batch_size=2, chunk_budget=1),
        abi.make_config(total_blocks=500, block_size=16, max_batch_size=1, chunk_budget=16,
                        c0_s=0.003, prefill_s_per_token=2.5e-5, decode_s_per_seq=7e-4,
                        context_s_per_token=3.3e-8),
        abi.make_config(total_blocks=6, block_size=16, max_batch_size=48, chunk_budget=512),
    ]
    return np.concatenate(cfgs)


def _blocks(t, bs):
    return 0 if t <= 0 else (t + bs - 1) // bs


def fuzz_set(seed: int, n: int, cfgs: np.ndarray | None = None,
             max_running: int = 60, max_waiting: int = 40) -> tuple[np.ndarray, abi.ScenarioSet]:
    rng = np.random.default_rng(seed)
    if cfgs is None:
        cfgs = fuzz_configs()
    snaps, cands, cfg_idx = [], [], []
    for _ in range(n):
        ci = int(rng.integers(len(cfgs)))
        c = cfgs[ci]
        bs, total, maxb = int(c["block_size"]), int(c["total_blocks"]), int(c["max_batch_size"])
        scale = max(4, min(300, total * bs // 8))
        run_n = int(rng.integers(0, min(max_running, maxb + 2) + 1))
        if rng.random() < 0.3:
            run_n = min(run_n, 3)
        running, held = [], 0
        overflow_ok = rng.random() < 0.05
        for _ in range(run_n):
            prompt = int(rng.integers(1, scale + 1))
            if rng.random() < 0.7:
                prefill = prompt
                decoded = int(rng.integers(0, max(1, scale // 3)))
            else:
                prefill = int(rng.integers(0, prompt))
                decoded = 0 if rng.random() < 0.9 else int(rng.integers(1, 5))
            est = int(rng.integers(1, max(2, scale // 2)))
            if rng.random() < 0.15:
                est = max(1, decoded - int(rng.integers(0, 3)))  # overrun / boundary
            b = _blocks(prefill + decoded, bs)
            if held + b > total and not overflow_ok:
                continue
            held += b
            running.append((prompt, est, prefill, decoded))
        wait_n = int(rng.integers(0, max_waiting + 1)) if rng.random() < 0.6 else 0
        waiting = []
        for _ in range(wait_n):
            prompt = int(rng.integers(1, scale + 1))
            est = int(rng.integers(1, max(2, scale // 2)))
            prefill = int(rng.integers(0, prompt + 1)) if rng.random() < 0.2 else 0
            decoded = int(rng.integers(0, est + 20)) if rng.random() < 0.1 else 0
            waiting.append((prompt, est, prefill, decoded))
        cp = int(rng.integers(1, scale + 1))
        ce = int(rng.integers(0, max(2, scale // 2)))
        r = rng.random()
        if r < 0.05:
            ce = 1
        elif r < 0.08:  # exactly at capacity (blocks_needed(prompt+est) == total)
            cp = max(1, min(cp, total * bs - 1))
            ce = total * bs - cp
        elif r < 0.10:  # one token over capacity
            cp = max(1, min(cp, total * bs))
            ce = total * bs - cp + 1
        snaps.append((running, waiting))
        cands.append((cp, ce))
        cfg_idx.append(ci)
    return cfgs, abi.ScenarioSet.from_snapshots(snaps, cands, cfg_idx)


# Scenarios restated from the reference's own tests (file:line under
# /root/reference/proj/tests). Each entry: (name, cfg kwargs, running, waiting, candidate).
def reference_kat_scenarios():
    R = dict()
    kats = []
    # test_predictor.cpp:55-73 — predict on an empty instance; 512-token prompt, 10 outputs
    kats.append(("predictor_empty_instance", R, [], [], (512, 10)))
    # test_predictor.cpp:75-85 — 47 running (64, 400, 64, 10) vs idle
    kats.append(("predictor_loaded_47", R, [(64, 400, 64, 10)] * 47, [], (512, 10)))
    # test_predictor.cpp:87-96 — determinism fixture
    kats.append(("predictor_determinism", R, [(128, 300, 128, 40)] * 20, [(900, 250, 0, 0)],
                 (700, 120)))
    # test_predictor.cpp:98-111 — exact cache transparency fixture
    kats.append(("predictor_exact_cache", dict(cache_mode=abi.CACHE_EXACT),
                 [(96, 280, 96, 15)] * 30, [(600, 100, 0, 0)], (444, 75)))
    # test_predictor.cpp:113-125 — bucketed fixture (exact and bucketed)
    kats.append(("predictor_bucketed_exact", R, [(200, 320, 200, 60)] * 24, [], (512, 64)))
    kats.append(("predictor_bucketed_256", dict(cache_mode=abi.CACHE_BUCKETED, context_bucket=256),
                 [(200, 320, 200, 60)] * 24, [], (512, 64)))
    # test_predictor.cpp:127-147 — predict_across instances 0,1,2 with id*10 running
    for i in range(3):
        kats.append((f"predictor_across_{i}", R, [(64, 200, 64, 20)] * (i * 10), [], (300, 40)))
    # test_predictor.cpp:149-158 — identical snapshots
    kats.append(("predictor_identical", R, [(64, 100, 64, 3)] * 5, [], (256, 32)))
    # test_predictor.cpp:160-171 — impossible candidate -> PredictionError
    kats.append(("predictor_impossible", dict(total_blocks=4, block_size=16, chunk_budget=64), [],
                 [], (512, 512)))
    # test_backend.cpp:82-96 — piggyback chunk 472 behind 40 decoders
    kats.append(("backend_piggyback_472", R, [(64, 512, 64, 8)] * 40, [(1200, 64, 0, 0)], (64, 4)))
    # test_backend.cpp:98-112, 114-126 — prefill priority
    kats.append(("backend_prefill_priority", dict(local_policy=abi.PREFILL_PRIORITY),
                 [(64, 512, 64, 8)] * 10, [(300, 64, 0, 0)], (64, 4)))
    kats.append(("backend_prefill_priority_decode", dict(local_policy=abi.PREFILL_PRIORITY),
                 [(64, 512, 64, 8)] * 10, [], (64, 4)))
    # test_backend.cpp:133-143 — block boundary allocation
    kats.append(("backend_block_boundary", R, [(32, 1000, 32, 0)], [], (16, 2)))
    # test_backend.cpp:145-166 — preemption of the newest member (6 blocks)
    kats.append(("backend_preempt_newest", dict(total_blocks=6, block_size=16),
                 [(32, 1000, 32, 0)] * 3, [], (16, 2)))
    # test_backend.cpp:168-179 — final decode completes
    kats.append(("backend_final_decode", R, [(32, 5, 32, 4)], [], (100, 3)))
    # test_backend.cpp:181-194 — finishing a prompt emits the first token
    kats.append(("backend_first_token", R, [], [], (100, 3)))
    # test_backend.cpp:196-211 — FCFS prefill order (6 x 700-token prompts)
    kats.append(("backend_fcfs", R, [], [(700, 16, 0, 0)] * 5, (700, 16)))
    # acceptance_main.cpp:675-699 — criterion 11 snapshot fixtures (candidate 300/80)
    c11 = [
        ([], []),
        ([(64, 300, 64, 10), (64, 300, 64, 20)], []),
        ([(64, 50, 64, 45)], []),
        ([(96, 100, 96, 120)], [(800, 100, 0, 0)]),
        ([(96, 100, 96, 20)], [(100, 50, 60, 0)]),
        ([(128, 260, 128, 40)] * 40, []),
        ([(64, 400, 64, 5)], []),
        ([], [(4000, 800, 0, 0)]),
        ([], [(900, 300, 0, 0), (200, 60, 0, 0)]),
        ([(300, 200, 300, 199)], []),
    ]
    for i, (run, wait) in enumerate(c11):
        kats.append((f"acceptance_c11_{i}", R, run, wait, (300, 80)))
    # acceptance C8 / test_predictor.cpp:41-53 — +10 correction on running and waiting
    kats.append(("correction_running_waiting", R,
                 [(100, 100, 100, 50), (100, 100, 100, 120), (100, 100, 100, 100)],
                 [(100, 80, 0, 0), (50, 5, 0, 9)], (100, 20)))
    return kats


def kat_set():
    kats = reference_kat_scenarios()
    cfgs, idx = [], []
    for name, kw, run, wait, cand in kats:
        cfgs.append(abi.make_config(**kw))
        idx.append(len(cfgs) - 1)
    ss = abi.ScenarioSet.from_snapshots([(k[2], k[3]) for k in kats], [k[4] for k in kats], idx)
    return [k[0] for k in kats], np.concatenate(cfgs), ss

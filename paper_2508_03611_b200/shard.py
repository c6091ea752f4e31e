"""Multi-GPU sharding of the what-if path.

Scenarios are independent, so the path shards with no data-path collective:

* throughput mode (bench.py, cfg1-3): weak scaling — each rank replays and
  simulates its own arrival stream (``weak_seed``); only the max-over-ranks
  time and summed counts cross ranks (``reduce_max_sum``).
* latency mode (one dispatch across GPUs, cfg4): instance ``i`` lives on rank
  ``i % world`` (``instance_shard``) with all of its samples, so each rank's
  score sum is local; the only exchange is the argmin (``global_argmin``),
  exact for any int64 score and lowest-id ties (scheduler.cpp:138-150).
* sweep mode (cfg5): whole closed-loop cells are assigned longest-first to the
  least-loaded rank (``assign_cells_lpt``).

Collectives go through torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import heapq

import numpy as np

INT64_MAX = np.iinfo(np.int64).max


def weak_seed(rank: int, base: int = 1) -> int:
    """Arrival-stream seed of rank ``rank`` in weak scaling."""
    return base + rank


def instance_shard(n_inst: int, world: int, rank: int) -> np.ndarray:
    """Instance indices simulated by ``rank`` in latency mode."""
    return np.arange(rank, n_inst, world, dtype=np.int32)


def local_best(scores: np.ndarray, ids: np.ndarray) -> tuple[int, int]:
    """(score, id) minimum with lowest-id ties; (INT64_MAX, INT32_MAX) if empty."""
    if len(scores) == 0:
        return INT64_MAX, np.iinfo(np.int32).max
    scores = np.asarray(scores, np.int64)
    ids = np.asarray(ids, np.int64)
    m = scores.min()
    return int(m), int(ids[scores == m].min())


PACK_BITS = 16                            # instance id field of the packed key
PACK_SAT = (1 << (63 - PACK_BITS)) - 1    # largest score the packed key holds exactly


def group_range(n_groups: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous arrival groups [g0, g1) of ``rank`` in strong scaling (all
    what-ifs of one arrival stay on one GPU, so its argmin is local)."""
    return n_groups * rank // world, n_groups * (rank + 1) // world


def pack_key(score: int, inst: int, failed: bool = False) -> int:
    """The packed argmin key: min(score, 2^47 - 1) << 16 | id; -1 = failed
    (an empty shard packs (INT64_MAX, 0xffff), which loses to any real key)."""
    if failed:
        return -1
    if score == INT64_MAX:
        return (PACK_SAT << PACK_BITS) | ((1 << PACK_BITS) - 1)
    return (min(score, PACK_SAT) << PACK_BITS) | inst


def reduce_key(key, scores: np.ndarray, ids: np.ndarray, device=None, group=None) -> int:
    """Cross-rank argmin from the per-rank packed key the dispatch kernel left
    in device memory (bsg_dispatch_mc_sampled dev_keys): ONE all_reduce MIN
    over NCCL on the device tensor, then one 8-byte read. Returns -1 on every
    rank when any rank's shard failed (key -1 wins the MIN), and falls back to
    the exact two-pass reduce (with this rank's host scores) only when the
    winning score saturated the 47-bit field."""
    import torch
    import torch.distributed as dist
    t = key if device is not None else key.cpu()  # gloo (one-GPU test mode) reduces host tensors
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    k = int(t.item())
    if k < 0:
        return -1
    if (k >> PACK_BITS) < PACK_SAT:
        return k & ((1 << PACK_BITS) - 1)
    s, i = local_best(scores, ids)
    return _global_argmin_two_pass(s, i, device, group)


def global_argmin(scores: np.ndarray, ids: np.ndarray, device=None, group=None,
                  failed: bool = False) -> int:
    """Exact cross-rank argmin with lowest-id ties (scheduler.cpp:138-150).

    One collective in the common case: all_reduce MIN of the packed
    key (min(score, 2^47 - 1) << 16 | id) — the minimum is exact whenever the
    winning score is below the saturation point, since every other rank's key
    is then larger. Only when the winner saturated (scores >= 2^47 ticks, i.e.
    sums of ~39 hours of e2e) does it fall back to the two-pass reduce (MIN of
    the score, then MIN of the ids attaining it)."""
    import torch
    import torch.distributed as dist
    # A local problem (this rank's prediction failed, or an id the key cannot
    # hold) must not raise before the collective — the other ranks would block
    # in all_reduce. It packs key -1, so the reduced key fails on EVERY rank.
    bad_ids = bool(len(ids)) and (int(np.max(ids)) >= (1 << PACK_BITS) - 1 or int(np.min(ids)) < 0)
    s, i = local_best(scores, ids)
    t = torch.tensor([pack_key(s, i, failed or bad_ids)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    k = int(t.item())
    if k < 0:  # the same reduced value on every rank: uniform branches
        return -1
    if (k >> PACK_BITS) < PACK_SAT:
        return k & ((1 << PACK_BITS) - 1)
    return _global_argmin_two_pass(s, i, device, group)


def _global_argmin_two_pass(s: int, i: int, device=None, group=None) -> int:
    import torch
    import torch.distributed as dist
    t = torch.tensor([s], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    cand = torch.tensor([i if s == int(t.item()) else np.iinfo(np.int64).max], dtype=torch.int64,
                        device=device)
    dist.all_reduce(cand, op=dist.ReduceOp.MIN, group=group)
    return int(cand.item())


def reduce_max_sum(maxes: list[float], sums: list[int], device=None, group=None):
    """Max-over-ranks of timings and sums of counts."""
    import torch
    import torch.distributed as dist
    a = torch.tensor(maxes, dtype=torch.float64, device=device)
    b = torch.tensor(sums, dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(a, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)
    return [float(x) for x in a.tolist()], [int(x) for x in b.tolist()]


def assign_cells_lpt(costs, world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of sweep cells to ranks
    (deterministic: ties by cell index, then rank index)."""
    order = sorted(range(len(costs)), key=lambda c: (-costs[c], c))
    heap = [(0.0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for c in order:
        load, r = heapq.heappop(heap)
        out[r].append(c)
        heapq.heappush(heap, (load + float(costs[c]), r))
    return [sorted(x) for x in out]

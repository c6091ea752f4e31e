"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in
paper_2508_03611_b200/shard.py: the exact cross-rank argmin used when one
dispatch's instances are sharded across GPUs, the max/sum reductions of the
weak-scaling bench, and deterministic LPT cell assignment for sweeps."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    from paper_2508_03611_b200 import shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)
        out = {}
        for case in range(40):
            n_inst = int(rng.integers(1, 70))
            scores = rng.integers(0, 6, n_inst).astype(np.int64) * (1 << 40)  # many ties, packed path
            if case % 5 == 0:
                scores[:] = np.iinfo(np.int64).max - 7  # all equal at the top: two-pass fallback
            if case % 5 == 1:
                scores = rng.integers(1 << 47, 1 << 50, n_inst).astype(np.int64)  # saturated keys
                scores[rng.integers(0, n_inst)] = 5  # ...except one winner below saturation
            if case % 5 == 2:
                scores = rng.integers(1 << 47, 1 << 48, n_inst).astype(np.int64) // 3 * 3  # ties, all saturated
            mine = shard.instance_shard(n_inst, world, rank)
            out[case] = (shard.global_argmin(scores[mine], mine), int(np.argmin(scores)))
        # a failure (or an id the packed key cannot hold) on ONE rank: no hang,
        # and every rank sees the failed decision (shard.py:61)
        out["fail"] = (shard.global_argmin(np.array([5, 6]), np.array([rank, 2 + rank]),
                                           failed=(rank == 1)), -1)
        out["bad_id"] = (shard.global_argmin(np.array([5]), np.array([70000 if rank == 0 else 1])), -1)
        # the device-key path (bench cfg4 multi-GPU): per-rank packed keys -> one MIN
        import torch
        for case, (keys, exp) in enumerate([((shard.pack_key(9, 3), shard.pack_key(4, 8)), 8),
                                            ((shard.pack_key(4, 5), shard.pack_key(4, 2)), 2),
                                            ((shard.pack_key(4, 5), -1), -1)]):
            t = torch.tensor([keys[rank]], dtype=torch.int64)
            out[f"key{case}"] = (shard.reduce_key(t, np.array([0]), np.array([0])), exp)
        maxes, sums = shard.reduce_max_sum([1.5 + rank, 10.0 * rank], [100 + rank, 7])
        q.put((rank, out, maxes, sums))
    finally:
        dist.destroy_process_group()


def test_sharded_argmin_and_reductions_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, maxes, sums in results:
        for case, (got, exp) in out.items():
            assert got == exp, (rank, case, got, exp)  # lowest id wins ties, across ranks
        assert maxes == [2.5, 10.0] and sums == [201, 14]


def test_instance_shards_partition():
    from paper_2508_03611_b200 import shard
    for n in (1, 7, 64, 128):
        for w in (1, 2, 4, 8):
            parts = np.concatenate([shard.instance_shard(n, w, r) for r in range(w)])
            assert sorted(parts.tolist()) == list(range(n))


def test_lpt_assignment_balanced_and_deterministic():
    from paper_2508_03611_b200 import shard
    rng = np.random.default_rng(5)
    costs = rng.lognormal(0, 1.5, 300)
    a = shard.assign_cells_lpt(costs, 8)
    assert a == shard.assign_cells_lpt(costs, 8)
    assert sorted(sum(a, [])) == list(range(300))
    loads = [costs[x].sum() for x in a]
    assert max(loads) <= (sum(loads) / 8) * 1.05 + costs.max()


def test_strong_scaling_groups_partition():
    from paper_2508_03611_b200 import shard
    for g in (1, 5, 4999, 5000):
        for w in (1, 2, 3, 8):
            rs = [shard.group_range(g, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == g
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (rendezvous
    on 127.0.0.1); --dist-probe runs only the rank plumbing (gloo, no GPU)."""
    import json
    import subprocess
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-probe"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert lines == [{"probe": "dist", "world": 2, "rank_sum": 1, "ranks": 2}]

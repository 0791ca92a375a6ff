"""Multi-process host logic of the query-sharded search, on CPU with gloo
(world size 2): shard bounds cover every query exactly once, and the gather
returns the union of the per-rank records with global query ids."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_2698_b200.dist import gather_results, shard_bounds, shard_by_trajectory


def test_shard_bounds_partition():
    for n in (0, 1, 7, 100, 9975, 50880):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_shard_by_trajectory_keeps_trajectories_whole():
    traj = np.repeat(np.arange(25), 399)
    for world in (2, 3, 8):
        spans = [shard_by_trajectory(traj, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == traj.size
        for (a, b), (c, _) in zip(spans, spans[1:]):
            assert b == c
        for a, b in spans:
            if a < b:
                assert a == 0 or traj[a] != traj[a - 1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nq = 101
    lo, hi = shard_bounds(nq, rank, world)
    # fake per-rank results: each local query row k hits entries 3k and 3k+1
    local_q = torch.arange(hi - lo, dtype=torch.int32).repeat_interleave(2)
    eid = (local_q + lo) * 3 + torch.tensor([0, 1], dtype=torch.int32).repeat(hi - lo)
    tin = (local_q + lo).to(torch.float32) * 0.5
    tout = tin + 0.25
    if rank == 1:                  # an empty shard result must still work
        local_q, eid, tin, tout = local_q[:0], eid[:0], tin[:0], tout[:0]
    g = gather_results(local_q, eid, tin, tout, q_offset=lo, dst=0)
    if rank == 0:
        q.put((g[0].tolist(), g[1].tolist(), g[2].tolist(), g[3].tolist(), (lo, hi)))
    else:
        assert g is None
    dist.barrier()
    dist.destroy_process_group()


def test_gather_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    qid, eid, tin, tout, (lo, hi) = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # rank 0's shard only (rank 1 contributed nothing)
    assert len(qid) == 2 * (hi - lo)
    assert sorted(set(qid)) == list(range(lo, hi))
    for k, e, a, b in zip(qid, eid, tin, tout):
        assert e in (3 * k, 3 * k + 1)
        assert a == pytest.approx(0.5 * k) and b == pytest.approx(0.5 * k + 0.25)


def test_time_partition_is_a_partition_in_time_order():
    rng = np.random.default_rng(0)
    t0 = np.round(rng.uniform(0, 10, 1001), 1)            # ties on purpose
    from paper_1410_2698_b200.dist import time_partition
    for world in (1, 2, 3, 8):
        parts = [time_partition(t0, r, world) for r in range(world)]
        allr = np.concatenate(parts)
        assert np.array_equal(np.sort(allr), np.arange(1001))
        for a, b in zip(parts, parts[1:]):
            assert t0[a].max() <= t0[b].min()              # contiguous time ranges
        sizes = [p.size for p in parts]
        assert max(sizes) - min(sizes) <= 1

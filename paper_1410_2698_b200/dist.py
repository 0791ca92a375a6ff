"""Multi-GPU query sharding.

The search is data-parallel over query segments (§4: one thread per
query): queries are independent and the result set is the
union of the per-query results.  On N GPUs every rank holds D and its index
(replicated, built from the same input: the build is deterministic), answers a
contiguous shard of Q, and keeps its records device-resident.  The only
exchange step is the optional gather of the records to one rank
(``gather_results``), done with ``torch.distributed`` collectives (NCCL over
NVLink on the B200 box; gloo in the CPU tests).  Timing is max over ranks.
"""
from __future__ import annotations

import math

import numpy as np


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of n rows for ``rank`` of ``world``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_by_trajectory(traj: np.ndarray, rank: int, world: int) -> tuple[int, int]:
    """Slice [lo, hi) of rows that keeps whole trajectories on one rank.

    ``traj`` is the (non-decreasing) trajectory id of each query row; segments of
    a query trajectory stay together, which keeps the per-rank work
    similar when trajectories have similar lengths."""
    traj = np.asarray(traj)
    n = traj.shape[0]
    lo, hi = shard_bounds(n, rank, world)

    def snap(i):
        if i <= 0 or i >= n:
            return min(max(i, 0), n)
        # move to the start of the trajectory containing row i
        return int(np.searchsorted(traj, traj[i], side="left"))
    return snap(lo), snap(hi)


def search_sharded(index, queries, d: float, kind: str = "spatiotemporal", window=(-math.inf, math.inf),
                   rank: int | None = None, world: int | None = None, capacity: int = 0):
    """Search this rank's shard of ``queries`` (all ranks pass the full query set).

    Returns (result, q_offset): query ids in ``result`` are rows of the shard;
    add ``q_offset`` for rows of the full query set."""
    import torch.distributed as dist
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    lo, hi = shard_bounds(int(queries.shape[0]), rank, world)
    res = index.search(queries[lo:hi], d, window=window, kind=kind, capacity=capacity)
    return res, lo


def gather_results(qid, eid, t_in, t_out, q_offset: int = 0, dst: int = 0, group=None):
    """Gather per-rank result columns to rank ``dst`` (the exchange step).

    Inputs are 1-D tensors of equal length on the rank's device (CUDA with NCCL,
    CPU with gloo); query ids are shifted by ``q_offset`` to rows of the full
    query set.  Counts are exchanged first (all_gather of one int64 per rank);
    records are then all-gathered padded to the largest count (a single
    collective, no per-peer loops).  Returns the concatenated columns on
    ``dst`` (rank order), None elsewhere."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = qid.device
    n = torch.tensor([qid.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    mx = max(counts) if counts else 0
    # pack as int32 x 4 columns (times bit-cast), pad to the max count
    pack = torch.zeros((mx, 4), dtype=torch.int32, device=dev)
    k = qid.numel()
    if k:
        pack[:k, 0] = qid.to(torch.int32) + int(q_offset)
        pack[:k, 1] = eid.to(torch.int32)
        pack[:k, 2] = t_in.to(torch.float32).view(torch.int32)
        pack[:k, 3] = t_out.to(torch.float32).view(torch.int32)
    bufs = [torch.empty_like(pack) for _ in range(world)]
    dist.all_gather(bufs, pack, group=group)
    if rank != dst:
        return None
    allp = torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)
    return (allp[:, 0].clone(), allp[:, 1].clone(), allp[:, 2].clone().view(torch.float32),
            allp[:, 3].clone().view(torch.float32))


# ---------------------------------------------------------------------------
# Time-partitioned D sharding (the paper's intended scenario of
# "a number of GPU-equipped compute nodes"): D is split into `world`
# contiguous t_start ranges of equal entry count; each rank indexes only its
# slice (memory per GPU ~ |D| / N) and answers every query against it; the
# union of the ranks' records is the answer (each entry lives on one rank, so
# the union has no duplicates).  Entry ids are mapped back to rows of D.
# ---------------------------------------------------------------------------
def time_partition(t_start: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Global rows of D owned by ``rank``: the rank-th of ``world`` equal-count
    slices of D in (t_start, row) order (stable)."""
    order = np.argsort(np.asarray(t_start), kind="stable")
    lo, hi = shard_bounds(order.size, rank, world)
    return np.sort(order[lo:hi])


class TimeShardedIndex:
    """This rank's index over its t_start slice of D."""

    def __init__(self, D, rank: int, world: int, kinds: int = 5, m: int = 1000, v: int = 1,
                 grid=(50, 50, 50), device=None):
        import torch
        import paper_1410_2698_b200 as tds
        Dn = D.cpu().numpy() if isinstance(D, torch.Tensor) else np.asarray(D)
        rows = time_partition(Dn[:, 3], rank, world)
        self.rows = torch.as_tensor(rows.astype(np.int32), device=device or "cuda")
        self.index = tds.Index(torch.as_tensor(np.ascontiguousarray(Dn[rows]), device=device or "cuda"),
                               kinds=kinds, m=m, v=v, grid=grid)
        self.rank, self.world = rank, world

    def search(self, queries, d: float, kind: str = "temporal", window=(-math.inf, math.inf), capacity: int = 0):
        """(qid, eid, t_in, t_out) device tensors for this slice; eid = rows of D."""
        r = self.index.search(queries, d, window=window, kind=kind, capacity=capacity)
        q, e, ti, to = r.fetch(device=True)
        e = self.rows[e.long()]
        r.close()
        return q, e, ti, to

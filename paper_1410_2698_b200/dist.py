"""Multi-GPU search.

The search is data-parallel over query segments (§4: one thread per
query): queries are independent and the result set is the
union of the per-query results.  Two partitionings, one process per GPU:

* **Query sharding, D replicated** (SURVEY §8(e)).  Every rank holds D and its
  index (built from the same input: the build is deterministic) and the full
  query set.  ``search_sharded`` runs part ``rank`` of ``world`` of a
  work-balanced split (``tds_search_part``): the library computes the schedule
  of the full query set on the device and evaluates the contiguous slice of the
  sorted schedule holding an equal share of the exact pair tests
  (Σ (hi − lo), prefix sum + binary search).  Results stay device-resident;
  ``gather_results`` is the one exchange step (counts, then each rank's
  records point-to-point to ``dst``: NCCL over NVLink on the B200 box).
* **Time-partitioned D** (the paper's distributed scenario
  "a number of GPU-equipped compute nodes"; reading C27).
  ``TimeShardedIndex`` gives rank r the r-th equal-count slice of D in
  (t_start, row) order, derived from a device sort of the t_start column
  (``tds_time_partition``), and indexes only that slice; every rank answers
  every query against its slice, entry ids are mapped back to rows of D on the
  device, and the union of the ranks' records (``gather_results``) is the
  answer (every entry lives on exactly one rank: no duplicates).

Timing is max over ranks.
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
    """Slice [lo, hi) of rows that keeps whole trajectories on one rank (for
    callers that shard the query input themselves)."""
    traj = np.asarray(traj)
    n = traj.shape[0]
    lo, hi = shard_bounds(n, rank, world)

    def snap(i):
        if i <= 0 or i >= n:
            return min(max(i, 0), n)
        return int(np.searchsorted(traj, traj[i], side="left"))
    return snap(lo), snap(hi)


def _rank_world(rank, world, group=None):
    import torch.distributed as dist
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    return rank, world


def search_sharded(index, queries, d: float, kind: str = "spatiotemporal", window=(-math.inf, math.inf),
                   rank: int | None = None, world: int | None = None, capacity: int = 0, stream=None):
    """This rank's work-balanced part of the search of the FULL query set
    (every rank passes the same ``queries``).  Query ids in the result are rows
    of the full query set; the parts are disjoint and their union is the
    single-GPU result."""
    rank, world = _rank_world(rank, world)
    return index.search(queries, d, window=window, kind=kind, capacity=capacity, stream=stream, part=rank,
                        nparts=world)


def _pack(qid, eid, t_in, t_out, q_offset, dev):
    import torch
    k = qid.numel()
    pack = torch.empty((k, 4), dtype=torch.int32, device=dev)
    if k:
        pack[:, 0] = qid.to(device=dev, dtype=torch.int32) + int(q_offset)
        pack[:, 1] = eid.to(device=dev, dtype=torch.int32)
        pack[:, 2] = t_in.to(device=dev, dtype=torch.float32).view(torch.int32)
        pack[:, 3] = t_out.to(device=dev, dtype=torch.float32).view(torch.int32)
    return pack


def gather_results(qid, eid, t_in, t_out, q_offset: int = 0, dst: int = 0, group=None):
    """Gather per-rank result columns to rank ``dst`` (the exchange step of
    SURVEY §8(e)).

    Inputs are 1-D tensors of equal length (CUDA or CPU).  Counts are
    exchanged first (all_gather of one int64 per rank), then every other rank
    sends its records, packed 16 B each, point-to-point to ``dst``, which
    receives them into one exactly sized buffer (no padding, no copies on the
    other ranks).  NCCL moves CUDA tensors over NVLink; with gloo the records
    travel through host memory.  Returns the concatenated columns (rank
    order) on ``dst``, None elsewhere."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = qid.device if nccl else torch.device("cpu")
    n = torch.tensor([qid.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    pack = _pack(qid, eid, t_in, t_out, q_offset, dev)
    gdst = dst if group is None else dist.get_global_rank(group, dst)
    if rank != dst:
        if counts[rank]:
            dist.send(pack, gdst, group=group)
        return None
    out = torch.empty((sum(counts), 4), dtype=torch.int32, device=dev)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    ops = []
    for r in range(world):
        if r == rank or counts[r] == 0:
            continue
        src = r if group is None else dist.get_global_rank(group, r)
        if nccl:
            ops.append(dist.P2POp(dist.irecv, out[offs[r]:offs[r + 1]], src, group=group))
        else:
            buf = out[offs[r]:offs[r + 1]]
            dist.recv(buf, src, group=group)
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    if counts[rank]:
        out[offs[rank]:offs[rank + 1]] = pack
    return (out[:, 0].clone(), out[:, 1].clone(), out[:, 2].clone().view(torch.float32),
            out[:, 3].clone().view(torch.float32))


# ---------------------------------------------------------------------------
# Time-partitioned D sharding
# ---------------------------------------------------------------------------
def time_partition(t_start: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Host statement of the partition rule C27 (for CPU tests of callers):
    rows of D at positions [rank n / world, (rank+1) n / world) of the stable
    (t_start, row) order.  The product path uses the device sort
    (``paper_1410_2698_b200.time_partition`` / tds_time_partition)."""
    order = np.argsort(np.asarray(t_start), kind="stable")
    n = order.size
    return order[n * rank // world: n * (rank + 1) // world]


class TimeShardedIndex:
    """This rank's index over its t_start slice of D.

    ``D`` is the full database as a float32 [n, 8] tensor, on the device or in
    (pinned) host memory; only its t_start column and this rank's rows are
    moved to the GPU."""

    def __init__(self, D, rank: int, world: int, kinds: int = 5, m: int = 1000, v: int = 1,
                 grid=(50, 50, 50), device=None):
        import torch
        import paper_1410_2698_b200 as tds
        dev = torch.device(device or "cuda")
        Dt = D if isinstance(D, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(D, dtype=np.float32))
        t0 = Dt[:, 3].contiguous()
        self.rows = tds.time_partition(t0, rank, world)          # device, (t_start, row) order
        if Dt.is_cuda:
            Ds = Dt.index_select(0, self.rows.long())
        else:
            Ds = Dt.index_select(0, self.rows.long().cpu()).to(dev)
        self.n_local = int(self.rows.numel())
        self.index = tds.Index(Ds.contiguous(), kinds=kinds, m=m, v=v, grid=grid)
        self.rank, self.world = rank, world

    def search(self, queries, d: float, kind: str = "temporal", window=(-math.inf, math.inf), capacity: int = 0):
        """(qid, eid, t_in, t_out) device tensors for this slice; eid = rows of D."""
        r = self.index.search(queries, d, window=window, kind=kind, capacity=capacity)
        q, e, ti, to = r.fetch(device=True)
        e = self.rows[e.long()]
        r.close()
        return q, e, ti, to

"""Seeded synthetic workloads shaped like the paper's datasets.

This module holds ONLY the input generators.  It contains none of the
method's arithmetic (no distance test, no index, no schedule), so that it can
serve both the oracle tests and the CUDA path without coupling them
(task rule ③: "only the seeded input generators serve both").

Segment record layout (shared by every consumer): float32 ``[n, 8]`` rows
``(x0, y0, z0, t0, x1, y1, z1, t1)`` — a 4-D line segment from a start point
to an end point (§3.1).  Consecutive segments of one
trajectory share endpoints bit-exactly (trajectories are polylines).

Datasets (§5.1, Table 1; readings in
DESIGN.md "Input recipe"):

* ``tiny``          — 50 random-walk trajectories x 20 segments, 5 separate
                       query trajectories x 20 (BASELINE.json configs[0]).
* ``random_1m``     — Random-1M: 2,500 trajectories x 400 timesteps = 997,500
                       segments, start times U[0,100].  Spatial
                       scale/step law unstated in the paper: cube 1000^3 centred
                       on the origin, per-dim steps U[-1,1].
* ``random_dense``  — Random-dense: 65,536 particles x 193 timesteps at
                       0.112 stars/pc^3 -> cube 83.64 pc, steps
                       0.001-0.005 kpc per dim, forced back when > 20% outside
                       (SURVEY C18).  Units: kpc.
* ``merger``        — Merger-shaped: 131,072 particles x 193 snapshots of two
                       rotating exponential disks on a merging orbit (the real
                       data, is unavailable).  Units: kpc.
* ``query_stride``  — the query trajectories drawn from D with a stride
                       (S2/S3 use 265 trajectories).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

BASE_SEED = 1410269800

__all__ = [
    "Workload", "BASE_SEED", "random_walk", "tiny", "random_1m", "random_1m_s1",
    "random_dense", "merger", "scale_out", "query_stride", "segments_from_positions",
    "dense_cube_side_kpc", "CONFIGS", "make_workload", "stationary_queries",
]


@dataclass
class Workload:
    """A database D, a query set Q and the parameters of one configuration."""
    name: str
    D: np.ndarray            # float32 [nD, 8]
    Q: np.ndarray            # float32 [nQ, 8]
    d: float                 # default distance threshold
    m_bins: int              # temporal bins
    v_subbins: int           # spatial subbins per temporal bin
    grid: tuple              # FSG cells per dim
    traj_D: np.ndarray       # int32 trajectory id per D row
    traj_Q: np.ndarray       # int32 trajectory id per Q row
    note: str = ""


def segments_from_positions(pos: np.ndarray, times: np.ndarray) -> np.ndarray:
    """Turn per-trajectory vertex positions into 4-D segment records.

    pos   : float32 [n_traj, n_steps, 3]
    times : float32 [n_traj, n_steps]
    returns float32 [n_traj * (n_steps - 1), 8], trajectory-major.
    """
    n_traj, n_steps, _ = pos.shape
    seg = np.empty((n_traj, n_steps - 1, 8), dtype=np.float32)
    seg[:, :, 0:3] = pos[:, :-1, :]
    seg[:, :, 3] = times[:, :-1]
    seg[:, :, 4:7] = pos[:, 1:, :]
    seg[:, :, 7] = times[:, 1:]
    return seg.reshape(-1, 8)


def random_walk(n_traj: int, n_steps: int, seed: int, *, t_window: float = 100.0,
                box: float = 1000.0, step_max: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """Random-walk trajectories (§5.1, SPEC S:156 defaults).

    Start times U[0, t_window]; unit-time steps; start positions uniform in a
    cube of side ``box`` centred on the origin; each step adds U[-step_max,
    step_max] independently per dimension.  Returns (segments, traj_id).
    """
    rng = np.random.Generator(np.random.Philox(key=seed))
    start = rng.uniform(-box / 2, box / 2, size=(n_traj, 1, 3))
    steps = rng.uniform(-step_max, step_max, size=(n_traj, n_steps - 1, 3))
    pos = np.concatenate([start, start + np.cumsum(steps, axis=1)], axis=1).astype(np.float32)
    t_start = rng.uniform(0.0, t_window, size=(n_traj, 1))
    times = (t_start + np.arange(n_steps)[None, :]).astype(np.float32)
    seg = segments_from_positions(pos, times)
    traj = np.repeat(np.arange(n_traj, dtype=np.int32), n_steps - 1)
    return seg, traj


def query_stride(D: np.ndarray, traj_D: np.ndarray, n_query_traj: int,
                 offset: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Query set = ``n_query_traj`` whole trajectories of D taken with a stride.

    The Merger query set can only have come from D; the same is
    done for Random-dense and for the "1% of trajectories"
    Random-1M set of BASELINE.json.  ``offset`` shifts the picked trajectories
    (used to give each rank its own equally-sized query set, weak scaling).
    """
    n_traj = int(traj_D.max()) + 1
    stride = n_traj // n_query_traj
    assert stride >= 1 and 0 <= offset < stride
    picked = offset + stride * np.arange(n_query_traj)
    mask = np.isin(traj_D, picked)
    return D[mask].copy(), traj_D[mask].copy()


def tiny(seed: int = BASE_SEED + 0) -> Workload:
    """BASELINE.json configs[0]: 50 trajectories x 20 segments, 5 query trajectories.

    t0 ~ U[0,5], unit-time steps, start positions U[0,10]^3 (centred), steps
    U[-0.5,0.5]; d = 2.0 (1-20% of temporally overlapping pairs hit).
    """
    D, tD = random_walk(50, 21, seed, t_window=5.0, box=10.0, step_max=0.5)
    Q, tQ = random_walk(5, 21, seed + 1, t_window=5.0, box=10.0, step_max=0.5)
    return Workload("tiny", D, Q, 2.0, 10, 2, (4, 4, 4), tD, tQ,
                    "50x20 D, 5x20 separate Q")


def random_1m(seed: int = BASE_SEED + 1, n_traj: int = 2500, query_frac_stride: int = 100,
              offset: int = 0, d: float = 50.0) -> Workload:
    """Random-1M-shaped (Table 1: 2,500 x 400 = 997,500).

    Query set = 1% of the trajectories (every 100th, a subset of D), as
    BASELINE.json configs[1] states.  m = 10,000 bins, FSG 50^3
    (P:1391), v = 4.
    """
    D, tD = random_walk(n_traj, 400, seed)
    Q, tQ = query_stride(D, tD, n_traj // query_frac_stride, offset)
    return Workload("random-1m", D, Q, d, 10000, 4, (50, 50, 50), tD, tQ,
                    f"Q = every {query_frac_stride}th trajectory of D (offset {offset})")


def random_1m_s1(seed: int = BASE_SEED + 1) -> Workload:
    """Scenario S1: Random-1M D with 100 separate query trajectories."""
    D, tD = random_walk(2500, 400, seed)
    Q, tQ = random_walk(100, 400, seed + 1)
    return Workload("random-1m-s1", D, Q, 50.0, 10000, 4, (50, 50, 50), tD, tQ,
                    "S1: 100 separate query trajectories = 39,900")


def dense_cube_side_kpc(n_particles: int, density_pc3: float = 0.112) -> float:
    """Cube side for ``n_particles`` at the solar-neighbourhood density."""
    return (n_particles / density_pc3) ** (1.0 / 3.0) / 1000.0


def random_dense(n_particles: int = 65536, n_timesteps: int = 193, seed: int = BASE_SEED + 2,
                 n_query_traj: int = 265, offset: int = 0, d: float = 0.03,
                 v_subbins: int = 2) -> Workload:
    """Random-dense-shaped (Table 1: 65,536 x 193 -> 12,582,912).

    All particles start at t = 0 uniformly inside a cube of side
    L = (N / 0.112 pc^-3)^(1/3) centred on the origin; timesteps are the
    integers 0..192; each step moves each coordinate by a magnitude
    U[0.001, 0.005] kpc with a random sign, except that a coordinate that is
    more than 0.2 L outside the cube steps back towards it.
    Units kpc.  m = 1,000, v = 2.
    """
    rng = np.random.Generator(np.random.Philox(key=seed))
    L = dense_cube_side_kpc(n_particles)
    half = L / 2.0
    pos = np.empty((n_particles, n_timesteps, 3), dtype=np.float64)
    pos[:, 0, :] = rng.uniform(-half, half, size=(n_particles, 3))
    for k in range(1, n_timesteps):
        prev = pos[:, k - 1, :]
        mag = rng.uniform(0.001, 0.005, size=(n_particles, 3))
        sign = np.where(rng.random(size=(n_particles, 3)) < 0.5, -1.0, 1.0)
        sign = np.where(prev > half + 0.2 * L, -1.0, sign)
        sign = np.where(prev < -half - 0.2 * L, 1.0, sign)
        pos[:, k, :] = prev + sign * mag
    pos32 = pos.astype(np.float32)
    times = np.broadcast_to(np.arange(n_timesteps, dtype=np.float32), (n_particles, n_timesteps))
    D = segments_from_positions(pos32, times)
    tD = np.repeat(np.arange(n_particles, dtype=np.int32), n_timesteps - 1)
    Q, tQ = query_stride(D, tD, n_query_traj, offset)
    return Workload("random-dense", D, Q, d, 1000, v_subbins, (50, 50, 50), tD, tQ,
                    f"cube {L * 1000:.2f} pc, {n_query_traj} query trajectories from D")


def merger(n_per_disk: int = 65536, n_timesteps: int = 193, seed: int = BASE_SEED + 3,
           n_query_traj: int = 265, offset: int = 0, d: float = 1.0) -> Workload:
    """Merger-shaped synthetic (stand-in for P:1207-1213; real data unavailable).

    Two disks of ``n_per_disk`` particles each.  Per particle: cylindrical
    radius from an exponential surface density (scale 3 kpc, truncated at
    15 kpc), uniform initial phase, Gaussian height sigma 0.3 kpc.  Circular
    orbits with rotation curve v(R) = v_c R / sqrt(R^2 + 1 kpc^2), v_c =
    3.2 kpc per snapshot (200 km/s x 15.625 Myr).  Disk 1 is tilted 60 deg
    about x and counter-rotates.  Disk centres sit at +/- sep(t)/2 along a
    direction u(t) = normalise(cos th, sin th, 0.9), th turning from 45 to
    135 deg; sep(t) = 80 cos(pi/2 * t/120) kpc, merged (sep = 0) from
    snapshot 120 on.  Generator self-check: admissible v >= 16 per dimension
    (P:816-821 with v = 16).
    193 snapshots 0..192 (3 Gyr).  m = 1,000, v = 16.
    """
    rng = np.random.Generator(np.random.Philox(key=seed))
    n = 2 * n_per_disk
    # exponential disk: surface density ~ exp(-R/Rd) -> R ~ Gamma(2, Rd), truncated
    R = rng.gamma(2.0, 3.0, size=n)
    while True:
        bad = R > 15.0
        if not bad.any():
            break
        R[bad] = rng.gamma(2.0, 3.0, size=int(bad.sum()))
    phi0 = rng.uniform(0.0, 2 * math.pi, size=n)
    zh = rng.normal(0.0, 0.3, size=n)
    omega = 3.2 / np.sqrt(R * R + 1.0)                 # rad per snapshot
    spin = np.concatenate([np.ones(n_per_disk), -np.ones(n_per_disk)])
    t = np.arange(n_timesteps, dtype=np.float64)
    ang = phi0[:, None] + (spin * omega)[:, None] * t[None, :]
    local = np.empty((n, n_timesteps, 3), dtype=np.float64)
    local[:, :, 0] = R[:, None] * np.cos(ang)
    local[:, :, 1] = R[:, None] * np.sin(ang)
    local[:, :, 2] = zh[:, None]
    # tilt disk 1 by 60 degrees about the x axis
    c, s = math.cos(math.radians(60.0)), math.sin(math.radians(60.0))
    y1 = local[n_per_disk:, :, 1].copy()
    z1 = local[n_per_disk:, :, 2].copy()
    local[n_per_disk:, :, 1] = c * y1 - s * z1
    local[n_per_disk:, :, 2] = s * y1 + c * z1
    # orbit of the two centres
    tm = np.minimum(t, 120.0) / 120.0
    sep = 80.0 * np.cos(0.5 * math.pi * tm)
    theta = 0.25 * math.pi + 0.5 * math.pi * tm
    u = np.stack([np.cos(theta), np.sin(theta), np.full_like(theta, 0.9)], axis=1)
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    centre = 0.5 * sep[:, None] * u                    # [T, 3]
    local[:n_per_disk] += centre[None, :, :]
    local[n_per_disk:] -= centre[None, :, :]
    pos32 = local.astype(np.float32)
    del local
    times = np.broadcast_to(np.arange(n_timesteps, dtype=np.float32), (n, n_timesteps))
    D = segments_from_positions(pos32, times)
    tD = np.repeat(np.arange(n, dtype=np.int32), n_timesteps - 1)
    Q, tQ = query_stride(D, tD, n_query_traj, offset)
    return Workload("merger", D, Q, d, 1000, 16, (50, 50, 50), tD, tQ,
                    f"two disks x {n_per_disk}, {n_query_traj} query trajectories from D")


def scale_out(n_traj: int = 250_000, n_steps: int = 400, seed: int = BASE_SEED + 4, query_stride: int = 10,
              shard: tuple = (0, 1), d: float = 50.0) -> Workload:
    """Scale-out (BASELINE.json configs[4]): a 100M-segment random-walk database
    (250,000 trajectories x 400 timesteps = 99,750,000 segments) at the Random-1M
    density (cube side 1000 * 100^(1/3) ~= 4642, steps U[-1,1], start times
    U[0,100]), and 10% of its trajectories (every 10th) as the query set
    (25,000 x 399 = 9,975,000 query segments).  ``shard = (rank, world)`` keeps
    every world-th query trajectory starting at rank (strong scaling: the query
    set is split across GPUs).  Generated in chunks of trajectories straight
    into the float32 output (peak host memory ~ 1.2x the 3.2 GB database).
    m = 10,000 bins, v = 4.
    """
    box = 1000.0 * (n_traj / 2500.0) ** (1.0 / 3.0)
    D = np.empty((n_traj * (n_steps - 1), 8), dtype=np.float32)
    chunk = 10_000
    rng = np.random.Generator(np.random.Philox(key=seed))
    for t0 in range(0, n_traj, chunk):
        nt = min(chunk, n_traj - t0)
        start = rng.uniform(-box / 2, box / 2, size=(nt, 1, 3))
        steps = rng.uniform(-1.0, 1.0, size=(nt, n_steps - 1, 3))
        pos = np.concatenate([start, start + np.cumsum(steps, axis=1)], axis=1).astype(np.float32)
        t_start = rng.uniform(0.0, 100.0, size=(nt, 1))
        times = (t_start + np.arange(n_steps)[None, :]).astype(np.float32)
        D[t0 * (n_steps - 1):(t0 + nt) * (n_steps - 1)] = segments_from_positions(pos, times)
    tD = np.repeat(np.arange(n_traj, dtype=np.int32), n_steps - 1)
    rank, world = shard
    qtraj = np.arange(0, n_traj, query_stride)[rank::world]
    Dr = D.reshape(n_traj, n_steps - 1, 8)
    Q = np.ascontiguousarray(Dr[qtraj].reshape(-1, 8))
    tQ = np.repeat(qtraj.astype(np.int32), n_steps - 1)
    return Workload("scale-out", D, Q, d, 10000, 4, (50, 50, 50), tD, tQ,
                    f"100M database at Random-1M density (cube {box:.0f}); query trajectories every "
                    f"{query_stride}th, shard {rank}/{world}")


def stationary_queries(D: np.ndarray, n_points: int, n_steps: int, seed: int = BASE_SEED + 5) -> np.ndarray:
    """Stationary-point queries (the paper's case (i), "a supernova explosion at a
    point over a time interval"): ``n_points`` fixed positions, each the
    start point of a random entry of D, observed over ``n_steps`` consecutive
    unit-time segments from that entry's t_start (P1 = P0 in every segment).
    float32 [n_points * n_steps, 8]."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    rows = rng.integers(0, D.shape[0], size=n_points)
    p = D[rows, 0:3].astype(np.float32)
    t = D[rows, 3].astype(np.float64)
    Q = np.empty((n_points, n_steps, 8), dtype=np.float32)
    for k in range(n_steps):
        Q[:, k, 0:3] = p
        Q[:, k, 4:7] = p
        Q[:, k, 3] = (t + k).astype(np.float32)
        Q[:, k, 7] = (t + k + 1).astype(np.float32)
    return Q.reshape(-1, 8)


CONFIGS = {
    "tiny": tiny,
    "random-1m": random_1m,
    "random-1m-s1": random_1m_s1,
    "random-dense": random_dense,
    "random-dense-1m": lambda **kw: random_dense(n_particles=5184, **kw),
    "merger": merger,
    "scale-out": scale_out,
}


def make_workload(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)

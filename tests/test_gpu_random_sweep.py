"""Seeded randomized parity sweep: small random workloads (uniform or clustered
positions, random segment durations, aligned or ragged times, stationary
segments), random index parameters (m, v within the admissible bound, grid),
random d, random query windows and capacities (including tiny ones that force
overflow re-plans), every variant including TDS_AUTO, compared element by
element with the fp64 oracle (pair set exact outside the 1e-5 d band, endpoints
within 1e-5)."""
import numpy as np
import pytest

import oracle
from parity import check

pytestmark = pytest.mark.gpu


def make_case(seed):
    rng = np.random.default_rng(1410269900 + seed)
    ntraj = int(rng.integers(20, 300))
    nseg = int(rng.integers(2, 40))
    box = float(rng.choice([1.0, 10.0, 1000.0]))
    if rng.random() < 0.5:
        start = rng.uniform(0, box, (ntraj, 1, 3))
    else:   # clustered
        centres = rng.uniform(0, box, (4, 3))
        start = centres[rng.integers(0, 4, ntraj)][:, None, :] + rng.normal(0, box / 50, (ntraj, 1, 3))
    step = box / 100 * rng.uniform(0.1, 2.0)
    steps = rng.uniform(-step, step, (ntraj, nseg, 3))
    steps[rng.random((ntraj, nseg)) < 0.1] = 0.0                     # stationary segments
    pos = np.concatenate([start, start + np.cumsum(steps, axis=1)], axis=1)
    if rng.random() < 0.5:   # aligned integer timesteps
        t = np.arange(nseg + 1, dtype=np.float64)[None, :] + rng.integers(0, 5, (ntraj, 1))
    else:                    # ragged durations and offsets
        dt = rng.uniform(0.2, 2.0, (ntraj, nseg))
        t = np.concatenate([np.zeros((ntraj, 1)), np.cumsum(dt, axis=1)], axis=1) + rng.uniform(0, 10, (ntraj, 1))
    P = np.concatenate([pos, t[:, :, None]], axis=2)
    D = np.concatenate([P[:, :-1, :], P[:, 1:, :]], axis=2).reshape(-1, 8).astype(np.float32)
    nq = int(rng.integers(1, 400))
    Q = D[rng.choice(D.shape[0], nq, replace=nq > D.shape[0])].copy()
    if rng.random() < 0.3:   # some queries not from D
        Q[:, [0, 1, 2, 4, 5, 6]] += rng.normal(0, step, (nq, 6)).astype(np.float32)
    d = float(step * rng.choice([0.3, 1.0, 5.0, 20.0]))
    tmin, tmax = float(D[:, 3].min()), float(D[:, 7].max())
    if rng.random() < 0.4:
        a, b = np.sort(rng.uniform(tmin, tmax, 2))
        window = (float(a), float(b))
    else:
        window = (-np.inf, np.inf)
    # admissible v: extent / max per-segment extent per dimension
    lo = np.minimum(D[:, [0, 1, 2]].min(0), D[:, [4, 5, 6]].min(0)).astype(np.float64)
    hi = np.maximum(D[:, [0, 1, 2]].max(0), D[:, [4, 5, 6]].max(0)).astype(np.float64)
    seg = np.abs(D[:, [4, 5, 6]] - D[:, [0, 1, 2]]).max(0).astype(np.float64)
    bound = np.where(seg > 0, (hi - lo) / np.maximum(seg, 1e-300), 64.0)
    vmax = int(max(1, np.floor(bound.min() * (1 - 1e-6))))
    params = dict(m=int(rng.integers(1, 200)), v=int(rng.integers(1, min(vmax, 8) + 1)),
                  grid=tuple(int(x) for x in rng.integers(1, 24, 3)))
    capacity = int(rng.choice([0, 0, 0, 7, 100, 1000]))
    return D, Q, d, window, params, capacity


@pytest.fixture(scope="module")
def tds():
    import paper_1410_2698_b200 as t
    t.load_library()
    return t


@pytest.mark.parametrize("seed", range(200))
def test_random_case(tds, seed):
    import torch
    D, Q, d, window, params, capacity = make_case(seed)
    ref = oracle.search(D, Q, d, window=window)
    idx = tds.Index(torch.from_numpy(D).cuda(), kinds=tds.ALL, **params)
    for kind in ("temporal", "spatiotemporal", "spatial", "auto"):
        try:
            r = idx.search(torch.from_numpy(Q).cuda(), d, window=window, kind=kind, capacity=capacity)
        except tds.TdsError as e:
            # a tiny capacity below one query's own output is the one allowed failure
            assert capacity and "ECAPACITY" in str(e), str(e)
            continue
        got = r.fetch(sorted=True, device=False)
        check(got, ref, D, Q, d, label=f"seed {seed} {kind} {params} cap {capacity} window {window}")

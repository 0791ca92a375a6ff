"""Generator pins: Table 1 counts, query-set sizes, the Random-dense cube side,
trajectory continuity, determinism, the Merger-shaped admissible v, and two
statistics the paper prints for Random-dense (S3) that pin density and
shape: the fraction of entries within d and the fraction of
queries that can use subbins."""
import math

import numpy as np
import pytest

import oracle
import synth
from oracle import index_ref as ir


def test_random_1m_counts_and_continuity():
    w = synth.random_1m()
    assert w.D.shape == (997_500, 8)                 # Table 1
    assert w.Q.shape == (9_975, 8)                   # 1% of trajectories x 399
    Dr = w.D.reshape(2500, 399, 8)
    assert np.array_equal(Dr[:, :-1, 4:8], Dr[:, 1:, 0:4])   # polylines: shared endpoints
    assert np.all(w.D[:, 7] > w.D[:, 3])
    t0 = Dr[:, 0, 3]
    assert t0.min() >= 0 and t0.max() <= 100                 # start times U[0,100]
    # Q is a subset of D (every 100th trajectory)
    assert np.array_equal(w.Q[:399], Dr[0]) and np.array_equal(w.Q[399:798], Dr[100])


def test_s1_query_count():
    Q, _ = synth.random_walk(100, 400, 7)
    assert Q.shape[0] == 39_900


def test_determinism():
    a = synth.tiny()
    b = synth.tiny()
    assert a.D.tobytes() == b.D.tobytes() and a.Q.tobytes() == b.Q.tobytes()
    assert synth.tiny(seed=5).D.tobytes() != a.D.tobytes()


def test_cube_side():
    assert synth.dense_cube_side_kpc(65536) * 1000 == pytest.approx(83.64, abs=0.01)


@pytest.fixture(scope="module")
def dense():
    return synth.random_dense()


def test_random_dense_counts(dense):
    assert dense.D.shape == (12_582_912, 8)           # Table 1
    assert dense.Q.shape == (50_880, 8)               # S3
    steps = np.abs(dense.D[:, 4:7] - dense.D[:, 0:3])
    assert steps.min() >= 0.001 * (1 - 1e-3) and steps.max() <= 0.005 * (1 + 1e-3)
    L = synth.dense_cube_side_kpc(65536)
    assert np.abs(dense.D[:, 0:3]).max() <= L / 2 + 0.2 * L + 0.006          # forced back at 20%


def test_random_dense_fraction_within_d(dense):
    """~0% of entries within d=0.001, 73.9% within d=0.09 (S3).

    Read as hits / temporally overlapping pairs, sampled at six timesteps with
    64 query particles each; the paper's figure is matched within +/-5 points."""
    Dr = dense.D.reshape(65536, 192, 8)
    rng = np.random.default_rng(0)
    frac = {}
    for d in (0.001, 0.09):
        hits = tot = 0
        for k in (0, 24, 48, 96, 144, 191):
            Dk = np.ascontiguousarray(Dr[:, k, :])
            Qk = Dk[rng.choice(65536, 64, replace=False)]
            r = oracle.search(Dk, Qk, d, near=1.0)
            hits += int(r["hit"].sum())
            tot += 64 * 65536
        frac[d] = hits / tot
    assert frac[0.001] < 1e-3
    assert abs(frac[0.09] - 0.739) <= 0.05


def test_random_dense_subbin_usage(dense):
    """at d=0.03, v=2 -> just over 60% of queries use subbins; v=4 -> none.

    A query uses subbins iff its d-inflated MBB lies in one slab in at least
    one dimension (reading C15)."""
    lo, hi, _ = ir.spatial_extent(dense.D)
    Q = dense.Q[:: 10]
    d = 0.03
    for v, (fmin, fmax) in ((2, (0.60, 0.85)), (4, (0.0, 0.02))):
        w = (hi - lo) / v
        used = 0
        for q in Q:
            ok = False
            for c in range(3):
                a = min(q[c], q[4 + c]) - d
                b = max(q[c], q[4 + c]) + d
                if ir.slab_of(a, lo[c], w[c], v) == ir.slab_of(b, lo[c], w[c], v):
                    ok = True
            used += ok
        assert fmin <= used / len(Q) <= fmax, (v, used / len(Q))


def test_merger_shape():
    w = synth.merger()
    assert w.D.shape == (25_165_824, 8)               # P:1210-1213, Table 1
    assert w.Q.shape == (50_880, 8)                   # S2
    assert np.all(ir.admissible_v(w.D) >= 16)         # v = 16 used in S2
    assert np.all(w.D[:, 7] - w.D[:, 3] == 1.0)

"""Pins for the oracle's all-pairs search (oracle_search).

The search must equal an independent pure-Python brute force that finds each
pair's minimum distance and interval by dense sampling + bisection of the two
segments' positions (no closed form), on inputs small enough for that loop.
"""
import numpy as np
import pytest

import oracle
import synth
from test_oracle_compare import _sampled


def _small(seed, nd=40, nq=25):
    rng = np.random.default_rng(seed)

    def segs(n):
        t0 = rng.uniform(0, 4, n)
        t1 = t0 + rng.uniform(0.3, 2.0, n)
        p0 = rng.uniform(-2, 2, (n, 3))
        p1 = p0 + rng.uniform(-1.5, 1.5, (n, 3))
        return np.concatenate([p0, t0[:, None], p1, t1[:, None]], axis=1).astype(np.float32)
    return segs(nd), segs(nq)


@pytest.mark.parametrize("seed", [1, 2])
def test_search_equals_sampled_brute_force(seed):
    D, Q = _small(seed)
    d = 1.2
    res = oracle.search(D, Q, d)
    got = {(int(q), int(e)): (ti, to) for q, e, ti, to, h in
           zip(res["qid"], res["eid"], res["t_in"], res["t_out"], res["hit"]) if h}
    band = set()
    want = {}
    for k in range(Q.shape[0]):
        for i in range(D.shape[0]):
            iv, dm = _sampled(Q[k].astype(np.float64), D[i].astype(np.float64), d, n=2001)
            if abs(dm - d) <= 1e-6:
                band.add((k, i))
                continue
            if iv is not None:
                want[(k, i)] = iv
    assert len(want) > 15
    assert set(got) - band == set(want)
    for key, (ti, to) in want.items():
        assert got[key][0] == pytest.approx(ti, abs=1e-7)
        assert got[key][1] == pytest.approx(to, abs=1e-7)


def test_search_order_near_misses_and_subset():
    w = synth.tiny()
    r = oracle.search(w.D, w.Q, w.d, near=1.05)
    key = r["qid"] * (1 << 32) + r["eid"]
    assert np.all(np.diff(key) > 0)                      # sorted by (qid, eid), unique
    assert np.all(r["dmin"][r["hit"]] <= w.d)
    miss = ~r["hit"]
    assert np.all((r["dmin"][miss] > w.d) & (r["dmin"][miss] <= 1.05 * w.d))
    assert np.all(r["t_in"][r["hit"]] <= r["t_out"][r["hit"]])
    # every query's own trajectory... tiny Q is separate from D: hits are 1-20% of overlapping pairs
    t0q, t1q = w.Q[:, 3][:, None], w.Q[:, 7][:, None]
    overl = ((np.maximum(t0q, w.D[:, 3][None]) < np.minimum(t1q, w.D[:, 7][None]))).sum()
    frac = r["hit"].sum() / overl
    assert 0.01 <= frac <= 0.20
    sel = np.array([3, 17, 42, 99])
    s = oracle.search(w.D, w.Q, w.d, near=1.05, qsel=sel)
    m = np.isin(r["qid"], sel)
    for k in ("qid", "eid", "t_in", "t_out", "dmin", "hit"):
        assert np.array_equal(s[k], r[k][m])


def test_window_restricts_interval():
    w = synth.tiny()
    full = oracle.search(w.D, w.Q, w.d)
    T0, T1 = 8.0, 12.0
    win = oracle.search(w.D, w.Q, w.d, window=(T0, T1))
    h = win["hit"]
    assert np.all(win["t_in"][h] >= T0) and np.all(win["t_out"][h] <= T1)
    fk = set(zip(full["qid"][full["hit"]].tolist(), full["eid"][full["hit"]].tolist()))
    wk = set(zip(win["qid"][h].tolist(), win["eid"][h].tolist()))
    assert wk <= fk and len(wk) < len(fk)


def test_self_join_contains_self_pairs():
    # Q subset of D (reading C10): every query hits its own segment over its full span
    w = synth.random_walk(20, 11, 5, t_window=3.0, box=20.0, step_max=0.5)[0]
    r = oracle.search(w, w[::7], 0.01)
    selfp = {(k, 7 * k) for k in range(w[::7].shape[0])}
    got = {(int(a), int(b)): (ti, to) for a, b, ti, to, h in
           zip(r["qid"], r["eid"], r["t_in"], r["t_out"], r["hit"]) if h}
    assert selfp <= set(got)
    for k, e in selfp:
        assert got[(k, e)] == (float(w[e, 3]), float(w[e, 7]))

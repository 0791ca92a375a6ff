"""Pins for the oracle's pair test (oracle_compare), independent of its own formula.

* hand-worked cases E1-E10 / W1-W3 (tests/golden/compare_cases.txt, each with
  its derivation and citation);
* dense time sampling + bisection on random pairs: the minimum distance and
  the interval endpoints found WITHOUT the closed form (sampling the two
  segments' positions independently, PAPER.md P:102-104 linear motion);
* invariants: swap symmetry, monotonicity in d.
"""
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "compare_cases.txt")


def _num(s):
    return float(eval(s, {"__builtins__": {}}, {"sqrt": math.sqrt, "inf": math.inf}))


def _cases():
    out = []
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f = [x.strip() for x in line.split("|", 7)]
        name, q, e, d, win, exp, dmin, src = f
        q = [_num(x) for x in q.split()]
        e = [_num(x) for x in e.split()]
        T0, T1 = [_num(x) for x in win.split()]
        exp = None if exp == "none" else tuple(_num(x) for x in exp.split())
        out.append((name.split()[0], q, e, _num(d), (T0, T1), exp, _num(dmin)))
    return out


CASES = _cases()


def test_golden_file_has_all_cases():
    names = {c[0] for c in CASES}
    for n in ["E1a", "E2a", "E2b", "E3a", "E3b", "E4", "E5", "E6a", "E6b", "E7", "E8", "E9", "E10"]:
        assert n in names


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_hand_worked(case):
    name, q, e, d, win, exp, dmin = case
    for a, b in ((q, e), (e, q)):                      # symmetric in the two roles
        hit, ti, to, dm = oracle.compare(a, b, d, win)
        if exp is None:
            assert not hit
        else:
            assert hit
            assert ti == pytest.approx(exp[0], abs=1e-12)
            assert to == pytest.approx(exp[1], abs=1e-12)
        if math.isinf(dmin):
            assert math.isinf(dm)
        else:
            assert dm == pytest.approx(dmin, abs=1e-12)


# ---------------------------------------------------------------------------
# independent check: dense sampling + bisection
# ---------------------------------------------------------------------------
def _pos(seg, t):
    seg = np.asarray(seg, np.float64)
    f = (t - seg[3]) / (seg[7] - seg[3])
    return seg[None, 0:3] + f[:, None] * (seg[None, 4:7] - seg[None, 0:3])


def _dist(q, e, t):
    return np.linalg.norm(_pos(q, t) - _pos(e, t), axis=1)


def _sampled(q, e, d, n=100001):
    a = max(q[3], e[3])
    b = min(q[7], e[7])
    if not a < b:
        return None, math.inf
    t = np.linspace(a, b, n)
    g = _dist(q, e, t)
    k = int(np.argmin(g))
    # refine the minimum by golden-section search in the bracketing cells
    lo, hi = t[max(k - 1, 0)], t[min(k + 1, n - 1)]
    for _ in range(200):
        m1, m2 = lo + (hi - lo) * 0.382, lo + (hi - lo) * 0.618
        if _dist(q, e, np.array([m1]))[0] <= _dist(q, e, np.array([m2]))[0]:
            hi = m2
        else:
            lo = m1
    tm = 0.5 * (lo + hi)
    dmin = min(g.min(), _dist(q, e, np.array([tm]))[0])
    if dmin > d:
        return None, dmin

    def f(x):
        return _dist(q, e, np.array([x]))[0] - d

    def bisect(x_in, x_out):              # f(x_in) <= 0 < f(x_out)
        for _ in range(200):
            mid = 0.5 * (x_in + x_out)
            if f(mid) <= 0:
                x_in = mid
            else:
                x_out = mid
        return x_in

    t_in = a if f(a) <= 0 else bisect(tm, a)
    t_out = b if f(b) <= 0 else bisect(tm, b)
    return (t_in, t_out), dmin


def _random_pairs(rng, n):
    pairs = []
    for k in range(n):
        kind = k % 4
        t0q = rng.uniform(0, 5)
        t1q = t0q + rng.uniform(0.2, 3)
        t0e = rng.uniform(t0q - 2, t1q - 0.1)
        t1e = max(t0e + rng.uniform(0.2, 3), t0q + 0.05)
        p0q = rng.uniform(-3, 3, 3)
        p1q = p0q + rng.uniform(-3, 3, 3)
        p0e = rng.uniform(-3, 3, 3)
        p1e = p0e + rng.uniform(-3, 3, 3)
        if kind == 1:                      # near parallel motion
            p1e = p0e + (p1q - p0q) * (t1e - t0e) / (t1q - t0q) + rng.normal(0, 1e-3, 3)
        if kind == 2:                      # stationary query (P:86-88 case (i))
            p1q = p0q.copy()
        q = np.array([*p0q, t0q, *p1q, t1q], np.float32)
        e = np.array([*p0e, t0e, *p1e, t1e], np.float32)
        pairs.append((q.astype(np.float64), e.astype(np.float64)))
    return pairs


def test_closed_form_matches_sampling():
    rng = np.random.default_rng(1410)
    n_hit = 0
    for q, e in _random_pairs(rng, 400):
        d = float(rng.uniform(0.3, 4.0))
        hit, ti, to, dm = oracle.compare(q, e, d)
        iv, dm_s = _sampled(q, e, d)
        assert dm == pytest.approx(dm_s, abs=1e-7)
        if abs(dm_s - d) <= 1e-6:          # too close to call for the sampler
            continue
        assert hit == (iv is not None)
        if hit:
            n_hit += 1
            span = min(q[7], e[7]) - max(q[3], e[3])
            assert abs(ti - iv[0]) <= 1e-7 * max(1.0, span)
            assert abs(to - iv[1]) <= 1e-7 * max(1.0, span)
            # boundary residual: |Delta(t)| = d at endpoints that are not span ends
            a, b = max(q[3], e[3]), min(q[7], e[7])
            for t in (ti, to):
                if a + 1e-9 < t < b - 1e-9:
                    assert _dist(q, e, np.array([t]))[0] == pytest.approx(d, abs=1e-9)
    assert n_hit > 50


def test_symmetry_and_monotone_in_d():
    rng = np.random.default_rng(7)
    for q, e in _random_pairs(rng, 300):
        ds = sorted(rng.uniform(0.1, 5.0, 4))
        prev = None
        for d in ds:
            r1 = oracle.compare(q, e, d)
            r2 = oracle.compare(e, q, d)
            assert r1[0] == r2[0]
            if r1[0]:
                assert r1[1] == pytest.approx(r2[1], abs=1e-12)
                assert r1[2] == pytest.approx(r2[2], abs=1e-12)
                assert r1[1] <= r1[2]
                if prev is not None and prev[0]:
                    assert r1[1] <= prev[1] + 1e-12 and r1[2] >= prev[2] - 1e-12
            else:
                assert prev is None or not prev[0]
            prev = r1


def test_stationary_pair_is_constant_distance():
    # both segments stationary: distance constant = |p - p'| (A = 0 path)
    q = [1, 2, 3, 0, 1, 2, 3, 4]
    e = [1, 2, 5, 1, 1, 2, 5, 6]
    assert oracle.compare(q, e, 2.0)[:3] == (True, 1.0, 4.0)
    assert oracle.compare(q, e, 1.999)[0] is False

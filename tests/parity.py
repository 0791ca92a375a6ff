"""Parity helpers: compare a CUDA-path result set with the oracle's.

The bar (BASELINE.json north_star):
* the (query, entry) pair set is bit-exact, except pairs whose oracle minimum
  distance lies within 1e-5*d of d (the exclusion band, logged and excluded);
* interval endpoints agree within 1e-5 * (b - a) + ulp32(|t_ref|) (reading C24:
  1e-5 relative to the shared span, plus the spacing of the fp32 output at t);
* no duplicate pairs.
"""
from __future__ import annotations

import numpy as np

BAND = 1e-5
TOL = 1e-5


def ulp32(t):
    """Spacing of float32 at |t| (the resolution of an fp32 output time)."""
    t = np.abs(np.asarray(t, np.float64)).astype(np.float32)
    return (np.nextafter(t, np.float32(np.inf)) - t).astype(np.float64)


def stratified(Q, n, seed=0):
    """a deterministic query subsample of size n stratified over
    time: Q rows in t_start order, one random row from each of n equal strata."""
    order = np.argsort(Q[:, 3], kind="stable")
    n = min(n, order.size)
    edges = np.linspace(0, order.size, n + 1).astype(np.int64)
    rng = np.random.default_rng(seed)
    pick = edges[:-1] + (rng.random(n) * (edges[1:] - edges[:-1])).astype(np.int64)
    return np.sort(order[pick])


def keys(q, e):
    return np.asarray(q, np.int64) * (1 << 32) + np.asarray(e, np.int64)


def check(got, ref, D, Q, d, window=(-np.inf, np.inf), label=""):
    """got = (qid, eid, t_in, t_out) numpy; ref = oracle.search(...) dict.
    Returns a small report dict; raises AssertionError on a mismatch."""
    gq, ge, gi, go = (np.asarray(x) for x in got)
    gk = keys(gq, ge)
    order_g = np.argsort(gk, kind="stable")
    gk_s = gk[order_g]
    assert not (gk_s[1:] == gk_s[:-1]).any(), f"{label}: duplicate pairs in GPU result"
    band = np.abs(ref["dmin"] - d) <= BAND * d
    rk = keys(ref["qid"], ref["eid"])
    excl = np.sort(rk[band])
    want_mask = ref["hit"] & ~band
    want = rk[want_mask]
    want_s = np.sort(want)
    # GPU pairs outside the exclusion band must be exactly the oracle's hits
    in_excl = np.isin(gk_s, excl, assume_unique=False)
    g_eff = gk_s[~in_excl]
    missing = np.setdiff1d(want_s, g_eff, assume_unique=True)
    extra = np.setdiff1d(g_eff, want_s, assume_unique=True)
    assert missing.size == 0 and extra.size == 0, (
        f"{label}: {missing.size} missing, {extra.size} extra "
        f"(e.g. missing {[divmod(int(k), 1 << 32) for k in missing[:5]]}, "
        f"extra {[divmod(int(k), 1 << 32) for k in extra[:5]]})")
    # endpoints
    pos = np.searchsorted(gk_s, want)
    ti_g = gi[order_g][pos].astype(np.float64)
    to_g = go[order_g][pos].astype(np.float64)
    qi = ref["qid"][want_mask]
    ei = ref["eid"][want_mask]
    a = np.maximum(np.maximum(Q[qi, 3], D[ei, 3]).astype(np.float64), window[0])
    b = np.minimum(np.minimum(Q[qi, 7], D[ei, 7]).astype(np.float64), window[1])
    ti_r, to_r = ref["t_in"][want_mask], ref["t_out"][want_mask]
    tol_i = TOL * (b - a) + ulp32(ti_r)
    tol_o = TOL * (b - a) + ulp32(to_r)
    err_i = np.abs(ti_g - ti_r)
    err_o = np.abs(to_g - to_r)
    bad = (err_i > tol_i) | (err_o > tol_o)
    assert not bad.any(), (f"{label}: {int(bad.sum())} endpoints out of tolerance, worst "
                           f"{float(max(err_i.max(initial=0), err_o.max(initial=0)))}")
    span = np.maximum(b - a, 1e-30)
    rel = float(max(((err_i - ulp32(ti_r)).clip(0) / span).max(initial=0),
                    ((err_o - ulp32(to_r)).clip(0) / span).max(initial=0)))
    assert rel <= TOL, rel
    return {"pairs": int(want.size), "band": int(band.sum()), "max_err_rel_span": rel,
            "max_err_abs": float(max(err_i.max(initial=0), err_o.max(initial=0)))}

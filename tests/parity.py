"""Parity helpers: compare a CUDA-path result set with the oracle's.

The bar (BASELINE.json north_star):
* the (query, entry) pair set is bit-exact, except pairs whose oracle minimum
  distance lies within 1e-5*d of d (the exclusion band, logged and excluded);
* interval endpoints agree within 1e-5 * max(|t_ref|, b - a) (reading C24);
* no duplicate pairs.
"""
from __future__ import annotations

import numpy as np

BAND = 1e-5
TOL = 1e-5


def keys(q, e):
    return np.asarray(q, np.int64) * (1 << 32) + np.asarray(e, np.int64)


def check(got, ref, D, Q, d, window=(-np.inf, np.inf), label=""):
    """got = (qid, eid, t_in, t_out) numpy; ref = oracle.search(...) dict.
    Returns a small report dict; raises AssertionError on a mismatch."""
    gq, ge, gi, go = (np.asarray(x) for x in got)
    gk = keys(gq, ge)
    assert np.unique(gk).size == gk.size, f"{label}: duplicate pairs in GPU result"
    band = np.abs(ref["dmin"] - d) <= BAND * d
    rk = keys(ref["qid"], ref["eid"])
    excl = set(rk[band].tolist())
    want_mask = ref["hit"] & ~band
    want = rk[want_mask]
    gset = set(gk.tolist()) - excl
    wset = set(want.tolist())
    missing = wset - gset
    extra = gset - wset
    assert not missing and not extra, (
        f"{label}: {len(missing)} missing, {len(extra)} extra "
        f"(e.g. missing {[divmod(k, 1 << 32) for k in list(missing)[:5]]}, "
        f"extra {[divmod(k, 1 << 32) for k in list(extra)[:5]]})")
    # endpoints
    order_g = np.argsort(gk)
    gk_s = gk[order_g]
    pos = np.searchsorted(gk_s, want)
    ti_g = gi[order_g][pos].astype(np.float64)
    to_g = go[order_g][pos].astype(np.float64)
    qi = ref["qid"][want_mask]
    ei = ref["eid"][want_mask]
    a = np.maximum(np.maximum(Q[qi, 3], D[ei, 3]).astype(np.float64), window[0])
    b = np.minimum(np.minimum(Q[qi, 7], D[ei, 7]).astype(np.float64), window[1])
    ti_r, to_r = ref["t_in"][want_mask], ref["t_out"][want_mask]
    tol_i = TOL * np.maximum(np.abs(ti_r), b - a)
    tol_o = TOL * np.maximum(np.abs(to_r), b - a)
    err_i = np.abs(ti_g - ti_r)
    err_o = np.abs(to_g - to_r)
    bad = (err_i > tol_i) | (err_o > tol_o)
    assert not bad.any(), (f"{label}: {int(bad.sum())} endpoints out of tolerance, worst "
                           f"{float(max(err_i.max(initial=0), err_o.max(initial=0)))}")
    span = np.maximum(b - a, 1e-30)
    return {"pairs": len(wset), "band": int(band.sum()),
            "max_err_rel_span": float(max((err_i / span).max(initial=0), (err_o / span).max(initial=0)))}

"""CPU oracle for the distance threshold search (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The CUDA
path (``paper_1410_2698_b200``) never imports it, and it never imports the
CUDA path: the two share only the seeded input generators in ``synth``.

* ``compare``  / ``search`` — fp64 all-pairs brute force in plain C
  (``tds_oracle.c``), the plain definition of the result set (§3.1
  P:186-203).
* ``index_ref`` — the paper's index structures (temporal bins, spatiotemporal
  subbin arrays, flatly structured grid) written out step by step in numpy,
  used to pin the GPU index builds against the paper's worked figures.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tds_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2 -fopenmp); returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.c_void_p
        lib.oracle_compare.argtypes = [fp, fp, ctypes.c_double, ctypes.c_double, ctypes.c_double, dp, dp, dp]
        lib.oracle_compare.restype = ctypes.c_int
        lib.oracle_search.argtypes = [fp, ctypes.c_int64, fp, ctypes.c_int64, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int]
        lib.oracle_search.restype = ctypes.c_int64
        lib.oracle_search_subset.argtypes = [fp, ctypes.c_int64, fp, fp, ctypes.c_int64, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int]
        lib.oracle_search_subset.restype = ctypes.c_int64
        lib.oracle_fetch.argtypes = [fp] * 6
        lib.oracle_fetch.restype = None
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _seg(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32).reshape(-1, 8))
    return a


def compare(q, e, d: float, window=(-np.inf, np.inf)):
    """Interaction of query segment q with entry segment e (8 floats each).

    Returns (hit, t_in, t_out, dmin); dmin = inf when the spans do not overlap.
    """
    lib = _load()
    qa, ea = _seg(q), _seg(e)
    ti, to, dm = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    hit = lib.oracle_compare(qa.ctypes.data, ea.ctypes.data, float(d), float(window[0]), float(window[1]),
                             ctypes.byref(ti), ctypes.byref(to), ctypes.byref(dm))
    return bool(hit), ti.value, to.value, dm.value


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def search(D, Q, d: float, window=(-np.inf, np.inf), near: float = 1.01, nthreads: int = 0,
           qsel=None) -> dict:
    """All-pairs brute force.  Returns a dict of numpy arrays ordered by (qid, eid):

    qid, eid (int64 row numbers in Q and D), t_in, t_out, dmin (float64),
    hit (bool).  Rows with hit=False are near misses (dmin <= near*d) kept for
    the parity exclusion band.  ``qsel`` restricts the search to those Q rows
    (record qid is still the original row number).
    """
    lib = _load()
    Da, Qa = _seg(D), _seg(Q)
    if qsel is None:
        n = lib.oracle_search(Da.ctypes.data, Da.shape[0], Qa.ctypes.data, Qa.shape[0], float(d),
                              float(window[0]), float(window[1]), float(near), int(nthreads))
    else:
        qs = np.ascontiguousarray(np.asarray(qsel, dtype=np.int64))
        n = lib.oracle_search_subset(Da.ctypes.data, Da.shape[0], Qa.ctypes.data, qs.ctypes.data,
                                     qs.shape[0], float(d), float(window[0]), float(window[1]),
                                     float(near), int(nthreads))
    out = {
        "qid": np.empty(n, np.int64), "eid": np.empty(n, np.int64),
        "t_in": np.empty(n, np.float64), "t_out": np.empty(n, np.float64),
        "dmin": np.empty(n, np.float64), "hit": np.empty(n, np.int32),
    }
    lib.oracle_fetch(*(out[k].ctypes.data for k in ("qid", "eid", "t_in", "t_out", "dmin", "hit")))
    out["hit"] = out["hit"].astype(bool)
    return out


def merge_trajectories(qid, eid, t_in, t_out, q_traj, e_traj, gap: float = 0.0) -> dict:
    """Trajectory-level answer ("find all trajectories within d",
    P:86-90 "and corresponding time periods"): for every pair
    (query trajectory, entry trajectory), the union of the closed intervals of
    its segment-pair records, as maximal disjoint intervals.  Two intervals
    merge when the next starts no later than ``gap`` after the current one
    ends (gap = 0: overlapping or touching).  Plain definition: sort by
    (q_traj, e_traj, t_in) and sweep.  Returns dict qtraj, etraj, t_in, t_out
    (ordered by qtraj, etraj, t_in)."""
    qt = np.asarray(q_traj)[np.asarray(qid, np.int64)]
    et = np.asarray(e_traj)[np.asarray(eid, np.int64)]
    ti = np.asarray(t_in, np.float64)
    to = np.asarray(t_out, np.float64)
    order = np.lexsort((ti, et, qt))
    out = {"qtraj": [], "etraj": [], "t_in": [], "t_out": []}
    cur = None
    for k in order:
        key = (int(qt[k]), int(et[k]))
        if cur is not None and cur[0] == key and ti[k] <= cur[2] + gap:
            cur[2] = max(cur[2], to[k])
            continue
        if cur is not None:
            for f, v in zip(("qtraj", "etraj", "t_in", "t_out"), (cur[0][0], cur[0][1], cur[1], cur[2])):
                out[f].append(v)
        cur = [key, ti[k], to[k]]
    if cur is not None:
        for f, v in zip(("qtraj", "etraj", "t_in", "t_out"), (cur[0][0], cur[0][1], cur[1], cur[2])):
            out[f].append(v)
    return {"qtraj": np.array(out["qtraj"], np.int64), "etraj": np.array(out["etraj"], np.int64),
            "t_in": np.array(out["t_in"], np.float64), "t_out": np.array(out["t_out"], np.float64)}

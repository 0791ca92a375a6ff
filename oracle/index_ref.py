"""The paper's three index structures, written out step by step (TEST INFRASTRUCTURE ONLY).

Plain numpy / Python, in the paper's order and notation, used to pin the GPU
index builds (exported through ``tds_index_export``) against the paper's
worked figures.  Shares no code with the CUDA path.

Readings of silent / garbled points are SURVEY §8c C12-C15 and DESIGN.md
"Readings":
* C12  bins are 0-based, ``j = clamp(floor((t_start - t_min) / b), 0, m-1)``.
* C15  spatial subbins ("slabs") per dimension are ``[o + j w, o + (j+1) w)``,
       the last one closed; an entry is placed in every slab its extent
       ``[min(c_start, c_end), max(c_start, c_end)]`` touches; the query MBB is
       inflated by the full d before the slab lookup.
* C14  FSG cells likewise; the query MBB is inflated by d.
* C20  where floating point decides an integer (a bin, slab or cell number),
       it is decided as the kernel decides it: fp32 round-to-nearest for the
       cell arithmetic, directed rounding for the d-inflated query box (the
       task's rule for integer decisions taken in floating point).
"""
from __future__ import annotations

import math

import numpy as np


# ---------------------------------------------------------------------------
# §4.2.1 GPUTemporal index (Fig. 3)
# ---------------------------------------------------------------------------
def temporal_sort(D: np.ndarray):
    """Sort D by ascending t_start and renumber.  Stable.

    Returns (D_sorted, perm) with D_sorted[i] = D[perm[i]].
    """
    perm = np.argsort(D[:, 3], kind="stable")
    return D[perm], perm


def morton30(cx, cy, cz) -> np.ndarray:
    """Morton (Z-order) code of 10-bit cell coordinates: bit k of x, y, z at bits
    3k + 2, 3k + 1, 3k."""
    cx, cy, cz = (np.asarray(c, np.int64) for c in (cx, cy, cz))
    code = np.zeros(np.broadcast(cx, cy, cz).shape, np.int64)
    for k in range(10):
        code |= ((cx >> k) & 1) << (3 * k + 2)
        code |= ((cy >> k) & 1) << (3 * k + 1)
        code |= ((cz >> k) & 1) << (3 * k)
    return code


def bin_of(D: np.ndarray, m: int) -> np.ndarray:
    """Temporal bin of every entry (C12): clamp(floor((t_start - t_min) / b), 0, m - 1),
    b = (t_max - t_min) / m, in fp64."""
    t0 = D[:, 3].astype(np.float64)
    t_min, t_max = t0.min(), D[:, 7].astype(np.float64).max()
    b = (t_max - t_min) / m
    if not b > 0:
        b = 1.0
    return np.clip(np.floor((t0 - t_min) / b), 0, m - 1).astype(np.int64)


def spatial_sort(D: np.ndarray, m: int):
    """The build's default renumbering (the paper's
    renumbering by t_start, is ``temporal_sort``): by temporal bin,
    then by the Morton code of the start point's cell on a 1024^3 grid over D's
    extent (cells decided in fp32, C29); stable, so ties keep the input order.
    Every bin holds the same entries as under ``temporal_sort``.
    Returns (D_sorted, perm) with D_sorted[i] = D[perm[i]]."""
    o, w = grid_geometry(D, (1024, 1024, 1024))
    cells = [np.array([slab_of(x, o[c], w[c], 1024) for x in D[:, c]]) for c in range(3)]
    key = morton30(*cells)
    perm = np.lexsort((np.arange(D.shape[0]), key, bin_of(D, m)))
    return D[perm], perm


def temporal_bins(D_sorted: np.ndarray, m: int):
    """Bins B_j = (B_j^start, B_j^end, B_j^first, B_j^last), j = 0..m-1.

    t_min = min t_start, t_max = max t_end, b = (t_max - t_min) / m;
    l_i in B_j iff floor((t_i^start - t_min) / b) = j (clamped, reading C12);
    B_j^start = t_min + j b;  B_j^end = max(t_min + (j+1) b, max_{l_i in B_j} t_i^end);
    B_j^first / B_j^last = first / last (renumbered) id in the bin; -1 if empty.
    Arithmetic in float64.  Returns dict of arrays and the per-entry bin ids.
    """
    t0 = D_sorted[:, 3].astype(np.float64)
    t1 = D_sorted[:, 7].astype(np.float64)
    t_min, t_max = t0.min(), t1.max()
    b = (t_max - t_min) / m
    j_of = np.clip(np.floor((t0 - t_min) / b), 0, m - 1).astype(np.int64)
    B_start = np.array([t_min + j * b for j in range(m)])
    B_end = np.empty(m)
    B_first = np.full(m, -1, np.int64)
    B_last = np.full(m, -1, np.int64)
    for j in range(m):
        members = np.nonzero(j_of == j)[0]
        end = t_min + (j + 1) * b
        if members.size:
            end = max(end, t1[members].max())
            B_first[j] = members.min()
            B_last[j] = members.max()
        B_end[j] = end
    return {"B_start": B_start, "B_end": B_end, "B_first": B_first, "B_last": B_last,
            "bin_of": j_of, "b": b, "t_min": t_min, "t_max": t_max}


def member_extent_bins(D_sorted: np.ndarray, bin_of: np.ndarray, m: int, t0q: float, t1q: float):
    """Bins a query (t0q, t1q) looks up under reading C13: the lookup uses the
    members' own extents, not the literal B^start / B^end (Fig. 3's B_0 ends at
    7.5 after B_1's 6.2, so B^end is not monotone).  Lower end: the
    first bin holding a member with t_end > t0q; upper end: the last bin holding
    a member with t_start < t1q (strict: segments that only touch do not
    interact, C5).  Returns (j_lo, j_hi) inclusive, or None when j_lo > j_hi.
    The candidate range is the hull of these bins."""
    t0 = D_sorted[:, 3].astype(np.float64)
    t1 = D_sorted[:, 7].astype(np.float64)
    j_lo = j_hi = None
    for j in range(m):
        members = np.nonzero(bin_of == j)[0]
        if members.size == 0:
            continue
        if j_lo is None and t1[members].max() > t0q:
            j_lo = j
        if t0[members].min() < t1q:
            j_hi = j
    if j_lo is None or j_hi is None or j_lo > j_hi:
        return None
    return j_lo, j_hi


def temporal_schedule(bins: dict, t0q: float, t1q: float):
    """E_k for one query: the bins whose extent [B^start, B^end]
    overlaps [t0q, t1q]; E_k = [min B^first, max B^last] over the non-empty ones.

    Returns (lo, hi) inclusive, or None if no non-empty bin overlaps.
    """
    lo, hi = None, None
    for j in range(len(bins["B_start"])):
        if bins["B_first"][j] < 0:
            continue
        if bins["B_start"][j] <= t1q and bins["B_end"][j] >= t0q:
            f, l_ = bins["B_first"][j], bins["B_last"][j]
            lo = f if lo is None else min(lo, f)
            hi = l_ if hi is None else max(hi, l_)
    return None if lo is None else (int(lo), int(hi))


# ---------------------------------------------------------------------------
# §4.3.1 GPUSpatioTemporal index (Fig. 4)
# ---------------------------------------------------------------------------
def spatial_extent(D: np.ndarray):
    """[c_min, c_max] over both endpoints and the maximum per-segment extent
    max |c_start - c_end| per dimension.  float64."""
    lo = np.minimum(D[:, 0:3], D[:, 4:7]).astype(np.float64).min(axis=0)
    hi = np.maximum(D[:, 0:3], D[:, 4:7]).astype(np.float64).max(axis=0)
    mx = np.abs(D[:, 0:3].astype(np.float64) - D[:, 4:7].astype(np.float64)).max(axis=0)
    return lo, hi, mx


def f32_sub_rd(a: float, b: float) -> np.float32:
    """a - b rounded toward -inf to float32 (a, b float32 values)."""
    x = float(np.float64(a) - np.float64(b))
    r = np.float32(x)
    return np.nextafter(r, np.float32(-np.inf)) if float(r) > x else r


def f32_add_ru(a: float, b: float) -> np.float32:
    """a + b rounded toward +inf to float32."""
    x = float(np.float64(a) + np.float64(b))
    r = np.float32(x)
    return np.nextafter(r, np.float32(np.inf)) if float(r) < x else r


def d_up32(d: float) -> np.float32:
    """The threshold as the fp32 stages use it: d rounded up to float32 (C25)."""
    r = np.float32(d)
    return np.nextafter(r, np.float32(np.inf)) if float(r) < d else r


def grid_geometry(D: np.ndarray, cells):
    """Origin and cell width per dimension of a grid of ``cells[c]`` equal cells
    over D's spatial extent (C14, C15): o = c_min, w = (c_max - c_min) / cells,
    in fp32 as the kernel computes them (w = 1 for a zero extent)."""
    lo, hi, _ = spatial_extent(D)
    o = np.array([np.float32(x) for x in lo], np.float32)
    w = np.empty(3, np.float32)
    for c in range(3):
        ext = np.float32(np.float32(hi[c]) - np.float32(lo[c]))
        w[c] = np.float32(ext / np.float32(cells[c])) if ext > 0 else np.float32(1.0)
    return o, w


def admissible_v(D: np.ndarray) -> np.ndarray:
    """Largest v per dimension with v <= (c_max - c_min) / max |c_start - c_end|."""
    lo, hi, mx = spatial_extent(D)
    with np.errstate(divide="ignore"):
        r = np.where(mx > 0, (hi - lo) / np.where(mx > 0, mx, 1.0), np.inf)
    return np.floor(r)


def slab_of(c: float, o: float, w: float, v: int) -> int:
    """Slab j of coordinate c: [o + j w, o + (j+1) w), last slab closed (C15);
    j = floor((c - o) / w) decided in fp32 (C20)."""
    q = np.float32(np.float32(np.float32(c) - np.float32(o)) / np.float32(w))
    return int(min(max(math.floor(q), 0), v - 1))


def query_slabs(q: np.ndarray, d: float, o, w, v: int):
    """Slabs [slab_lo[c], slab_hi[c]] of a query's MBB inflated by the full d in
    every dimension (C15; the expansion is silent in P:1036-1050), the box's
    ends rounded outward (C20)."""
    dd = d_up32(d)
    lo, hi = [], []
    for c in range(3):
        a, b = np.float32(min(q[c], q[4 + c])), np.float32(max(q[c], q[4 + c]))
        lo.append(slab_of(f32_sub_rd(a, dd), o[c], w[c], v))
        hi.append(slab_of(f32_add_ru(b, dd), o[c], w[c], v))
    return lo, hi


def st_arrays(D_sorted: np.ndarray, bin_of: np.ndarray, m: int, v: int, origin, width):
    """Arrays X, Y, Z: per dimension, the ids of the entries that
    overlap each subbin B̂_{i,j} (temporal bin i, slab j), stored contiguously
    with the subbins in (j, i) lexicographic order; ids ascending inside a
    subbin.  Also the subbin descriptors: for each (i, j) and each
    dimension the inclusive index range [first, last] (None if empty).

    Returns (arrays[3], ranges[3]) where ranges[c][(i, j)] = (first, last) or None.
    """
    arrays, ranges = [], []
    for c in range(3):
        w = float(width[c])
        o = float(origin[c])
        members = {(i, j): [] for i in range(m) for j in range(v)}
        for e in range(D_sorted.shape[0]):
            a, bb = float(D_sorted[e, c]), float(D_sorted[e, 4 + c])
            s_lo, s_hi = slab_of(min(a, bb), o, w, v), slab_of(max(a, bb), o, w, v)
            for j in range(s_lo, s_hi + 1):
                members[(int(bin_of[e]), j)].append(e)
        arr, rng = [], {}
        for j in range(v):
            for i in range(m):
                ids = sorted(members[(i, j)])
                rng[(i, j)] = (len(arr), len(arr) + len(ids) - 1) if ids else None
                arr.extend(ids)
        arrays.append(np.array(arr, dtype=np.int64))
        ranges.append(rng)
    return arrays, ranges


def plan(D: np.ndarray, Q: np.ndarray, d: float, m: int, v: int, kind: str = "spatiotemporal",
         window=(-np.inf, np.inf), order: str = "time"):
    """The schedule entry of every query in the layout
    of tds_plan: (sel, lo, hi) with sel = -1 for the temporal range [lo, hi) of
    sorted entries (GPUTemporal, or the GPUSpatioTemporal fallback), 0/1/2 for
    the range [lo, hi) of X/Y/Z, 3 for no candidates (lo = hi = 0).  Queries
    are clipped to the window and need t0 < t1 after clipping (C5, C8)."""
    Ds, _ = temporal_sort(D) if order == "time" else spatial_sort(D, m)
    b = temporal_bins(Ds, m)
    bin_of = b["bin_of"]
    off = np.searchsorted(bin_of, np.arange(m + 1), side="left")        # bin j = sorted ids [off[j], off[j+1])
    if kind == "spatiotemporal":
        o, w = grid_geometry(D, (v, v, v))
        _, ranges = st_arrays(Ds, bin_of, m, v, o, w)
    out = []
    for k in range(Q.shape[0]):
        t0c = max(float(Q[k, 3]), float(np.float32(window[0])))      # the window is float32 (tds.h)
        t1c = min(float(Q[k, 7]), float(np.float32(window[1])))
        if not t0c < t1c:
            out.append((3, 0, 0))
            continue
        jj = member_extent_bins(Ds, bin_of, m, t0c, t1c)
        if jj is None:
            out.append((3, 0, 0))
            continue
        entry = (-1, int(off[jj[0]]), int(off[jj[1] + 1]))
        if entry[1] >= entry[2]:
            out.append((3, 0, 0))
            continue
        if kind == "spatiotemporal":
            sl, sh = query_slabs(Q[k], d, o, w, v)
            sel, first, last = st_select(ranges, jj[0], jj[1], sl, sh)
            if sel >= 0:
                entry = (sel, first, last + 1) if last >= first else (3, 0, 0)
        out.append(entry)
    return np.array(out, np.int64).reshape(-1, 3)


def st_select(ranges, bins_lo: int, bins_hi: int, slab_lo, slab_hi):
    """Schedule entry of one query.

    ``bins_lo..bins_hi``: the temporal bins the query overlaps; ``slab_lo[c]``,
    ``slab_hi[c]``: the slabs its (d-inflated) MBB overlaps in dimension c.
    A dimension is usable only if the query lies in a single slab there
    (otherwise duplicates would occur); among usable dimensions pick the one
    with the fewest entries, ties to the lowest dimension (x < y < z).
    Returns (sel, first, last): sel in {0,1,2} with an inclusive range into
    X/Y/Z (first > last = empty), or (-1, None, None) for the temporal fallback.
    """
    best = None
    for c in range(3):
        if slab_lo[c] != slab_hi[c]:
            continue
        j = slab_lo[c]
        parts = [ranges[c][(i, j)] for i in range(bins_lo, bins_hi + 1)]
        nonempty = [p for p in parts if p is not None]
        count = sum(p[1] - p[0] + 1 for p in nonempty)
        if nonempty:
            first, last = nonempty[0][0], nonempty[-1][1]
            assert last - first + 1 == count, "subbins of one slab must be contiguous"
        else:
            first, last = 0, -1
        if best is None or count < best[0]:
            best = (count, c, first, last)
    if best is None:
        return (-1, None, None)
    return (best[1], best[2], best[3])


# ---------------------------------------------------------------------------
# §4.1 GPUSpatial flatly structured grid (Fig. 1-2, Alg. 1)
# ---------------------------------------------------------------------------
def linearize(cx: int, cy: int, cz: int, grid) -> int:
    """Row-major linearised cell coordinate h."""
    return (cx * grid[1] + cy) * grid[2] + cz


def cell_range(lo: float, hi: float, o: float, w: float, g: int):
    """Cells [floor((lo-o)/w), floor((hi-o)/w)] clamped to [0, g-1] (decided in fp32, C20)."""
    return slab_of(lo, o, w, g), slab_of(hi, o, w, g)


def rasterize(mbb_min, mbb_max, origin, width, grid):
    """All cells (cx, cy, cz) overlapped by an MBB (Fig. 1)."""
    rs = [cell_range(mbb_min[c], mbb_max[c], origin[c], width[c], grid[c]) for c in range(3)]
    return [(x, y, z) for x in range(rs[0][0], rs[0][1] + 1)
            for y in range(rs[1][0], rs[1][1] + 1)
            for z in range(rs[2][0], rs[2][1] + 1)]


def fsg_build(D: np.ndarray, grid, origin, width):
    """G (non-empty cells (h, A_min, A_max) sorted by h) and lookup array A
    (P:296-299).  Entry ids inside a cell by (t_start, id), the order
    the per-cell time trimming needs (ascending id when D is sorted by t_start)."""
    cells = {}
    for e in range(D.shape[0]):
        mn = np.minimum(D[e, 0:3], D[e, 4:7]).astype(np.float64)
        mx = np.maximum(D[e, 0:3], D[e, 4:7]).astype(np.float64)
        for (x, y, z) in rasterize(mn, mx, origin, width, grid):
            cells.setdefault(linearize(x, y, z, grid), []).append(e)
    G, A = [], []
    for h in sorted(cells):
        ids = sorted(cells[h], key=lambda e: (float(D[e, 3]), e))
        G.append((h, len(A), len(A) + len(ids) - 1))
        A.extend(ids)
    return np.array(G, dtype=np.int64).reshape(-1, 3), np.array(A, dtype=np.int64)


def fsg_candidates(G: np.ndarray, A: np.ndarray, hs):
    """getCandidates: for each overlapped cell h, binary-search G
    for h and append A[A_h^min : A_h^max] to the candidate buffer, keeping
    duplicates."""
    keys = G[:, 0]
    U = []
    for h in hs:
        k = int(np.searchsorted(keys, h))
        if k < len(keys) and keys[k] == h:
            U.extend(A[G[k, 1]:G[k, 2] + 1].tolist())
    return U

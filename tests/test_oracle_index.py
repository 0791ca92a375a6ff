"""Pins for oracle/index_ref.py against the paper's worked figures.

Fig. 3 temporal bins (exact), Fig. 4 X array and descriptors (exact), Y/Z
corrected by hand (golden file documents the derivation), the dimension
selection example of P:1054-1071, Fig. 1 rasterisation and Fig. 2 lookup.
"""
import os

import numpy as np

from oracle import index_ref as ir

G = os.path.join(os.path.dirname(__file__), "golden")


def _rows(fname, tag):
    out = []
    for line in open(os.path.join(G, fname)):
        f = line.split()
        if f and f[0] == tag:
            out.append(f[1:])
    return out


def fig3_segments():
    rows = _rows("fig3_temporal_bins.txt", "seg")
    D = np.zeros((len(rows), 8), np.float32)
    for r in rows:
        i = int(r[0])
        D[i, 3], D[i, 7] = float(r[1]), float(r[2])
    return D


def test_fig3_bins():
    D = fig3_segments()
    Ds, perm = ir.temporal_sort(D)
    assert np.array_equal(perm, np.arange(15))          # already in t_start order
    b = ir.temporal_bins(Ds, 4)
    assert b["b"] == 3.0
    for r in _rows("fig3_temporal_bins.txt", "bin"):
        j = int(r[0])
        assert b["B_start"][j] == float(r[1])
        assert abs(b["B_end"][j] - float(r[2])) < 1e-6
        assert b["B_first"][j] == int(r[3]) and b["B_last"][j] == int(r[4])
    # text P:671-674: B_2 = {l9, l10, l11}, B_2^start = 2 x (12/4) = 6, B_2^end = t_11^end
    assert list(np.nonzero(b["bin_of"] == 2)[0]) == [9, 10, 11]
    assert abs(b["B_end"][2] - D[11, 7]) < 1e-6


def test_fig3_schedule():
    b = ir.temporal_bins(ir.temporal_sort(fig3_segments())[0], 4)
    # query [5.0, 5.5] overlaps B0 [0,7.5] and B1 [3,6.2] only -> E = [0, 8]
    assert ir.temporal_schedule(b, 5.0, 5.5) == (0, 8)
    # query [11.95, 12.5]: B2 ends at 11 -> only B3 -> [12, 14]
    assert ir.temporal_schedule(b, 11.95, 12.5) == (12, 14)
    # query [6.5, 6.9]: B0 (to 7.5) and B2 ([6,11]); B1 ends at 6.2 -> hull [0, 11]
    assert ir.temporal_schedule(b, 6.5, 6.9) == (0, 11)


def fig4():
    rows = _rows("fig4_spatiotemporal.txt", "entry")
    D = np.zeros((len(rows), 8), np.float32)
    binof = np.zeros(len(rows), np.int64)
    for r in rows:
        i = int(r[0])
        D[i, 0:3] = [float(x) for x in r[1:4]]
        D[i, 4:7] = [float(x) for x in r[4:7]]
        D[i, 3], D[i, 7] = float(i), float(i) + 1.0
        binof[i] = int(r[7])
    return D, binof


def test_fig4_arrays():
    D, binof = fig4()
    arrays, ranges = ir.st_arrays(D, binof, 3, 3, (0, 0, 0), (4, 4, 5))
    want = {k: [int(x) for x in _rows("fig4_spatiotemporal.txt", k)[0]] for k in ("X", "Y", "Z")}
    assert arrays[0].tolist() == want["X"]
    assert arrays[1].tolist() == want["Y"]
    assert arrays[2].tolist() == want["Z"]
    assert arrays[1].tolist() != [int(x) for x in _rows("fig4_spatiotemporal.txt", "Y_figure")[0]]
    for r in _rows("fig4_spatiotemporal.txt", "xdesc"):
        i, j = int(r[0]), int(r[1])
        exp = None if r[2] == "-" else (int(r[2]), int(r[3]))
        assert ranges[0][(i, j)] == exp
    # each entry occupies at most 2 slabs per dimension (width constraint)
    for c in range(3):
        assert len(arrays[c]) <= 2 * D.shape[0]


def _fig_desc():
    rng = [{}, {}, {}]
    for r in _rows("fig4_spatiotemporal.txt", "fdesc"):
        i, j = int(r[0]), int(r[1])
        for c in range(3):
            s = r[2 + c]
            rng[c][(i, j)] = None if s == "-" else tuple(int(x) for x in s.split("-"))
    return rng


def test_selection_worked_example():
    # P:1054-1071 with the figure's own descriptors: query over bins 0-1, in x
    # slab 0, y slab 1, z slab 0 -> x: 4 entries, y: 3 (Y[7..9]), z: 4 -> pick Y [7, 9]
    assert ir.st_select(_fig_desc(), 0, 1, (0, 1, 0), (0, 1, 0)) == (1, 7, 9)
    # same query on the corrected arrays: x 4, y 4, z 5 -> tie broken to x: X[0..3]
    D, binof = fig4()
    _, ranges = ir.st_arrays(D, binof, 3, 3, (0, 0, 0), (4, 4, 5))
    assert ir.st_select(ranges, 0, 1, (0, 1, 0), (0, 1, 0)) == (0, 0, 3)
    # a query spanning two slabs in every dimension falls back to temporal
    assert ir.st_select(ranges, 0, 1, (0, 0, 0), (1, 1, 1)) == (-1, None, None)
    # only z usable -> z even if larger
    assert ir.st_select(ranges, 0, 1, (0, 0, 0), (1, 1, 0)) == (2, 0, 4)


def test_linearize_spec_examples():
    assert ir.linearize(0, 0, 0, (4, 5, 6)) == 0
    assert ir.linearize(1, 2, 3, (4, 5, 6)) == 45
    assert ir.linearize(3, 4, 5, (4, 5, 6)) == 119


def test_fig1_rasterization():
    # 5 x 4 cells of unit size in x-y (one z cell); l1 (2.6,1.2)-(1.2,3.5), l2 (4.1,2.1)-(4.8,2.9)
    grid, o, w = (5, 4, 1), (0, 0, 0), (1, 1, 1)
    l1 = ir.rasterize((1.2, 1.2, 0.5), (2.6, 3.5, 0.5), o, w, grid)
    l2 = ir.rasterize((4.1, 2.1, 0.5), (4.8, 2.9, 0.5), o, w, grid)
    assert sorted((x, y) for x, y, _ in l1) == sorted([(1, 1), (2, 1), (1, 2), (2, 2), (1, 3), (2, 3)])
    assert [(x, y) for x, y, _ in l2] == [(4, 2)]


def test_fig2_lookup_keeps_duplicates():
    # Fig. 2 (text P:449-463): G has h=0 -> A[0..2] = {2, 100, 22},
    # h=7 -> A[25..90] with A[25]=100, A[26]=867, A[90]=400; C1 is empty.
    A = np.arange(126) + 10000
    A[0:3] = [2, 100, 22]
    A[25], A[26], A[90] = 100, 867, 400
    A[124], A[125] = 1, 100
    Gm = np.array([(0, 0, 2), (2, 3, 24), (7, 25, 90), (12, 91, 123), (20, 124, 125)])
    U = ir.fsg_candidates(Gm, A, [0, 1, 7])
    assert U[:5] == [2, 100, 22, 100, 867] and U[-1] == 400 and len(U) == 3 + 66
    assert U.count(100) == 2


def test_fsg_build_roundtrip():
    rng = np.random.default_rng(3)
    D = rng.uniform(0, 10, (60, 8)).astype(np.float32)
    grid, o, w = (4, 3, 5), (0, 0, 0), (2.5, 10 / 3, 2)
    Gm, A = ir.fsg_build(D, grid, o, w)
    assert np.all(np.diff(Gm[:, 0]) > 0)
    total = 0
    for e in range(60):
        mn, mx = np.minimum(D[e, :3], D[e, 4:7]), np.maximum(D[e, :3], D[e, 4:7])
        cells = ir.rasterize(mn, mx, o, w, grid)
        total += len(cells)
        for c in cells:
            k = np.searchsorted(Gm[:, 0], ir.linearize(*c, grid))
            assert e in A[Gm[k, 1]:Gm[k, 2] + 1]
    assert len(A) == total                                # #A = sum of cells per MBB


# ---------------------------------------------------------------------------
# extents, admissible v, geometry, C13 lookup and the schedule
# ---------------------------------------------------------------------------
def test_spatial_extent_and_admissible_v_fig4():
    """Hand-derived from the Fig. 4 entry rows (golden file): x spans [0, 10]
    (l9 starts at 0, l6 ends at 10) with the largest per-segment x extent 2
    (l2, l4, l6, l9); y spans [2, 9] with largest extent 3 (l5, l9); z spans
    [1, 13] with largest extent 6 (l4: 1 -> 7).  P:816-821: v <= floor(ext /
    max extent) -> 5, 2 and exactly 12 / 6 = 2 (an integral bound)."""
    D, _ = fig4()
    lo, hi, mx = ir.spatial_extent(D)
    assert lo.tolist() == [0.0, 2.0, 1.0]
    assert hi.tolist() == [10.0, 9.0, 13.0]
    assert mx.tolist() == [2.0, 3.0, 6.0]
    assert ir.admissible_v(D).tolist() == [5.0, 2.0, 2.0]


def test_spatial_extent_uses_both_endpoints_and_the_max():
    # every extreme sits at a segment END, and the two segments have different
    # per-dimension extents (a mean or a start-only reduction fails this)
    D = np.array([[0, 0, 0, 0, 3, -1, 2, 1],
                  [1, 1, 1, 0, -2, 4, 0, 1]], np.float32)
    lo, hi, mx = ir.spatial_extent(D)
    assert lo.tolist() == [-2.0, -1.0, 0.0]
    assert hi.tolist() == [3.0, 4.0, 2.0]
    assert mx.tolist() == [3.0, 3.0, 2.0]          # |3-0|, |4-1|, |2-0|
    assert ir.admissible_v(D).tolist() == [1.0, 1.0, 1.0]
    # 2.9999 -> 2 (floor), a zero extent -> unbounded
    D2 = np.array([[0, 0, 5, 0, 1, 0, 5, 1], [2.9999, 0, 5, 1, 1.9999, 0, 5, 2]], np.float32)
    v = ir.admissible_v(D2)
    assert v[0] == 2.0 and np.isinf(v[1]) and np.isinf(v[2])


def test_grid_geometry():
    D = np.array([[0, 5, -1, 0, 12, 5, 2, 1]], np.float32)
    o, w = ir.grid_geometry(D, (3, 4, 2))
    assert o.tolist() == [0.0, 5.0, -1.0]
    assert w.tolist() == [4.0, 1.0, 1.5]            # 12/3, zero extent -> 1, 3/2


def test_member_extent_bins_fig3():
    """C13 on Fig. 3 (m = 4): bin j's members end by 7.5, 6.2, 11, 12 and start
    from 0, 3.9, 6.5, 9.3 (golden rows).  (3.0, 3.5): B_0 has members ending
    after 3.0 and starting before 3.5; B_1's members all start at >= 3.9 ->
    bins 0..0, although the literal B_1 = [3, 6.2] overlaps the query."""
    Ds, _ = ir.temporal_sort(fig3_segments())
    b = ir.temporal_bins(Ds, 4)
    f = lambda a, z: ir.member_extent_bins(Ds, b["bin_of"], 4, a, z)
    assert f(5.0, 5.5) == (0, 1)
    assert f(3.0, 3.5) == (0, 0)
    assert ir.temporal_schedule(b, 3.0, 3.5) == (0, 8)         # the literal bins: a superset
    assert f(6.5, 6.9) == (0, 2)
    assert f(7.55, 7.6) == (2, 2)                              # B_0 ends at 7.5 < 7.55
    assert f(11.95, 12.5) == (3, 3)
    assert f(12.5, 13.0) is None                               # nothing ends after 12.5
    assert f(11.5, 11.6) == (3, 3)                             # B_2's members end by 11 < 11.5
    assert f(-1.0, 0.0) is None                                # touches l0's start only (C5)


def test_query_slabs_round_outward():
    # 1 - 1e-8 rounds to 1.0 under round-to-nearest (slab 1); rounded down it is
    # 0.99999994 (slab 0): the inflated box must include slab 0 (completeness)
    lo, hi = ir.query_slabs(np.array([1, 1, 1, 0, 1, 1, 1, 1], np.float32), 1e-8, (0, 0, 0), (1, 1, 1), 4)
    assert lo == [0, 0, 0] and hi == [1, 1, 1]
    assert ir.d_up32(0.1) >= 0.1 and float(ir.d_up32(0.1)) == float(np.nextafter(np.float32(0.1), np.inf)) \
        or float(np.float32(0.1)) >= 0.1


def _plan_fixture():
    # 4 entries, m = 2 bins over t in [0, 3] (b = 1.5), v = 2 slabs per dimension
    # over x [0, 4], y [0, 2], z [0, 1] (widths 2, 1, 0.5)
    D = np.array([[0, 0, 0, 0, 1, 0, 0, 1],
                  [3, 1, 0, 0, 4, 1, 0, 1],
                  [0, 0, 0, 2, 0, 1, 0, 3],
                  [4, 2, 1, 2, 4, 2, 1, 3]], np.float32)
    Q = np.array([[0.5, 0.2, 0, 0.2, 0.5, 0.2, 0, 0.8],      # x/y/z slab 0, bin 0: x and y tie at 1 -> x
                  [1.9, 1.5, 0.5, 2.1, 2.1, 1.5, 0.5, 2.9],  # only y usable (slab 1), bin 1: Y[3:5]
                  [1.9, 0.95, 0.5, 0.1, 2.1, 1.05, 0.5, 0.9],  # two slabs everywhere: temporal fallback
                  [0.5, 0.2, 0, 5, 0.5, 0.2, 0, 6],          # after every entry: nothing
                  [0.5, 0.2, 0, 1, 0.5, 0.2, 0, 2],          # touches bin 0's ends and bin 1's starts (C5)
                  [0.5, 0.2, 0.8, 0.2, 0.5, 0.2, 0.8, 0.8]], np.float32)   # z slab 1 of bin 0 is empty -> picked
    d = [0.25, 0.05, 0.05, 0.05, 0.05, 0.05]
    return D, Q, d


def test_st_arrays_and_plan_hand_example():
    D, Q, d = _plan_fixture()
    Ds, _ = ir.temporal_sort(D)
    b = ir.temporal_bins(Ds, 2)
    assert b["bin_of"].tolist() == [0, 0, 1, 1]
    o, w = ir.grid_geometry(D, (2, 2, 2))
    assert w.tolist() == [2.0, 1.0, 0.5]
    arrays, _ = ir.st_arrays(Ds, b["bin_of"], 2, 2, o, w)
    assert [a.tolist() for a in arrays] == [[0, 2, 1, 3], [0, 2, 1, 2, 3], [0, 1, 2, 3]]
    st = [tuple(ir.plan(D, Q[k:k + 1], d[k], 2, 2, "spatiotemporal")[0]) for k in range(len(Q))]
    assert st == [(0, 0, 1), (1, 3, 5), (-1, 0, 2), (3, 0, 0), (3, 0, 0), (3, 0, 0)]
    tp = [tuple(ir.plan(D, Q[k:k + 1], d[k], 2, 2, "temporal")[0]) for k in range(len(Q))]
    assert tp == [(-1, 0, 2), (-1, 2, 4), (-1, 0, 2), (3, 0, 0), (3, 0, 0), (-1, 0, 2)]
    # a window that clips the query to nothing
    assert tuple(ir.plan(D, Q[:1], 0.25, 2, 2, "temporal", window=(0.5, 1.0))[0]) == (-1, 0, 2)
    assert tuple(ir.plan(D, Q[:1], 0.25, 2, 2, "temporal", window=(0.8, 1.0))[0]) == (3, 0, 0)


def test_morton30_hand_values():
    # bit k of x, y, z -> bits 3k+2, 3k+1, 3k
    assert ir.morton30([1, 0, 0, 1, 2, 1023], [0, 1, 0, 1, 0, 1023], [0, 0, 1, 1, 0, 1023]).tolist() == \
        [4, 2, 1, 7, 32, (1 << 30) - 1]


def test_spatial_sort_hand_example():
    """Default renumbering: by temporal bin, then Morton code of the start cell on
    a 1024^3 grid over the extent.  Extent [0, 1024]^3 -> unit cells."""
    D = np.array([[2, 0, 0, 0.0, 2, 0, 0, 1],       # bin 0, cell (2,0,0) -> 32
                  [0, 0, 1, 0.5, 0, 0, 1, 1.5],     # bin 0, (0,0,1) -> 1
                  [1, 1, 1, 0.2, 1, 1, 1, 1.2],     # bin 0, (1,1,1) -> 7
                  [0, 0, 0, 3.0, 0, 0, 0, 4.0],     # bin 1, (0,0,0) -> 0
                  [0, 1, 0, 2.5, 1024, 1024, 1024, 3.5],   # bin 1, (0,1,0) -> 2
                  [0, 0, 1, 0.1, 0, 0, 1, 1.1]],    # bin 0, (0,0,1) -> 1, after row 1 (stable)
                 np.float32)
    Ds, perm = ir.spatial_sort(D, 2)               # t in [0, 4]: b = 2, bins t0 < 2 | >= 2
    assert perm.tolist() == [1, 5, 2, 0, 3, 4]
    assert ir.temporal_sort(D)[1].tolist() == [0, 5, 2, 1, 4, 3]
    # the same entries per bin under both orders
    b_s = ir.temporal_bins(Ds, 2)
    b_t = ir.temporal_bins(ir.temporal_sort(D)[0], 2)
    for j in range(2):
        assert b_s["B_first"][j] == b_t["B_first"][j] and b_s["B_last"][j] == b_t["B_last"][j]
        assert b_s["B_end"][j] == b_t["B_end"][j]

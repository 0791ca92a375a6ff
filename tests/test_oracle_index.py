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

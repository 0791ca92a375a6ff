"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Marked gpu: run on a B200 via gpurun."""
import math

import numpy as np
import pytest

import oracle
import synth
from parity import check, keys

pytestmark = pytest.mark.gpu

KINDS = ("temporal", "spatiotemporal", "spatial")


@pytest.fixture(scope="module")
def tds():
    import torch
    import paper_1410_2698_b200 as t
    t.load_library()
    assert torch.cuda.is_available()
    return t


def _cuda(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(idx, Q, d, kind, window=(-math.inf, math.inf), capacity=0):
    r = idx.search(_cuda(Q), d, window=window, kind=kind, capacity=capacity)
    got = r.fetch(sorted=True, device=False)
    st = r.stats()
    r.close()
    return got, st


@pytest.fixture(scope="module")
def tiny():
    w = synth.tiny()
    return w, oracle.search(w.D, w.Q, w.d)


@pytest.mark.parametrize("kind", KINDS)
def test_tiny_default(tds, tiny, kind):
    w, ref = tiny
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    got, st = _run(idx, w.Q, w.d, kind)
    rep = check(got, ref, w.D, w.Q, w.d, label=kind)
    assert rep["pairs"] > 50
    assert st["n_results"] == len(got[0])


@pytest.mark.parametrize("m", [1, 3, 10, 100])
@pytest.mark.parametrize("v", [1, 2, 3])
def test_tiny_param_sweep_temporal_st(tds, tiny, m, v):
    w, ref = tiny
    idx = tds.Index(_cuda(w.D), kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=m, v=v)
    for kind in ("temporal", "spatiotemporal"):
        got, _ = _run(idx, w.Q, w.d, kind)
        check(got, ref, w.D, w.Q, w.d, label=f"{kind} m={m} v={v}")


@pytest.mark.parametrize("g", [1, 4, 10, 33])
def test_tiny_grid_sweep_spatial(tds, tiny, g):
    w, ref = tiny
    idx = tds.Index(_cuda(w.D), kinds=tds.SPATIAL, m=10, grid=(g, g, max(1, g // 2)))
    got, _ = _run(idx, w.Q, w.d, "spatial")
    check(got, ref, w.D, w.Q, w.d, label=f"spatial g={g}")


@pytest.mark.parametrize("cap", [1, 7, 100, 1000])
@pytest.mark.parametrize("kind", KINDS)
def test_tiny_forced_capacity(tds, tiny, cap, kind):
    """Overflow re-launch: results identical whatever the buffer size."""
    w, ref = tiny
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    if cap == 1:
        # some query has more than one record -> one query alone exceeds the capacity
        with pytest.raises(tds.TdsError) as ei:
            _run(idx, w.Q, w.d, kind, capacity=cap)
        assert ei.value.status == "TDS_ECAPACITY"
        return
    got, st = _run(idx, w.Q, w.d, kind, capacity=cap)
    check(got, ref, w.D, w.Q, w.d, label=f"{kind} cap={cap}")
    if cap < len(got[0]):
        assert st["passes"] > 1


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("window", [(8.0, 12.0), (0.0, 3.5), (13.2, 13.2000005), (30.0, 40.0)])
def test_tiny_window(tds, tiny, kind, window):
    w, _ = tiny
    ref = oracle.search(w.D, w.Q, w.d, window=window)
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    got, _ = _run(idx, w.Q, w.d, kind, window=window)
    check(got, ref, w.D, w.Q, w.d, window=window, label=f"{kind} {window}")


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("d", [1e-3, 0.3, 7.0, 50.0])
def test_tiny_d_sweep(tds, tiny, kind, d):
    w, _ = tiny
    ref = oracle.search(w.D, w.Q, d)
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=1, grid=w.grid)
    got, _ = _run(idx, w.Q, d, kind)
    check(got, ref, w.D, w.Q, d, label=f"{kind} d={d}")


def test_edge_cases(tds, tiny):
    w, _ = tiny
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    # empty query set
    r = idx.search(_cuda(np.zeros((0, 8), np.float32)), 1.0)
    assert r.count == 0
    # queries entirely outside the data in time and space
    Q = w.Q.copy()
    Q[:, 3] += 1000
    Q[:, 7] += 1000
    for kind in KINDS:
        assert idx.search(_cuda(Q), w.d, kind=kind).count == 0
    # stationary queries and a query identical to an entry (self hit over its span)
    Q = np.concatenate([w.D[:7], w.D[:3]]).copy()
    Q[7:, 4:7] = Q[7:, 0:3]
    ref = oracle.search(w.D, Q, 0.5)
    for kind in KINDS:
        got, _ = _run(idx, Q, 0.5, kind)
        check(got, ref, w.D, Q, 0.5, label=f"edge {kind}")
    # error paths
    bad = w.Q.copy()
    bad[5, 7] = bad[5, 3]
    with pytest.raises(tds.TdsError) as ei:
        idx.search(_cuda(bad), 1.0)
    assert ei.value.status == "TDS_EDATA"
    with pytest.raises(tds.TdsError) as ei:
        idx.search(_cuda(w.Q), 0.0)
    assert ei.value.status == "TDS_EINVAL"
    with pytest.raises(tds.TdsError) as ei:
        tds.Index(_cuda(w.D), kinds=tds.SPATIOTEMPORAL, m=10, v=10_000)
    assert ei.value.status == "TDS_EINVAL"
    badD = w.D.copy()
    badD[17, 2] = np.nan
    with pytest.raises(tds.TdsError) as ei:
        tds.Index(_cuda(badD), kinds=tds.TEMPORAL, m=10)
    assert ei.value.status == "TDS_EDATA" and "17" in str(ei.value)


def test_host_inputs_and_host_fetch(tds, tiny):
    """The C-ABI accepts host buffers (e2e path)."""
    w, ref = tiny
    idx = tds.Index(w.D, kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    r = idx.search(w.Q, w.d, kind="temporal")
    got = r.fetch(sorted=True, device=False)
    check(got, ref, w.D, w.Q, w.d, label="host")


@pytest.mark.parametrize("order", ["time", "spatial"])
def test_index_build_matches_paper_structures(tds, tiny, order):
    """GPU extents / renumbering / bins / X-Y-Z / FSG arrays equal oracle/index_ref
    on the same data, for the paper's t_start renumbering and for the default
    (bin, Morton) one; the geometry (extents, slab and cell widths) is computed
    by index_ref from D, not taken from the GPU."""
    from oracle import index_ref as ir
    w, _ = tiny
    m, v, grid = 7, 2, (4, 3, 5)
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=m, v=v, grid=grid, time_order=(order == "time"))
    ext = idx.export("extents")
    lo, hi, mx = ir.spatial_extent(w.D)
    assert np.array_equal(ext[2:5], lo.astype(np.float32)) and np.array_equal(ext[5:8], hi.astype(np.float32))
    assert np.array_equal(ext[8:11], mx.astype(np.float32))      # |c1 - c0| rounded to float32
    assert ext[0] == w.D[:, 3].min() and ext[1] == w.D[:, 7].max()
    Ds, perm = ir.temporal_sort(w.D) if order == "time" else ir.spatial_sort(w.D, m)
    assert np.array_equal(idx.export("perm"), perm)
    b = ir.temporal_bins(Ds, m)
    off = idx.export("bin_off").astype(np.int64)
    for j in range(m):
        if b["B_first"][j] >= 0:
            assert off[j] == b["B_first"][j] and off[j + 1] - 1 == b["B_last"][j]
            assert max(b["B_start"][j] + b["b"], idx.export("bin_hi")[j]) == pytest.approx(b["B_end"][j])
        else:
            assert off[j] == off[j + 1]
    o, wst = ir.grid_geometry(w.D, (v, v, v))
    assert np.array_equal(ext[11:14], wst)
    arrays, ranges = ir.st_arrays(Ds, b["bin_of"], m, v, o, wst)
    for c, name in enumerate(("st_x", "st_y", "st_z")):
        assert np.array_equal(idx.export(name), arrays[c])
        offs = idx.export(["st_off_x", "st_off_y", "st_off_z"][c])
        for (i, j), rg in ranges[c].items():
            a0, a1 = offs[j * m + i], offs[j * m + i + 1]
            assert (rg is None and a0 == a1) or (rg is not None and (a0, a1 - 1) == rg)
    o_f, wf = ir.grid_geometry(w.D, grid)
    G, A = ir.fsg_build(Ds, grid, o_f, wf)
    cell_off = idx.export("fsg_cell_off")
    A_gpu = idx.export("fsg_A")
    assert np.array_equal(A_gpu, A)
    for h, a0, a1 in G:
        assert cell_off[h] == a0 and cell_off[h + 1] == a1 + 1


def _window_boxes_np(D, rows, W=128):
    """Per aligned window of W candidate positions: the segments' MBB and time span."""
    nw = (len(rows) + W - 1) // W
    out = np.empty((nw, 8), np.float32)
    for k in range(nw):
        s = D[rows[k * W:(k + 1) * W]]
        out[k, 0:3] = np.minimum(s[:, 0:3], s[:, 4:7]).min(axis=0)
        out[k, 3] = s[:, 3].min()
        out[k, 4:7] = np.maximum(s[:, 0:3], s[:, 4:7]).max(axis=0)
        out[k, 7] = s[:, 7].max()
    return out


@pytest.mark.parametrize("order", ["time", "spatial"])
def test_window_boxes_match_segment_mbbs(tds, tiny, order):
    """The index's window boxes (the range kernel skips a window whose box no
    query box meets) equal the MBB / time span of the segments of each aligned
    128-position window, for every candidate order, ragged last window included."""
    w, _ = tiny
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=7, v=2, grid=(4, 3, 5), time_order=(order == "time"))
    perm = idx.export("perm").astype(np.int64)
    assert len(perm) % 128 != 0
    assert np.array_equal(idx.export("wb_rec").reshape(-1, 8), _window_boxes_np(w.D, perm))
    for c in "xyz":
        ids = idx.export("st_" + c).astype(np.int64)
        assert np.array_equal(idx.export("wb_" + c).reshape(-1, 8), _window_boxes_np(w.D, perm[ids]))
    A = idx.export("fsg_A").astype(np.int64)
    assert np.array_equal(idx.export("wb_fsg").reshape(-1, 8), _window_boxes_np(w.D, perm[A]))


def test_admissible_v_matches_index_ref(tds, tiny):
    """the build accepts v up to index_ref.admissible_v (same v in all
    dimensions, so the smallest bound) and rejects the next."""
    from oracle import index_ref as ir
    w, _ = tiny
    vmax = int(ir.admissible_v(w.D).min())
    assert vmax >= 1
    tds.Index(_cuda(w.D), kinds=tds.SPATIOTEMPORAL, m=5, v=vmax).close()
    with pytest.raises(tds.TdsError) as ei:
        tds.Index(_cuda(w.D), kinds=tds.SPATIOTEMPORAL, m=5, v=vmax + 1)
    assert ei.value.status == "TDS_EINVAL"


@pytest.mark.parametrize("case", ["tiny", "tiny-window", "dense-small", "hand"])
@pytest.mark.parametrize("kind", ["temporal", "spatiotemporal"])
def test_plan_matches_index_ref(tds, case, kind):
    """tds_plan (the GPU schedule: C13 bin lookup, slab choice, fallback) equals
    index_ref.plan query by query: same selector (dimension or temporal
    fallback or empty) and the same range."""
    from oracle import index_ref as ir
    window = (-math.inf, math.inf)
    if case.startswith("tiny"):
        w = synth.tiny()
        D, Q, d, m, v = w.D, w.Q, w.d, 10, 2
        if case == "tiny-window":
            window = (1.5, 4.25)
    elif case == "dense-small":
        w = synth.random_dense(n_particles=512, n_timesteps=13, n_query_traj=64)
        D, Q, d, m, v = w.D, w.Q, 0.001, 12, 2
    else:
        import test_oracle_index as toi
        D, Q, ds = toi._plan_fixture()
        d, m, v = ds[0], 2, 2
    idx = tds.Index(_cuda(D), kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=m, v=v)
    sel, lo, hi = idx.plan(_cuda(Q), d, window=window, kind=kind)
    want = ir.plan(D, Q, d, m, v, kind, window=window, order="spatial")
    got = np.stack([sel.astype(np.int64), lo.astype(np.int64), hi.astype(np.int64)], 1)
    bad = np.nonzero((got != want).any(1))[0]
    assert bad.size == 0, f"{bad.size} queries differ, e.g. {[(int(k), got[k].tolist(), want[k].tolist()) for k in bad[:5]]}"
    if kind == "spatiotemporal" and case != "hand":
        assert ((sel >= 0) & (sel < 3)).any()             # both subbin and fallback paths exercised
        assert ((sel == -1) | (sel == 3)).any()


@pytest.fixture(scope="module")
def r1m():
    w = synth.random_1m()
    rng = np.random.default_rng(11)
    sel = np.sort(rng.choice(w.Q.shape[0], 600, replace=False))
    return w, sel


@pytest.mark.parametrize("d", [5.0, 50.0])
def test_random_1m_subsample(tds, r1m, d):
    """Random-1M-shaped at full size, the bench's launch configuration; oracle on
    a query subsample, all three variants cross-checked on the full query set."""
    w, sel = r1m
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    full = {}
    for kind in KINDS:
        got, st = _run(idx, w.Q, d, kind)
        full[kind] = (keys(got[0], got[1]), got)
    ref = oracle.search(w.D, w.Q, d, qsel=sel)
    m = np.isin(full["temporal"][1][0], sel)
    for kind in KINDS:
        g = full[kind][1]
        mk = np.isin(g[0], sel)
        check(tuple(x[mk] for x in g), ref, w.D, w.Q, d, label=f"r1m {kind} d={d}")
    # full-set cross-variant equality (all variants are filters of the same set)
    base = np.sort(full["temporal"][0])
    for kind in ("spatiotemporal", "spatial"):
        assert np.array_equal(np.sort(full[kind][0]), base), kind
    assert m.sum() > 0


@pytest.mark.parametrize("name,kinds", [("random-dense-1m", ("spatiotemporal", "temporal")),
                                        ("merger-small", KINDS)])
def test_dense_and_merger_subsample(tds, name, kinds):
    if name == "merger-small":
        w = synth.merger(n_per_disk=8192)
        d = 1.0
    else:
        w = synth.make_workload(name)
        d = 0.01
    rng = np.random.default_rng(5)
    sel = np.sort(rng.choice(w.Q.shape[0], 300, replace=False))
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins if name != "random-dense-1m" else 2,
                    grid=w.grid)
    ref = oracle.search(w.D, w.Q, d, qsel=sel)
    sets = []
    for kind in kinds:
        got, _ = _run(idx, w.Q, d, kind)
        mk = np.isin(got[0], sel)
        check(tuple(x[mk] for x in got), ref, w.D, w.Q, d, label=f"{name} {kind}")
        sets.append(np.sort(keys(got[0], got[1])))
    for s2 in sets[1:]:
        assert np.array_equal(s2, sets[0])


@pytest.mark.parametrize("name", ["tiny", "merger-small"])
def test_fsg_time_trim_equals_literal(tds, name, monkeypatch):
    """GPUSpatial with per-cell time trimming returns exactly the paper-literal
    FSG result (TDS_FSG_LITERAL=1: whole cells as candidates), and
    the literal result equals the oracle's."""
    w = synth.tiny() if name == "tiny" else synth.merger(n_per_disk=4096)
    d = w.d if name == "tiny" else 1.5
    idx = tds.Index(_cuda(w.D), kinds=tds.SPATIAL, m=10, grid=w.grid)
    got, st = _run(idx, w.Q, d, "spatial")
    monkeypatch.setenv("TDS_FSG_LITERAL", "1")
    lit, st_l = _run(idx, w.Q, d, "spatial")
    monkeypatch.delenv("TDS_FSG_LITERAL")
    assert np.array_equal(np.sort(keys(got[0], got[1])), np.sort(keys(lit[0], lit[1])))
    # the literal mode (and so the trimmed one) against the oracle: all queries on
    # tiny, 64 time-stratified queries on the Merger-shaped case
    from parity import stratified
    sel = np.arange(w.Q.shape[0]) if name == "tiny" else stratified(w.Q, 64, seed=5)
    ref = oracle.search(w.D, w.Q, d, qsel=sel)
    lq = np.asarray(lit[0])
    keep = np.isin(lq, sel)
    check(tuple(np.asarray(x)[keep] for x in lit), ref, w.D, w.Q, d, label=f"FSG literal {name}")
    assert st["pair_tests"] <= st_l["pair_tests"]
    if name != "tiny":
        assert st["pair_tests"] < st_l["pair_tests"] / 4      # time trimming prunes most of a cell


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gap", [0.0, 0.75])
def test_trajectory_merge(tds, tiny, kind, gap):
    """tds_merge_trajectories equals oracle.merge_trajectories applied to the
    oracle's segment-level result (pairs in the 1e-5 d band excluded on both
    sides: their presence may differ)."""
    w, ref = tiny
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    r = idx.search(_cuda(w.Q), w.d, kind=kind)
    m = r.merge_trajectories(w.traj_Q.astype(np.uint32), w.traj_D.astype(np.uint32), gap=gap)
    gq, ge, gi, go = m.fetch(sorted=True, device=False)
    band = np.abs(ref["dmin"] - w.d) <= 1e-5 * w.d
    if band.any():
        pytest.skip("band pairs present: trajectory-level comparison would need band handling")
    h = ref["hit"]
    om = oracle.merge_trajectories(ref["qid"][h], ref["eid"][h], ref["t_in"][h], ref["t_out"][h],
                                   w.traj_Q, w.traj_D, gap=gap)
    order = np.lexsort((gi, ge, gq))
    assert len(gq) == len(om["qtraj"])
    assert np.array_equal(gq[order], om["qtraj"]) and np.array_equal(ge[order], om["etraj"])
    span = np.maximum(1.0, np.abs(om["t_in"]))
    assert np.all(np.abs(gi[order] - om["t_in"]) <= 1e-5 * span)
    assert np.all(np.abs(go[order] - om["t_out"]) <= 1e-5 * np.maximum(1.0, np.abs(om["t_out"])))
    assert len(gq) < r.count                       # trajectory answers merge segment records


def test_trajectory_merge_crossing_boundary(tds):
    Q = np.array([[-5, 0, 0, 0, 0, 0, 0, 5], [0, 0, 0, 5, 5, 0, 0, 10]], np.float32)
    D = np.array([[0, 0, 0, 0, 0, 0, 0, 5], [0, 0, 0, 5, 0, 0, 0, 10]], np.float32)
    idx = tds.Index(_cuda(D), kinds=tds.ALL, m=2, v=1, grid=(2, 2, 2))
    for kind in KINDS:
        r = idx.search(_cuda(Q), 1.0, kind=kind)
        m = r.merge_trajectories(np.array([7, 7], np.uint32), np.array([3, 3], np.uint32))
        q, e, ti, to = m.fetch(device=False)
        assert (q.tolist(), e.tolist(), ti.tolist(), to.tolist()) == ([7], [3], [4.0], [6.0])


@pytest.mark.parametrize("world", [2, 3])
def test_time_partitioned_union_equals_single_index(tds, world):
    """SURVEY §8f-1 on one GPU: the union over `world` time slices of D (each
    with its own index, every query against every slice) equals the single-index
    result, without duplicates, with entry ids mapped back to rows of D."""
    import torch
    from paper_1410_2698_b200.dist import TimeShardedIndex
    w = synth.random_1m(n_traj=400)
    ref = oracle.search(w.D, w.Q, 20.0)
    full = tds.Index(_cuda(w.D), kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=1000, v=2)
    for kind in ("temporal", "spatiotemporal"):
        r = full.search(_cuda(w.Q), 20.0, kind=kind)
        a = r.fetch(sorted=True, device=False)
        ka = np.sort(keys(a[0], a[1]))
        parts = []
        for rank in range(world):
            sh = TimeShardedIndex(w.D, rank, world, kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=1000, v=2)
            q, e, ti, to = sh.search(_cuda(w.Q), 20.0, kind=kind)
            parts.append([x.cpu().numpy() for x in (q, e, ti, to)])
        u = [np.concatenate([p_[k] for p_ in parts]) for k in range(4)]
        check(tuple(u), ref, w.D, w.Q, 20.0, label=f"time slices x{world} {kind}")   # the oracle, no duplicates
        assert np.array_equal(ka, np.sort(keys(u[0], u[1])))


@pytest.mark.parametrize("kind", ["temporal", "spatiotemporal", "spatial"])
def test_touching_spans_dense_window(tds, kind):
    """C5 on the in-place (dense window) path: 200 entries whose spans touch the
    query's span at one instant (t_end = 1 or t_start = 2) sit next to 200 that
    overlap it, all within d of the stationary query; only the overlapping ones
    interact.  (The fp32 filter passes touching spans; the later stages decide.)"""
    import torch
    rng = np.random.default_rng(7)
    n = 200
    pos = rng.uniform(-0.1, 0.1, (3 * n, 3)).astype(np.float32)
    t0 = np.concatenate([np.full(n, 0.0), np.full(n, 2.0), rng.uniform(0.5, 1.5, n)]).astype(np.float32)
    t1 = np.concatenate([np.full(n, 1.0), np.full(n, 3.0), t0[2 * n:] + 1.0]).astype(np.float32)
    order = rng.permutation(3 * n)
    D = np.concatenate([pos, t0[:, None], pos, t1[:, None]], axis=1)[order].astype(np.float32)
    Q = np.array([[0, 0, 0, 1.0, 0, 0, 0, 2.0]], np.float32)
    ref = oracle.search(D, Q, 1.0)
    idx = tds.Index(_cuda(D), kinds=tds.ALL, m=4, v=1, grid=(4, 4, 4))
    got = idx.search(_cuda(Q), 1.0, kind=kind).fetch(sorted=True, device=False)
    rep = check(got, ref, D, Q, 1.0, label=f"touching {kind}")
    assert rep["pairs"] == n


@pytest.mark.parametrize("kind", ["temporal", "spatiotemporal", "spatial"])
def test_output_bound_windows(tds, kind):
    """Output-bound regime (most candidate windows dense: the in-place fp32
    interval path, hit_kind2, and the fused dense-window mode): 20,000 short
    random-walk segments in a small box, 300 queries from D, d chosen so that
    about half of the time-overlapping pairs interact; full comparison."""
    import torch
    rng = np.random.default_rng(11)
    ntraj, nseg = 400, 50
    start = rng.uniform(0, 4, (ntraj, 1, 3))
    steps = rng.uniform(-0.2, 0.2, (ntraj, nseg, 3))
    pos = np.concatenate([start, start + np.cumsum(steps, axis=1)], axis=1)
    t = np.arange(nseg + 1, dtype=np.float64)[None, :, None] + rng.uniform(0, 3, (ntraj, 1, 1))
    P = np.concatenate([pos, np.broadcast_to(t, (ntraj, nseg + 1, 1))], axis=2)
    D = np.concatenate([P[:, :-1, :], P[:, 1:, :]], axis=2).reshape(-1, 8).astype(np.float32)
    Q = D[rng.choice(D.shape[0], 300, replace=False)]
    d = 3.0
    ref = oracle.search(D, Q, d)
    idx = tds.Index(_cuda(D), kinds=tds.ALL, m=40, v=2, grid=(8, 8, 8))
    r = idx.search(_cuda(Q), d, kind=kind)
    got = r.fetch(sorted=True, device=False)
    rep = check(got, ref, D, Q, d, label=f"output-bound {kind}")
    assert rep["pairs"] > 90000


def test_search_many_equals_single_searches(tds):
    """tds_search_many: the three variants concurrently on three streams, plus two
    requests sharing a stream (a serial lane), give exactly the single searches'
    records (same pair sets, same endpoints bit for bit)."""
    import torch
    w = synth.random_1m(n_traj=300)
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=1000, v=2)
    Q = _cuda(w.Q)
    streams = [torch.cuda.Stream() for _ in range(3)]
    reqs = [{"queries": Q, "d": 25.0, "kind": k, "stream": streams[j].cuda_stream}
            for j, k in enumerate(("temporal", "spatiotemporal", "spatial"))]
    reqs.append({"queries": Q[: Q.shape[0] // 2], "d": 10.0, "kind": "temporal", "window": (20.0, 60.0),
                 "stream": streams[0].cuda_stream})
    many = idx.search_many(reqs)
    torch.cuda.synchronize()
    for r, res in zip(reqs, many):
        one = idx.search(r["queries"], r["d"], kind=r["kind"], window=r.get("window", (-np.inf, np.inf)))
        a = res.fetch(sorted=True, device=False)
        b = one.fetch(sorted=True, device=False)
        assert len(a[0]) == len(b[0]) > 0
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_search_many_error_frees_all(tds):
    import torch
    w = synth.tiny()
    idx = tds.Index(_cuda(w.D), kinds=tds.TEMPORAL, m=10)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with pytest.raises(tds.TdsError) as ei:
        idx.search_many([{"queries": _cuda(w.Q), "d": w.d, "kind": "temporal", "stream": s1.cuda_stream},
                         {"queries": _cuda(w.Q), "d": w.d, "kind": "spatial", "stream": s2.cuda_stream}])
    assert "not built" in str(ei.value)
    assert idx.search_many([]) == []


def test_st_materialised_ablation_same_result(tds, monkeypatch):
    """TDS_ST_MATERIALISE=1 (records copied in X/Y/Z order) gives
    exactly the default (indirect) GPUSpatioTemporal records."""
    w = synth.random_1m(n_traj=300)
    base = tds.Index(_cuda(w.D), kinds=tds.SPATIOTEMPORAL, m=1000, v=4)
    a = base.search(_cuda(w.Q), 30.0, kind="spatiotemporal").fetch(sorted=True, device=False)
    monkeypatch.setenv("TDS_ST_MATERIALISE", "1")
    mat = tds.Index(_cuda(w.D), kinds=tds.SPATIOTEMPORAL, m=1000, v=4)
    b = mat.search(_cuda(w.Q), 30.0, kind="spatiotemporal").fetch(sorted=True, device=False)
    assert len(a[0]) > 0
    check(b, oracle.search(w.D, w.Q, 30.0), w.D, w.Q, 30.0, label="ST materialised")
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("v, expect", [(4, "spatiotemporal"), (1, "temporal")])
def test_auto_kind_choice(tds, v, expect):
    """TDS_AUTO: with v = 4 and a small d
    the subbins cut the pair tests far below GPUTemporal's, so GPUSpatioTemporal
    runs; with v = 1 every subbin range equals the temporal range, so the
    cheaper-per-pair GPUTemporal runs.  The records equal that variant's."""
    w = synth.random_1m(n_traj=300)
    idx = tds.Index(_cuda(w.D), kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=1000, v=v)
    r = idx.search(_cuda(w.Q), 5.0, kind="auto")
    st = r.stats()
    assert st["kind"] == tds.KINDS[expect]
    assert st["pair_tests_alt"] > 0
    if expect == "spatiotemporal":
        assert st["pair_tests"] * 1.5 <= st["pair_tests_alt"]
    else:
        assert st["pair_tests_alt"] * 1.5 >= st["pair_tests"]
    a = r.fetch(sorted=True, device=False)
    b = idx.search(_cuda(w.Q), 5.0, kind=expect).fetch(sorted=True, device=False)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name", ["tiny", "random-1m-small"])
@pytest.mark.parametrize("kind", ["temporal", "spatiotemporal"])
def test_tight_range_equals_bin_hull(tds, name, kind, monkeypatch):
    """Entry-exact candidate ranges (TDS_TIGHT_RANGE=1; they need the
    paper's t_start renumbering inside the bins) return exactly the result of the
    paper-granularity bin hull with no more pair tests."""
    if name == "tiny":
        w = synth.tiny()
        d = w.d
    else:
        w = synth.random_1m(n_traj=300, query_frac_stride=10)
        d = 20.0
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid, time_order=True)
    hull, st_h = _run(idx, w.Q, d, kind)
    monkeypatch.setenv("TDS_TIGHT_RANGE", "1")
    got, st = _run(idx, w.Q, d, kind)
    monkeypatch.delenv("TDS_TIGHT_RANGE")
    assert np.array_equal(np.sort(keys(got[0], got[1])), np.sort(keys(hull[0], hull[1])))
    check(got, oracle.search(w.D, w.Q, d), w.D, w.Q, d, label=f"tight ranges {kind}")
    assert st["pair_tests"] <= st_h["pair_tests"]
    if name != "tiny" and kind == "temporal":
        assert st["pair_tests"] < st_h["pair_tests"]


@pytest.mark.parametrize("name", ["tiny", "random-dense-1m"])
@pytest.mark.parametrize("kind", KINDS)
def test_dense_windows_match_oracle(tds, name, kind):
    """Hit-heavy searches run the fused dense-window step (whole-span hits appended
    at once with [a, b], the rest through the refine queue), with ragged and
    partial windows: the oracle's pair set and intervals."""
    if name == "tiny":
        w = synth.tiny()
        d = w.d * 3.0
        qsel = np.arange(w.Q.shape[0])
    else:
        w = synth.make_workload("random-dense-1m")
        d = 0.09
        qsel = np.arange(0, w.Q.shape[0], 97)[:64]
    Q = w.Q[qsel]
    ref = oracle.search(w.D, Q, d)
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    got, st = _run(idx, Q, d, kind)
    assert st["n_results"] > 0.15 * st["pair_tests"] or kind == "spatial"    # hit-heavy: dense windows
    check(got, ref, w.D, Q, d, label=f"{kind} dense windows")


@pytest.mark.parametrize("kind", ["temporal", "spatiotemporal"])
def test_enomem_fallback_injected(tds, kind):
    """Fault injection: the automatic result capacity survives failed
    allocations of its pass buffer (tds_test_inject_enomem) by halving the
    capacity and re-taking the memory budget; the result is the same pair set as
    without failures, the failures were injected, and the capacity halved once
    per failure.  Failures down to the capacity floor surface as TDS_ENOMEM."""
    w = synth.random_1m(n_traj=300, query_frac_stride=10)
    d = 20.0
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    base, st = _run(idx, w.Q, d, kind)
    assert st["pair_tests"] > (1 << 20)              # above the halving floor
    nfail = 2 if st["pair_tests"] > 4 * (1 << 20) else 1
    n0 = tds.test_inject_enomem(nfail)
    got, st2 = _run(idx, w.Q, d, kind)
    assert tds.test_inject_enomem(0) == n0 + nfail
    assert st2["capacity"] == st["capacity"] >> nfail
    assert np.array_equal(np.sort(keys(got[0], got[1])), np.sort(keys(base[0], base[1])))
    ref = oracle.search(w.D, w.Q[:400], d)
    sel = got[0] < 400
    check(tuple(x[sel] for x in got), ref, w.D, w.Q[:400], d, label=f"{kind} enomem")
    small = w.Q[:50]
    n1 = tds.test_inject_enomem(64)                 # every attempt fails: halving reaches the floor
    with pytest.raises(tds.TdsError) as ei:
        _run(idx, small, d, kind)
    n2 = tds.test_inject_enomem(0)
    assert ei.value.status == "TDS_ENOMEM"
    assert n2 > n1 + 1                              # halved at least once before giving up


def test_enomem_injected_spatial_surfaces(tds):
    """GPUSpatial: injected pass-buffer allocation failures down to the capacity
    floor surface as TDS_ENOMEM, and the next search succeeds."""
    w = synth.tiny()
    idx = tds.Index(_cuda(w.D), kinds=tds.SPATIAL, m=w.m_bins, grid=w.grid)
    n0 = tds.test_inject_enomem(64)
    with pytest.raises(tds.TdsError) as ei:
        _run(idx, w.Q, w.d, "spatial")
    assert ei.value.status == "TDS_ENOMEM"
    assert tds.test_inject_enomem(0) > n0
    got, _ = _run(idx, w.Q, w.d, "spatial")
    check(got, oracle.search(w.D, w.Q, w.d), w.D, w.Q, w.d, label="spatial after injected ENOMEM")


def test_real_memory_pressure(tds):
    """Real memory pressure (no injection): a ballast allocation leaves the search
    room for 3/4 of its automatic pass buffer; the capacity halves on a real
    ENOMEM until the buffer fits (overflowing and spilling if it then holds
    fewer records than the result), and the records equal the unconstrained
    search's."""
    import torch
    w = synth.random_dense(n_particles=8192, n_timesteps=49, n_query_traj=1024)
    d = 0.03
    idx = tds.Index(_cuda(w.D), kinds=tds.TEMPORAL, m=200)
    Q = _cuda(w.Q)
    r = idx.search(Q, d, kind="temporal")
    base = r.fetch(sorted=True, device=False)
    st0 = r.stats()
    need = 16 * r.count
    r.close()
    assert need > (256 << 20)
    tds.trim()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    cap0 = 16 * st0["capacity"]
    if cap0 < (13 * need) // 10:
        pytest.skip("automatic capacity too close to the result size to squeeze")
    # leave room for 3/4 of the automatic pass buffer (at least 1.2x the records):
    # the first allocation fails for real and the capacity halves
    room = max((12 * need) // 10, (3 * cap0) // 4)
    ballast = torch.empty(max(0, free - room - (64 << 20)), dtype=torch.uint8, device="cuda")
    try:
        tds.trim()
        r = idx.search(Q, d, kind="temporal")
        st = r.stats()
    finally:
        del ballast
        torch.cuda.empty_cache()
    got = r.fetch(sorted=True, device=False)        # the sorted fetch needs its own temporaries
    r.close()
    assert st["capacity"] < st0["capacity"]         # the buffer shrank under real pressure
    for x, y in zip(got, base):
        assert np.array_equal(x, y)


def test_overflow_store_spills_to_host(tds):
    """Overflow re-plan when the exact store cannot be allocated beside the pass
    buffer (the second large allocation fails): the kept records spill to host
    memory, the pass buffer is released, and the result equals the oracle's."""
    w = synth.random_1m(n_traj=300, query_frac_stride=10)
    d = 20.0
    idx = tds.Index(_cuda(w.D), kinds=tds.TEMPORAL, m=w.m_bins)
    base, _ = _run(idx, w.Q, d, "temporal")
    n0 = tds.test_inject_enomem(1, skip=1)          # pass buffer OK, exact store fails once
    got, st = _run(idx, w.Q, d, "temporal", capacity=len(base[0]) // 3)
    assert tds.test_inject_enomem(0) == n0 + 1
    assert st["passes"] > 1
    for x, y in zip(got, base):
        assert np.array_equal(x, y)
    ref = oracle.search(w.D, w.Q[:400], d)
    sel = got[0] < 400
    check(tuple(x[sel] for x in got), ref, w.D, w.Q[:400], d, label="spill to host")


@pytest.mark.parametrize("kind", KINDS)
def test_stationary_queries(tds, kind):
    """Stationary-point queries (case (i)): the range kernel's
    stationary filter (groups whose queries all have P1 = P0) returns the oracle's
    result, and the same records as the general filter (TDS_NO_STATIC=1)."""
    import os
    w = synth.random_dense(n_particles=4096, n_timesteps=25, n_query_traj=16)
    Q = synth.stationary_queries(w.D, 64, 3)
    assert np.array_equal(Q[:, 0:3], Q[:, 4:7])
    d = 0.02
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=(16, 16, 16))
    got, st = _run(idx, Q, d, kind)
    check(got, oracle.search(w.D, Q, d), w.D, Q, d, label=f"stationary {kind}")
    os.environ["TDS_NO_STATIC"] = "1"
    try:
        gen, _ = _run(idx, Q, d, kind)
    finally:
        del os.environ["TDS_NO_STATIC"]
    for x, y in zip(got, gen):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("pinned", [True, False])
def test_search_stream_equals_search(tds, kind, pinned):
    """tds_search_stream (host queries in chunks, copies overlapped, host-resident
    result) returns exactly the records of tds_search, with query ids
    of the full set, for ragged chunk sizes; fetches of ranges and sorted fetches
    work on the host-resident result; the oracle agrees."""
    import torch
    w = synth.random_dense(n_particles=2048, n_timesteps=25, n_query_traj=64)
    d = 0.02
    idx = tds.Index(_cuda(w.D), kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=(16, 16, 16))
    base = idx.search(_cuda(w.Q), d, kind=kind).fetch(sorted=True, device=False)
    Qh = torch.from_numpy(w.Q)
    Qh = Qh.pin_memory() if pinned else Qh
    for chunk in (w.Q.shape[0], 997, 128):
        r = idx.search_stream(Qh, d, kind=kind, chunk=chunk)
        assert r.count == len(base[0])
        got = r.fetch(sorted=True, device=False)
        for x, y in zip(got, base):
            assert np.array_equal(x, y)
        part = r.fetch(device=False, first=5, count=50)          # unsorted host range
        allr = r.fetch(device=False)
        for x, y in zip(part, allr):
            assert np.array_equal(x, y[5:55])
        hr = np.concatenate(r.host_records())                   # zero-copy blocks
        assert np.array_equal(hr["qid"], allr[0]) and np.array_equal(hr["t_out"], allr[3])
        r.close()
    check(got, oracle.search(w.D, w.Q, d), w.D, w.Q, d, label=f"stream {kind}")

"""Pins for the trajectory-level answer (oracle.merge_trajectories): hand-worked
cases and properties against a time-sampled union of the segment intervals."""
import numpy as np

import oracle
import synth


def test_crossing_over_a_segment_boundary_is_one_interval():
    # q: trajectory moving along x through (0,0,0) at t=5, polyline with a vertex at t=5
    # e: trajectory fixed at the origin over [0,10] in two segments [0,5], [5,10]
    Q = np.array([[-5, 0, 0, 0, 0, 0, 0, 5], [0, 0, 0, 5, 5, 0, 0, 10]], np.float32)
    D = np.array([[0, 0, 0, 0, 0, 0, 0, 5], [0, 0, 0, 5, 0, 0, 0, 10]], np.float32)
    r = oracle.search(D, Q, 1.0)
    h = r["hit"]
    # segment level: [4,5] for (q0,e0) and [5,6] for (q1,e1); (q0,e1), (q1,e0) only touch at t=5 (C5)
    assert sorted(zip(r["qid"][h].tolist(), r["eid"][h].tolist())) == [(0, 0), (1, 1)]
    m = oracle.merge_trajectories(r["qid"][h], r["eid"][h], r["t_in"][h], r["t_out"][h], [7, 7], [3, 3])
    assert m["qtraj"].tolist() == [7] and m["etraj"].tolist() == [3]
    assert (m["t_in"][0], m["t_out"][0]) == (4.0, 6.0)


def test_separate_contacts_stay_separate_and_gap_merges():
    qid = [0, 0, 0, 1]
    eid = [0, 1, 2, 0]
    t_in = [1.0, 2.5, 4.0, 1.5]
    t_out = [2.0, 3.0, 4.5, 1.7]
    qt, et = [10, 11], [20, 20, 21]
    m = oracle.merge_trajectories(qid, eid, t_in, t_out, qt, et)
    got = list(zip(m["qtraj"].tolist(), m["etraj"].tolist(), m["t_in"].tolist(), m["t_out"].tolist()))
    assert got == [(10, 20, 1.0, 2.0), (10, 20, 2.5, 3.0), (10, 21, 4.0, 4.5), (11, 20, 1.5, 1.7)]
    m2 = oracle.merge_trajectories(qid, eid, t_in, t_out, qt, et, gap=0.5)
    assert list(zip(m2["t_in"].tolist(), m2["t_out"].tolist()))[:2] == [(1.0, 3.0), (4.0, 4.5)]


def test_merge_equals_sampled_union():
    w = synth.tiny()
    r = oracle.search(w.D, w.Q, w.d)
    h = r["hit"]
    m = oracle.merge_trajectories(r["qid"][h], r["eid"][h], r["t_in"][h], r["t_out"][h], w.traj_Q, w.traj_D)
    # maximal, disjoint, sorted
    key = m["qtraj"] * 100000 + m["etraj"]
    same = key[1:] == key[:-1]
    assert np.all(m["t_in"][1:][same] > m["t_out"][:-1][same])
    # the union covers exactly the sampled times covered by the segment intervals
    ts = np.linspace(0, 30, 6001)
    for qt_, et_ in set(zip(m["qtraj"].tolist(), m["etraj"].tolist())):
        sel = (w.traj_Q[r["qid"][h]] == qt_) & (w.traj_D[r["eid"][h]] == et_)
        cov_seg = np.zeros_like(ts, bool)
        for a, b in zip(r["t_in"][h][sel], r["t_out"][h][sel]):
            cov_seg |= (ts >= a) & (ts <= b)
        ms = (m["qtraj"] == qt_) & (m["etraj"] == et_)
        cov_m = np.zeros_like(ts, bool)
        for a, b in zip(m["t_in"][ms], m["t_out"][ms]):
            cov_m |= (ts >= a) & (ts <= b)
        assert np.array_equal(cov_seg, cov_m)

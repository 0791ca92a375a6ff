"""A/B of the stationary-query filter: pair-kernel time of a search
of stationary-point queries against Random-dense-shaped D, with the stationary
filter (default) and with the general filter (TDS_NO_STATIC=1).
python tools/ab_static.py [n_points] [steps] [d]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1410_2698_b200 as tds  # noqa: E402
import synth  # noqa: E402

n_points = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
d = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
w = synth.random_dense()
Q = torch.from_numpy(synth.stationary_queries(w.D, n_points, steps)).cuda()
idx = tds.Index(torch.from_numpy(w.D).cuda(), kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=w.m_bins, v=w.v_subbins)
for kind in ("temporal", "spatiotemporal"):
    res = {}
    for mode in ("static", "general"):
        if mode == "general":
            os.environ["TDS_NO_STATIC"] = "1"
        ms = []
        for it in range(8):
            r = idx.search(Q, d, kind=kind)
            st = r.stats()
            r.close()
            if it >= 3:
                ms.append(st["ms_pairs"])
        os.environ.pop("TDS_NO_STATIC", None)
        res[mode] = (statistics.median(ms), st["pair_tests"], st["pairs_executed"], st["n_results"])
    print(f"{kind}: stationary filter {res['static'][0]:.3f} ms, general filter {res['general'][0]:.3f} ms "
          f"(pair tests {res['static'][1]}, executed {res['static'][2]}, results {res['static'][3]}, "
          f"same: {res['static'][3] == res['general'][3]})", flush=True)

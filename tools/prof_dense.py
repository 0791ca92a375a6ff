"""Random-dense at a large d on a query subset (for ncu of the output-bound path):
python tools/prof_dense.py [d] [nq] [kind]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1410_2698_b200 as tds  # noqa: E402
import synth  # noqa: E402

d = float(sys.argv[1]) if len(sys.argv) > 1 else 0.09
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
kind = sys.argv[3] if len(sys.argv) > 3 else "temporal"
w = synth.make_workload("random-dense")
D = torch.from_numpy(w.D).cuda()
Q = torch.from_numpy(w.Q[:nq]).cuda()
idx = tds.Index(D, kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=w.m_bins, v=w.v_subbins)
for it in range(6):
    r = idx.search(Q, d, kind=kind)
    st = r.stats()
    print(it, r.count, {k: st[k] for k in ("ms_pairs", "pair_tests", "refined_pairs", "passes")}, flush=True)
    r.close()

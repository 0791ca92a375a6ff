"""Small end-to-end run for compute-sanitizer: build + the three variants + overflow + sorted fetch."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import synth, paper_1410_2698_b200 as tds
w = synth.tiny()
D = torch.from_numpy(w.D).cuda(); Q = torch.from_numpy(w.Q).cuda()
idx = tds.Index(D, kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
tot = 0
for kind in ("temporal", "spatiotemporal", "spatial"):
    for cap in (0, 50):
        r = idx.search(Q, w.d, kind=kind, capacity=cap)
        q, e, ti, to = r.fetch(sorted=True, device=False)
        tot += r.count
        r.close()
torch.cuda.synchronize()
print("sanitize smoke ok", tot)

"""Print the records that fail parity at full size (diagnostic)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import oracle, synth, paper_1410_2698_b200 as tds
from parity import keys
d = float(sys.argv[1]) if len(sys.argv) > 1 else 0.09
kind = sys.argv[2] if len(sys.argv) > 2 else "spatiotemporal"
w = synth.random_dense()
rng = np.random.default_rng(int(d * 1000))
sel = np.sort(rng.choice(w.Q.shape[0], 96, replace=False))
ref = oracle.search(w.D, w.Q, d, qsel=sel)
idx = tds.Index(torch.from_numpy(w.D).cuda(), kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=w.m_bins, v=w.v_subbins)
Qd = torch.from_numpy(w.Q).cuda()
r = idx.search(Qd, d, kind=kind)
q, e, ti, to = r.fetch(device=True)
lut = torch.zeros(w.Q.shape[0], dtype=torch.bool, device='cuda'); lut[torch.as_tensor(sel, device='cuda')] = True
m = lut[q]
g = [x[m].cpu().numpy() for x in (q, e, ti, to)]
gk = keys(g[0], g[1]); o = np.argsort(gk)
want = ref['hit'] & (np.abs(ref['dmin'] - d) > 1e-5 * d)
rk = keys(ref['qid'], ref['eid'])[want]
pos = np.searchsorted(gk[o], rk)
gi, go = g[2][o][pos].astype(np.float64), g[3][o][pos].astype(np.float64)
ri, ro = ref['t_in'][want], ref['t_out'][want]
qi, ei = ref['qid'][want], ref['eid'][want]
a = np.maximum(w.Q[qi, 3], w.D[ei, 3]).astype(np.float64); b = np.minimum(w.Q[qi, 7], w.D[ei, 7]).astype(np.float64)
tol_i = 1e-5 * np.maximum(np.abs(ri), b - a); tol_o = 1e-5 * np.maximum(np.abs(ro), b - a)
bad = (np.abs(gi - ri) > tol_i) | (np.abs(go - ro) > tol_o)
print("n checked", want.sum(), "bad", bad.sum())
for k in np.nonzero(bad)[0][:5]:
    print("q", qi[k], w.Q[qi[k]].tolist()); print("e", ei[k], w.D[ei[k]].tolist())
    print("ref", ri[k], ro[k], "gpu", gi[k], go[k], "dmin", ref['dmin'][want][k], "a,b", a[k], b[k])
    np.save('gpurun_out/badpair.npy', np.stack([w.Q[qi[k]], w.D[ei[k]]]))

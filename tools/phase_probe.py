import sys, time, json
sys.path.insert(0, '.')
import torch, numpy as np, synth, paper_1410_2698_b200 as tds
w = synth.random_dense(d=0.01)
D = torch.from_numpy(w.D).cuda(); Q = torch.from_numpy(w.Q).cuda()
cap = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for step in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    idx = tds.Index(D, kinds=tds.TEMPORAL | tds.SPATIOTEMPORAL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    out = []
    for kind in ("temporal", "spatiotemporal"):
        ta = time.perf_counter()
        r = idx.search(Q, w.d, kind=kind, capacity=cap)
        tb = time.perf_counter()
        f = r.fetch(); torch.cuda.synchronize(); tc = time.perf_counter()
        st = r.stats(); r.close()
        out.append((kind, round(1e3*(tb-ta),2), round(1e3*(tc-tb),2), round(st['ms_total'],2), round(st['ms_pairs'],2), round(st['ms_schedule'],2)))
    idx.close(); torch.cuda.synchronize()
    print(step, 'build', round(1e3*(t1-t0),2), out, flush=True)

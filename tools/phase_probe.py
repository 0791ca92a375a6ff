"""Per-phase timing of build / search / fetch (host wall clock + library CUDA-event stats)."""
import argparse
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1410_2698_b200 as tds  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="random-1m")
ap.add_argument("--d", type=float, default=None)
ap.add_argument("--cap", type=int, default=0)
ap.add_argument("--kinds", default="temporal,spatiotemporal,spatial")
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
w = synth.make_workload(a.config)
d = a.d if a.d is not None else w.d
D = torch.from_numpy(w.D).cuda()
Q = torch.from_numpy(w.Q).cuda()
kinds = a.kinds.split(",")
for step in range(a.steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    idx = tds.Index(D, kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out = []
    for kind in kinds:
        ta = time.perf_counter()
        r = idx.search(Q, d, kind=kind, capacity=a.cap)
        tb = time.perf_counter()
        r.fetch()
        torch.cuda.synchronize()
        tc = time.perf_counter()
        st = r.stats()
        r.close()
        out.append(f"{kind[:4]} host {1e3*(tb-ta):.3f} fetch {1e3*(tc-tb):.3f} | ev total {st['ms_total']:.3f} "
                   f"sched {st['ms_schedule']:.3f} pairs {st['ms_pairs']:.3f} compact {st['ms_compact']:.3f}")
    idx.close()
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    print(step, f"build {1e3*(t1-t0):.3f}", " || ".join(out),
          f"| torch reserved {torch.cuda.memory_reserved() / 1e9:.1f} GB, device free {free / 1e9:.1f} GB", flush=True)

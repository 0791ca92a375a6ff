"""Stall reasons by SASS region of one ncu source-page CSV (--print-source sass).
Usage: python tools/ncu_stall_regions.py <source.csv> [window_bytes=1024] [reasons=no_inst,long_sb,wait,short_sb,branch_resolving]"""
import collections
import csv
import sys

path = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reasons = (sys.argv[3] if len(sys.argv) > 3 else "no_inst,long_sb,wait,short_sb,branch_resolving,selected").split(",")
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
cols = {r: h.index("stall_" + r) for r in reasons}
itot = h.index("Warp Stall Sampling (All Samples)")
L = []
for r in rows[hi + 1:]:
    try:
        L.append((int(r[ia], 16), r[isrc], float(r[itot] or 0), float(r[iex] or 0),
                  {k: float(r[c] or 0) for k, c in cols.items()}))
    except (ValueError, IndexError):
        continue
base = min(x[0] for x in L)
tot = sum(x[2] for x in L) or 1
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter(), ""])
for a, src, st, ex, rs in L:
    w = (a - base) // win
    agg[w][0] += st
    agg[w][1] += ex
    agg[w][2].update(rs)
    if not agg[w][3]:
        agg[w][3] = src[:40]
allr = collections.Counter()
for a, src, st, ex, rs in L:
    allr.update(rs)
print("total (% of all samples):", " ".join(f"{k} {100 * v / tot:.1f}" for k, v in allr.items()))
print(f"{'offset':>7} {'all%':>6} " + " ".join(f"{k[:8]:>8}" for k in reasons) + "  first")
for w in sorted(agg):
    st, ex, rs, src = agg[w]
    if st / tot >= 0.01:
        print(f"{w * win:7x} {100 * st / tot:5.1f} " + " ".join(f"{100 * rs[k] / tot:8.1f}" for k in reasons) + "  " + src)

"""Hot spots of one ncu --page source --print-source sass CSV: warp-stall samples and
executed instructions per SASS line, aggregated by address window and by opcode.
Usage: python tools/ncu_sass_hot.py <source.csv> [window_bytes=256] [top=40]"""
import collections
import csv
import sys

path = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 256
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ia, isrc = h.index("Address"), h.index("Source")
ist = h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
lines = []
for r in rows[hi + 1:]:
    if len(r) <= max(ia, ist, iex):
        continue
    try:
        addr = int(r[ia], 16)
        st = float(r[ist] or 0)
        ex = float(r[iex] or 0)
    except ValueError:
        continue
    lines.append((addr, r[isrc].strip(), st, ex))
base = min(a for a, *_ in lines)
tot_st = sum(x[2] for x in lines) or 1
tot_ex = sum(x[3] for x in lines) or 1
print(f"{len(lines)} SASS lines, {tot_st:.0f} stall samples, {tot_ex:.3g} warp instructions executed")
byw = collections.defaultdict(lambda: [0.0, 0.0, ""])
for a, src, st, ex in lines:
    w = (a - base) // win
    byw[w][0] += st
    byw[w][1] += ex
    if not byw[w][2]:
        byw[w][2] = src[:60]
print(f"\n{'offset':>8} {'stall%':>7} {'inst%':>7}  first instruction (windows of {win} B with >= 0.5 % of either)")
for w in sorted(byw):
    st, ex, src = byw[w]
    if st / tot_st >= 0.005 or ex / tot_ex >= 0.005:
        print(f"{w * win:8x} {100 * st / tot_st:6.1f}% {100 * ex / tot_ex:6.1f}%  {src}")
byop = collections.defaultdict(lambda: [0.0, 0.0])
for a, src, st, ex in lines:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    byop[op][0] += st
    byop[op][1] += ex
print(f"\n{'opcode':>10} {'stall%':>7} {'inst%':>7}")
for op, (st, ex) in sorted(byop.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{op:>10} {100 * st / tot_st:6.1f}% {100 * ex / tot_ex:6.1f}%")
print(f"\ntop {top} lines by stall samples:")
for a, src, st, ex in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{a - base:8x} {100 * st / tot_st:5.1f}% ex {ex:10.3g}  {src[:80]}")

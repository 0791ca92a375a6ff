"""Warp-stall samples and executed warp instructions per CUDA source line of one
ncu capture (ncu -i <rep> --page source --csv --print-source cuda,sass):
python tools/ncu_lines.py <cuda_sass.csv> [top=45]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ist, iin = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
lines = []
for r in rows[hi + 1:]:
    if r and r[0]:
        try:
            lines.append((int(r[0]), r[1].strip()[:90], float(r[ist] or 0), float(r[iin] or 0)))
        except ValueError:
            pass
ts = sum(x[2] for x in lines) or 1
ti = sum(x[3] for x in lines) or 1
print(f"{len(lines)} source lines, {ts:.0f} stall samples, {ti:.3g} warp instructions")
print(f"{'line':>5} {'stall%':>6} {'inst%':>6}  source")
for ln, src, s, i in sorted(lines, key=lambda x: -(x[2] / ts + x[3] / ti))[:top]:
    print(f"{ln:5d} {100 * s / ts:6.2f} {100 * i / ti:6.2f}  {src}")

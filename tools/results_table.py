"""Markdown results table from committed bench lines:
python tools/results_table.py profiles/r1_v6_bench_*.json"""
import json
import sys

print("| workload (bench `--config`) | step ms (median / mean) | value: query answers/s | search-only q/s "
      "| dominant pair kernel | kernel ms | pair tests | results | roofline (bound: achieved / peak) |")
print("|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    c, b, r = d["config"], d["breakdown"], d["roofline"]
    v = b["variants"]
    dom = r["kernel"].split("(")[1].rstrip(")")
    x = v[dom]
    name = f"{c['workload']} d={c['d']:g} ({', '.join({'temporal': 'T', 'spatiotemporal': 'ST', 'spatial': 'S'}[k] for k in c['variants'])})"
    roof = f"{r['bound']}: {r['achieved']:.3g} / {r['peak']:.4g} {r['unit']} = **{100 * r['frac']:.1f} %**"
    print(f"| {name} | {b['step_ms_median']:.3g} / {d['ms_per_step']:.3g} | {d['value']:.3g} | "
          f"{d['search_only']['value']:.3g} | {r['kernel']} | {x['pair_kernel_ms']:.3g} | {x['pair_tests']:.3g} | "
          f"{x['results']:.3g} | {roof} |")

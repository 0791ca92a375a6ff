"""Markdown results table from committed bench lines (round-2 format: one row per
variant of each line): python tools/results_table.py profiles/r2_v1_bench_*.json"""
import json
import sys

ABBR = {"temporal": "T", "spatiotemporal": "ST", "spatial": "S"}
print("| workload | variant | T_search ms | query segments/s | pair kernel ms | scheduled pair tests "
      "| executed | records | fp64 share | §8(d) ALU frac | HBM frac |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    c, v, r = d["config"], d["breakdown"]["variants"], d["roofline"]
    for k, x in v.items():
        if k == c["headline_variant"]:
            alu, hbm = r["alu"]["frac"], r["hbm"]["frac"]
        else:
            alu, hbm = x["roofline"]["alu_frac"], x["roofline"]["hbm_frac"]
        f64 = x["refined_pairs_fp64"] / max(1, x["results"])
        print(f"| {c['workload']} d={c['d']:g} | {ABBR[k]} | {x['t_search_ms']:.3g} | {x['query_segments_per_s']:.3g} "
              f"| {x['pair_kernel_ms']:.3g} | {x['pair_tests']:.3g} | {x['pairs_executed']:.3g} | {x['results']:.3g} "
              f"| {100 * f64:.1f} % | {alu:.2f} | {hbm:.2f} |")

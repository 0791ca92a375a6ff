#!/bin/bash
# Pair-kernel and search times of the current build over the main configurations
# (GPU box): tools/kbench.sh [tag] [steps]
tag=${1:-kb}; steps=${2:-5}
out=gpurun_out/kb; mkdir -p $out
for cfg in "random-dense 0.01 spatiotemporal,temporal" "random-dense 0.03 spatiotemporal,temporal" \
           "random-dense 0.09 spatiotemporal,temporal" "merger 1 spatiotemporal,temporal,spatial" \
           "merger 5 spatiotemporal,temporal,spatial" "random-1m 50 spatiotemporal,temporal,spatial"; do
  set -- $cfg
  f=$out/${tag}_$1_$2.json
  timeout 900 python bench.py --config $1 --d $2 --variants $3 --steps $steps --warmup 3 --no-cpu-baseline --no-e2e \
      > $f 2> ${f%.json}.err
  python - "$f" "$1 d=$2" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    v = d["breakdown"]["variants"]
    print(f"{sys.argv[2]:18s}", " | ".join(f"{k[:6]} search {x['t_search_ms']:.3f} kern {x['pair_kernel_ms']:.3f} fp64 {x['refined_pairs_fp64']}" for k, x in v.items()),
          f"| frac {d['roofline']['frac']:.3f} ({d['roofline']['bound']})", flush=True)
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done

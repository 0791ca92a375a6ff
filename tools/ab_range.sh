#!/bin/bash
# A/B of the range kernels (TDS_RANGE_OLD=1: round-1 lane-per-candidate kernel;
# default: broadcast-candidate kernel): pair-kernel ms per workload / variant.
#   tools/ab_range.sh [steps]
steps=${1:-5}
out=gpurun_out/ab; mkdir -p $out
for cfg in "random-dense 0.01" "random-dense 0.03" "random-dense 0.09" "merger 1" "merger 5" "random-1m 50"; do
  set -- $cfg
  for old in 1 0; do
    TDS_RANGE_OLD=$old timeout 900 python bench.py --config $1 --d $2 --variants spatiotemporal,temporal --steps $steps \
        --warmup 3 --no-cpu-baseline --no-e2e > $out/ab_$1_$2_$old.json 2> $out/ab_$1_$2_$old.err
    python - "$out/ab_$1_$2_$old.json" "$1 d=$2 old=$old" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    v = d["breakdown"]["variants"]
    print(sys.argv[2], " ".join(f"{k}: search {x['t_search_ms']:.3f} kernel {x['pair_kernel_ms']:.3f} res {x['results']} fp64 {x['refined_pairs_fp64']}" for k, x in v.items()),
          f"frac {d['roofline']['frac']:.3f} ({d['roofline']['bound']})", flush=True)
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  done
done

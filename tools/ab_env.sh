#!/bin/bash
# Interleaved A/B over (library, environment) arms on chosen configurations:
#   tools/ab_env.sh "<cfg> <d> <variants>;..." "name|lib|ENV=V ENV2=V" ...   (lib relative to paper_1410_2698_b200/)
# prints the pair-kernel ms per variant (2 rounds, interleaved)
cfgs=$1; shift
out=gpurun_out/abe; mkdir -p $out
IFS=';' read -ra CF <<< "$cfgs"
for rep in 1 2; do
for c in "${CF[@]}"; do
  read -r cfg d var <<< "$c"
  for arm in "$@"; do
    IFS='|' read -r name lib envs <<< "$arm"
    f=$out/${name}_${cfg}_${d}_$rep.json
    env TDS_LIB=$PWD/paper_1410_2698_b200/$lib $envs timeout 600 python bench.py --config $cfg --d $d --variants $var \
        --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $f 2> ${f%.json}.err
    python - "$f" "$name $cfg d=$d r$rep" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    v = d["breakdown"]["variants"]
    print(f"{sys.argv[2]:42s}", " | ".join(f"{k[:6]} kern {x['pair_kernel_ms']:.3f} fp64 {x['refined_pairs_fp64']:.3g}" for k, x in v.items()), flush=True)
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  done
done
done

#!/bin/bash
# Interleaved A/B of library builds (TDS_LIB) on chosen configurations:
#   tools/ab_libs2.sh "<cfg> <d> <variants>;..." lib1 lib2 ...   (libs relative to paper_1410_2698_b200/)
cfgs=$1; shift
out=gpurun_out/ab2; mkdir -p $out
IFS=';' read -ra CF <<< "$cfgs"
for rep in 1 2; do
for c in "${CF[@]}"; do
  set -- $c "$@"
  cfg=$1 d=$2 var=$3; shift 3
  for lib in "$@"; do
    f=$out/${lib%.so}_${cfg}_${d}_$rep.json
    TDS_LIB=$PWD/paper_1410_2698_b200/$lib timeout 600 python bench.py --config $cfg --d $d --variants $var --steps 10 --warmup 3 \
        --no-cpu-baseline --no-e2e > $f 2> ${f%.json}.err
    python - "$f" "$lib $cfg d=$d r$rep" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    v = d["breakdown"]["variants"]
    print(f"{sys.argv[2]:40s}", " | ".join(f"{k[:6]} kern {x['pair_kernel_ms']:.3f}" for k, x in v.items()), flush=True)
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  done
done
done

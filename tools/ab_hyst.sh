#!/bin/bash
# Dense-window hysteresis sweep (TDS_HYST_HI / TDS_HYST_LO, % of a window's
# evaluated pairs passing the filter): pair-kernel ms of GPUTemporal /
# GPUSpatioTemporal on Random-dense-shaped over d.   tools/ab_hyst.sh
out=gpurun_out/ab; mkdir -p $out
for hl in "50 25" "25 12" "15 8" "10 5" "6 3"; do
  set -- $hl
  for d in 0.01 0.03 0.05 0.09; do
    TDS_HYST_HI=$1 TDS_HYST_LO=$2 timeout 300 python bench.py --d $d --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
        > $out/hyst_$1_$d.json 2>/dev/null
    python -c "
import json,sys
d=json.loads(open('$out/hyst_$1_$d.json').read().strip().splitlines()[-1]);v=d['breakdown']['variants']
print('hyst $1/$2 d=$d', ' '.join(f'{k} {x[\"pair_kernel_ms\"]:.3f}' for k,x in v.items()))" 2>/dev/null || echo "hyst $1/$2 d=$d FAILED"
  done
done

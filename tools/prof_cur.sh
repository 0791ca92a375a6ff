#!/bin/bash
# ncu --set full (+ source page) of the range kernel at Random-dense d = 0.03 / 0.09 (GPUTemporal)
# and of the spatial kernel at Merger d = 1, current build.  tools/prof_cur.sh <tag>
set -u
tag=${1:-cur}
out=gpurun_out/prof; mkdir -p $out
ncu_one() {
  local name=$1 skip=$2 kern=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kern -c 1 --launch-skip $skip \
      -o $out/$name -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/$name.log 2>&1
  ncu -i $out/$name.ncu-rep --page details --csv > $out/$name.details.csv 2>/dev/null
  ncu -i $out/$name.ncu-rep --page raw --csv > $out/$name.raw.csv 2>/dev/null
  ncu -i $out/$name.ncu-rep --page source --csv --print-source sass > $out/$name.source.csv 2>/dev/null
  rm -f $out/$name.ncu-rep
}
ncu_one ${tag}_ncu_rdense003_t 3 k_pair_range --d 0.03 --variants temporal
ncu_one ${tag}_ncu_rdense009_t 3 k_pair_range --d 0.09 --variants temporal
ncu_one ${tag}_ncu_rdense003_st 3 k_pair_range --d 0.03 --variants spatiotemporal
ncu_one ${tag}_ncu_merger1_spatial 3 k_pair_range --config merger --d 1 --variants spatial

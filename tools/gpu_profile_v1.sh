#!/bin/bash
# round-2 evidence pass: bench lines, the default bench's launch list, ncu --set full of
# the headline pair kernel (Random-dense d=0.03 ST and T, d=0.09 T) and single-pass DRAM bytes
set -u
tag=${1:-r2_v1}
out=gpurun_out/prof; mkdir -p $out
tools/profile_r2.sh $tag bench launches
ncu_one() {
  local name=$1 skip=$2 kern=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kern -c 1 --launch-skip $skip \
      -o $out/${tag}_ncu_$name -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/${tag}_ncu_$name.log 2>&1
  ncu -i $out/${tag}_ncu_$name.ncu-rep --page details --csv > $out/${tag}_ncu_$name.details.csv 2>/dev/null
  ncu -i $out/${tag}_ncu_$name.ncu-rep --page raw --csv > $out/${tag}_ncu_$name.raw.csv 2>/dev/null
  ncu -i $out/${tag}_ncu_$name.ncu-rep --page source --csv --print-source sass > $out/${tag}_ncu_$name.source.csv 2>/dev/null
  rm -f $out/${tag}_ncu_$name.ncu-rep
}
ncu_one rdense003_st 3 k_pair_range --variants spatiotemporal
ncu_one rdense003_t 3 k_pair_range --variants temporal
ncu_one rdense009_t 3 k_pair_range --d 0.09 --variants temporal
for v in spatiotemporal temporal; do for d in 0.03 0.09; do tools/ncu_dram.sh $d $v random-dense; done; done
tools/ncu_dram.sh 1 spatial merger
ls -la $out | head -80

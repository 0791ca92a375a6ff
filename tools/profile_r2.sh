#!/bin/bash
# Round-2 evidence on the GPU box (one GPU): bench lines, the launch list of the
# default bench, and ncu --set full (with the source page) of the dominant pair
# kernels.  Outputs under gpurun_out/prof/ (summaries are copied to profiles/).
#   tools/profile_r2.sh [tag] [what...]   what = bench | launches | ncu | dram | all (default)
set -u
tag=${1:-r2}; shift || true
what=${*:-all}
out=gpurun_out/prof; mkdir -p $out
has() { [[ " $what " == *" all "* || " $what " == *" $1 "* ]]; }
run() { local name=$1; shift; timeout 600 python bench.py "$@" > $out/${tag}_bench_$name.json 2> $out/${tag}_bench_$name.err;
        tail -1 $out/${tag}_bench_$name.json | cut -c1-160; }
ncu_one() {   # name skip kernel-regex bench-args...
  local name=$1 skip=$2 kern=$3; shift 3
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$kern -c 1 --launch-skip $skip \
      -o $out/${tag}_ncu_$name -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
      > $out/${tag}_ncu_$name.log 2>&1
  ncu -i $out/${tag}_ncu_$name.ncu-rep --page details --csv > $out/${tag}_ncu_$name.details.csv 2>/dev/null
  ncu -i $out/${tag}_ncu_$name.ncu-rep --page raw --csv > $out/${tag}_ncu_$name.raw.csv 2>/dev/null
  ncu -i $out/${tag}_ncu_$name.ncu-rep --page source --csv --print-source sass > $out/${tag}_ncu_$name.source.csv 2>/dev/null
  rm -f $out/${tag}_ncu_$name.ncu-rep
}
if has bench; then
  run rdense_0.03 --steps 20
  run rdense_0.01 --d 0.01 --steps 10 --no-cpu-baseline --no-e2e
  run rdense_0.09 --d 0.09 --steps 5 --no-cpu-baseline --no-e2e
  run merger_1 --config merger --steps 5 --no-cpu-baseline --no-e2e
  run merger_5 --config merger --d 5 --steps 3 --no-cpu-baseline --no-e2e
  run random1m --config random-1m --steps 20 --no-cpu-baseline --no-e2e
fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches_rdense003.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/ncu_launches.py $out/${tag}_launches_rdense003.csv > $out/${tag}_launches_rdense003.txt
fi
if has ncu; then
  # bench order per step: GPUSpatioTemporal then GPUTemporal; 3 warm-up steps -> the timed
  # step's launches are the 7th (ST) and 8th (T) range-kernel launches
  ncu_one rdense003_st 6 k_pair_range
  ncu_one rdense003_t 7 k_pair_range
  ncu_one rdense009_t 7 k_pair_range --d 0.09
  ncu_one rdense001_t 7 k_pair_range --d 0.01
  ncu_one merger1_spatial 2 k_pair_range --config merger --variants spatial
  ncu_one merger5_spatial 2 k_pair_range --config merger --d 5 --variants spatial
  ncu_one merger5_st 2 k_pair_range --config merger --d 5 --variants spatiotemporal
fi
if has dram; then   # single-pass DRAM bytes at the full bench configurations -> profiles/ncu_traffic.json
  for v in spatiotemporal temporal; do for d in 0.01 0.03 0.09; do tools/ncu_dram.sh $d $v random-dense; done; done
  for v in spatiotemporal temporal spatial; do tools/ncu_dram.sh 1 $v merger; tools/ncu_dram.sh 5 $v merger; done
  for v in spatiotemporal temporal spatial; do tools/ncu_dram.sh 50 $v random-1m; done
fi
ls $out | head -100

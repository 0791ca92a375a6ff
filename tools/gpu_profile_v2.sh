#!/bin/bash
# round-2 evidence pass: bench lines, the default bench's launch list, ncu --set full of the
# headline pair kernel (kept as .ncu-rep for the source view) and single-pass DRAM bytes
set -u
tag=${1:-r2_v8}
out=gpurun_out/prof; mkdir -p $out gpurun_out/rep
tools/profile_r2.sh $tag bench launches
for a in "rdense003_st --variants spatiotemporal" "rdense009_t --d 0.09 --variants temporal" "merger1_s --config merger --d 1 --variants spatial"; do
  set -- $a; n=$1; shift
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair_range -c 1 --launch-skip 3 \
      -o gpurun_out/rep/${tag}_$n -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/rep/${tag}_$n.log 2>&1
done
for v in spatiotemporal temporal; do for d in 0.01 0.03 0.09; do tools/ncu_dram.sh $d $v random-dense; done; done
tools/ncu_dram.sh 1 spatial merger; tools/ncu_dram.sh 1 spatiotemporal merger
ls $out gpurun_out/rep | head -80

#!/bin/bash
# ncu --set full capture of one range-kernel launch, the .ncu-rep kept (read locally with
# ncu -i ... --page source --print-source cuda,sass).  tools/ncu_rep.sh <name> <bench args...>
set -u
name=$1; shift
out=gpurun_out/rep; mkdir -p $out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair_range -c 1 --launch-skip 3 \
    -o $out/$name -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/$name.log 2>&1
ls -la $out/$name.ncu-rep

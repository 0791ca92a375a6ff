#!/bin/bash
# One ncu --set full capture of the first timed k_pair_range launch of a bench
# configuration (run on the GPU box): tools/ncu_pair.sh <name> <bench args...>
name=$1; shift
ncu --set full --import-source on --clock-control none -k regex:k_pair_range -c 1 --launch-skip 4 \
    -o gpurun_out/ncu_$name -f python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e "$@" \
    > gpurun_out/ncu_$name.log 2>&1
ncu -i gpurun_out/ncu_$name.ncu-rep --page details --csv > gpurun_out/ncu_$name.details.csv 2>/dev/null
ncu -i gpurun_out/ncu_$name.ncu-rep --page source --csv > gpurun_out/ncu_$name.source.csv 2>/dev/null
ncu -i gpurun_out/ncu_$name.ncu-rep --page raw --csv > gpurun_out/ncu_$name.raw.csv 2>/dev/null

#!/bin/bash
# DRAM bytes of the range kernel at a full bench configuration (single-pass metrics,
# no replay of the multi-GB output buffers): tools/ncu_dram.sh <d> <variant>
d=$1; var=$2; out=gpurun_out/dram_${d}_${var}
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_pair_range -c 1 --launch-skip 2 --csv --page raw --log-file $out.csv \
    python bench.py --config random-dense --d $d --variants $var --steps 1 --warmup 2 --no-cpu-baseline --no-e2e \
    > $out.log 2>&1
tail -3 $out.csv

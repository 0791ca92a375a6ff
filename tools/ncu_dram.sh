#!/bin/bash
# DRAM bytes of the range kernel at a full bench configuration (single-pass metrics,
# no replay of the multi-GB output buffers):
#   tools/ncu_dram.sh <d|default> <variant> [config=random-dense] [tag]
# then: python tools/ncu_traffic.py gpurun_out/dram_<config>_<d>_<variant>.csv <config> <d> k_pair_range <variant>
d=$1; var=$2; cfg=${3:-random-dense}; out=gpurun_out/dram_${cfg}_${d}_${var}
darg=(); [[ $d != default ]] && darg=(--d $d)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_pair_range -c 1 --launch-skip 2 --csv --page raw --log-file $out.csv \
    python bench.py --config $cfg "${darg[@]}" --variants $var --steps 1 --warmup 2 --no-cpu-baseline --no-e2e \
    > $out.log 2>&1
tail -3 $out.csv
python tools/ncu_traffic.py $out.csv $cfg $d k_pair_range $var

#!/bin/bash
# Round evidence on the GPU box: bench lines for every workload, the launch list of
# the default bench, ncu --set full of the dominant pair kernel.  Outputs under
# gpurun_out/prof/ (copy the summaries to profiles/ afterwards).
set -u
out=gpurun_out/prof; mkdir -p $out
run() { local name=$1; shift; timeout 1200 python bench.py "$@" > $out/bench_$name.json 2> $out/bench_$name.err; tail -1 $out/bench_$name.json | cut -c1-200; }
run random1m
run rdense_0.01 --config random-dense --d 0.01 --variants temporal,spatiotemporal --steps 10 --no-cpu-baseline
run rdense_0.03 --config random-dense --d 0.03 --variants temporal,spatiotemporal --steps 10 --no-cpu-baseline
run rdense_0.09 --config random-dense --d 0.09 --variants temporal,spatiotemporal --steps 5 --no-cpu-baseline --no-e2e
run merger_1 --config merger --steps 5 --no-cpu-baseline
run scaleout --config scale-out --variants temporal,spatiotemporal --steps 2 --warmup 3 --no-cpu-baseline --no-e2e
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_random1m.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_launches.py $out/launches_random1m.csv > $out/launches_random1m.txt
for spec in "random1m_temporal --variants temporal" "rdense01_temporal --config random-dense --d 0.01 --variants temporal" \
            "merger1_spatial --config merger --variants spatial"; do
  set -- $spec; name=$1; shift
  kern=k_pair_range; [[ $name == *spatial ]] && kern=k_pair_spatial
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kern -c 1 --launch-skip 4 \
      -o $out/ncu_$name -f python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e "$@" > $out/ncu_$name.log 2>&1
  ncu -i $out/ncu_$name.ncu-rep --page details --csv > $out/ncu_$name.details.csv 2>/dev/null
  ncu -i $out/ncu_$name.ncu-rep --page raw --csv > $out/ncu_$name.raw.csv 2>/dev/null
  rm -f $out/ncu_$name.ncu-rep
done
# output-bound range kernel on a query subsample (tools/prof_dense.py), with the source page
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair_range -c 1 --launch-skip 3 \
    -o $out/ncu_rdense09_temporal -f python tools/prof_dense.py 0.09 5000 temporal > $out/ncu_rdense09_temporal.log 2>&1
ncu -i $out/ncu_rdense09_temporal.ncu-rep --page details --csv > $out/ncu_rdense09_temporal.details.csv 2>/dev/null
ncu -i $out/ncu_rdense09_temporal.ncu-rep --page raw --csv > $out/ncu_rdense09_temporal.raw.csv 2>/dev/null
ncu -i $out/ncu_rdense09_temporal.ncu-rep --page source --csv > $out/ncu_rdense09_temporal.source.csv 2>/dev/null
rm -f $out/ncu_rdense09_temporal.ncu-rep
ls $out

#!/bin/bash
# A/B of library builds on the GPUSpatial workloads: tools/ab_spatial.sh libA.so libB.so
for i in 1 2; do
for lib in "$@"; do
  for cfg in "--config random-1m --steps 30" "--config merger --variants spatial --steps 5" "--config merger --d 5 --variants spatial --steps 3"; do
    TDS_LIB=paper_1410_2698_b200/$lib python bench.py $cfg --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || { tail -2 gpurun_out/ab.err; continue; }
    python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', '$cfg'.split()[1], d['config']['d'], round(d['breakdown']['step_ms_median'],3), 'build', round(d['breakdown']['build_index_ms'],3), {k:round(v['pair_kernel_ms'],3) for k,v in d['breakdown']['variants'].items()})"
  done
done
done

#!/bin/bash
# A/B of library builds across the hit density of Random-dense: tools/ab_density.sh libA.so libB.so ...
for lib in "$@"; do
  for d in ${DS:-0.02 0.03 0.05 0.07 0.09}; do
    TDS_LIB=paper_1410_2698_b200/$lib python bench.py --config random-dense --d $d --variants temporal,spatiotemporal --steps 4 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || { tail -2 gpurun_out/ab.err; continue; }
    python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', d['config']['d'], {k:round(v['pair_kernel_ms'],3) for k,v in d['breakdown']['variants'].items()})"
  done
done

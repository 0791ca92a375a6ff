#!/bin/bash
# quick pair-kernel comparison on the three main workloads (GPU box)
for cfg in "--config random-1m" "--config random-dense --d 0.01 --variants temporal,spatiotemporal --steps 10" "--config merger --variants temporal,spatiotemporal --steps 5" "$@"; do
  [ -z "$cfg" ] && continue
  python bench.py $cfg --no-cpu-baseline --no-e2e > gpurun_out/qb.json 2>gpurun_out/qb.err || { tail -3 gpurun_out/qb.err; continue; }
  python -c "
import json
d=json.loads(open('gpurun_out/qb.json').read().strip().splitlines()[-1])
print('$cfg'.split()[1], round(d['ms_per_step'],3), round(d['roofline']['frac'],3), {k:round(v['pair_kernel_ms'],4) for k,v in d['breakdown']['variants'].items()})"
done

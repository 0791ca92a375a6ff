for i in 1 2; do
for lib in libtds.so libtds_bps3.so; do
  for cfg in "--config random-1m" "--config random-dense --d 0.01 --variants temporal,spatiotemporal --steps 10"; do
    TDS_LIB=paper_1410_2698_b200/$lib python bench.py $cfg --no-cpu-baseline --no-e2e > gpurun_out/c.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/c.json').read().strip().splitlines()[-1])
print('$lib', '$cfg'.split()[1], round(d['ms_per_step'],3), {k:round(v['pair_kernel_ms'],4) for k,v in d['breakdown']['variants'].items()})"
  done
done
done

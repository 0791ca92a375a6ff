# T_search A/B (bench t_search_ms) for two libs
for rep in 1 2; do for lib in d w; do
  TDS_LIB=$PWD/paper_1410_2698_b200/libtds_$lib.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ts_$lib.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ts_$lib.json').read().strip().splitlines()[-1]); print('$lib', {k:(round(v['t_search_ms'],4), round(v['pair_kernel_ms'],4), round(v['ms_schedule'],4)) for k,v in d['breakdown']['variants'].items()})"
done; done

#!/bin/bash
for v in T0 T1 T2; do
  RAS_LIB_PATH=$PWD/variants/lib_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_$v.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/var_$v.json')); print('$v', round(d['ms_per_step'],3), round(d['kernel_pass_ms_per_step'],3), ' '.join(k+':'+str(round(v['avg_us'],1)) for k,v in d['kernels'].items()))"
done

#!/bin/bash
# RESIDENT path variants on C2, interleaved for a fair same-box comparison
for v in "$@"; do
  RAS_LIB_PATH=$PWD/variants/lib_$v.so timeout -s KILL 200 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k:(v['launches'],round(v['avg_us'],1)) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/var_$v.err
done

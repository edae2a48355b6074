#!/bin/bash
# TILED path variants on C2 (forced TILED), interleaved for a same-box comparison
for v in "$@"; do
  RAS_LIB_PATH=$PWD/variants/lib_$v.so timeout -s KILL 200 python bench.py --path tiled --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-tts > gpurun_out/tvar_$v.json 2>gpurun_out/tvar_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/tvar_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k:(v['launches'],round(v['avg_us'],1)) for k,v in d['kernels'].items()})" || tail -3 gpurun_out/tvar_$v.err
done

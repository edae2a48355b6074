#!/bin/bash
# k_trsv_pf chunk-size variants (same box): one 256^3 subdomain IC(0) to 1e-8, and the
# 2x2x2 256^3 per-level time with k_trsv_pf forced
for v in "$@"; do
  RAS_LIB_PATH=$PWD/variants/lib_$v.so timeout 300 python tools/c4_run.py --grid 256 256 256 --parts 1 1 1 --solvers ic0:10 --modes sync > gpurun_out/pfvar_${v}.json 2> gpurun_out/pfvar_${v}.err
  RAS_LIB_PATH=$PWD/variants/lib_$v.so RAS_TRSV=pf timeout 300 python tools/c4_demo.py --side 256 --sweeps 6 > gpurun_out/pfvar_${v}_demo.json 2>> gpurun_out/pfvar_${v}.err
  python -c "
import json; d=json.loads(open('gpurun_out/pfvar_${v}.json').read().strip().splitlines()[-1]); e=json.loads(open('gpurun_out/pfvar_${v}_demo.json').read().strip().splitlines()[-1]); print('$v', 'c4_1sub_s', round(d['time_s'],2), d['status'], 'demo_us_per_level', round(e['us_per_level'],3))" || tail -3 gpurun_out/pfvar_${v}.err
done

#!/bin/bash
for v in "$@"; do
  RAS_LIB_PATH=$PWD/variants/lib_$v.so timeout -s KILL 300 python tools/c4_demo.py --side 160 --sweeps 4 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_sweep'],2), round(d['kernels']['k_trsv']['ms_per_sweep'],2))"
done

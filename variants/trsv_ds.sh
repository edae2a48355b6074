#!/bin/bash
# k_trsv_ds variants on the C4 shape (same box): c4_demo 128^3 and 256^3
for v in "$@"; do
  for side in 128 256; do
    RAS_LIB_PATH=$PWD/variants/lib_$v.so timeout 300 python tools/c4_demo.py --side $side --sweeps 6 > gpurun_out/dsvar_${v}_$side.json 2> gpurun_out/dsvar_${v}_$side.err
    python -c "
import json; d=json.loads(open('gpurun_out/dsvar_${v}_$side.json').read().strip().splitlines()[-1]); print('$v', $side, round(d['ms_per_sweep'],3), round(d['us_per_level'],3))" || tail -3 gpurun_out/dsvar_${v}_$side.err
  done
done

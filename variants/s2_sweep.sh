#!/bin/bash
# Round 2 session 2 tuning sweep (same box): k_residual CTA shape on C2, k_trsv_pf
# poll back-off on the C4 shape (256^3, 8 subdomains, level-counter kernel forced).
bash variants/resid.sh base mb6 mb4 nt512 > gpurun_out/s2_var_resid.txt 2>&1
for v in base sleep16 sleep0; do
  RAS_LIB_PATH=$PWD/variants/lib_$v.so RAS_TRSV=pf timeout 300 python tools/c4_demo.py --side 256 --sweeps 6 > gpurun_out/s2_var_trsv_$v.json 2> gpurun_out/s2_var_trsv_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/s2_var_trsv_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_sweep'],3), round(d['us_per_level'],3))" >> gpurun_out/s2_var_trsv.txt
done
cat gpurun_out/s2_var_resid.txt gpurun_out/s2_var_trsv.txt

#!/bin/bash
# round measurement: bench line, ncu launch list, ncu --set full of the dominant kernel
timeout -s KILL 600 python bench.py > gpurun_out/bench_final.log 2>&1 || exit 1
echo bench-ok
timeout -s KILL 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 || exit 1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo launches-ok
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_resident_pcg -s 1 -c 1 \
  -o gpurun_out/final_resid python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
echo full-ok
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 2 -c 1 \
  -o gpurun_out/final_residual python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full2.log 2>&1
echo done

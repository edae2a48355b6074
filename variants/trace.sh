#!/bin/bash
for v in TRACE; do
RAS_TRACE_FILE=gpurun_out/trace_$v.bin RAS_LIB_PATH=$PWD/variants/lib_$v.so timeout -s KILL 200 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
done

#!/bin/bash
# Round 2, session 2: parity of the changed kernels (k_trsv_cl), the loopback
# suite, the C2 bench, and the C4-shape trisolve timing (cluster-resident vs the
# level-counter kernel).
set -x
mkdir -p gpurun_out
P=${P:-s2c}
python -m pytest tests/test_gpu_ic0.py tests/test_gpu_loopback.py -q --timeout 300 > gpurun_out/${P}_tests.txt 2>&1
tail -3 gpurun_out/${P}_tests.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-tts --no-e2e > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
tail -c 400 gpurun_out/${P}_bench.json
for side in 128 256; do
  RAS_TRSV_DEBUG=1 timeout 300 python tools/c4_demo.py --side $side --sweeps 6 >> gpurun_out/${P}_c4.jsonl 2>> gpurun_out/${P}_c4.err
  RAS_TRSV=level timeout 300 python tools/c4_demo.py --side $side --sweeps 6 >> gpurun_out/${P}_c4.jsonl 2>> gpurun_out/${P}_c4.err
done
cut -c1-400 gpurun_out/${P}_c4.jsonl
cat gpurun_out/${P}_c4.err | sort | uniq -c | head

#!/bin/bash
# time-to-solution (rel. residual 1e-8) at growing sizes, sync and async
for sc in 256 512; do
  for md in async; do
    timeout 1500 python bench.py --scale $sc --mode $md --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --tts > gpurun_out/tts_${sc}_${md}.json 2> gpurun_out/tts_${sc}_${md}.err
    python -c "
import json; d=json.load(open('gpurun_out/tts_${sc}_${md}.json')); t=d['tts']; print('$sc $md', d['config']['grid'], 'ms/step', round(d['ms_per_step'],2), 'tts', t)" || tail -3 gpurun_out/tts_${sc}_${md}.err
  done
done

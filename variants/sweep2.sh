#!/bin/bash
for f in "" "--plain" "--fuse-p"; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $f > gpurun_out/fmt.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/fmt.json')); print('[$f]', round(d['ms_per_step'],3), round(d['kernel_pass_ms_per_step'],3), ' '.join(k+':'+str(round(v['avg_us'],1))+'/'+str(round(v['gbs'] or 0)) for k,v in d['kernels'].items()))"
done

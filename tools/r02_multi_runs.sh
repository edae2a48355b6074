set -x
python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/r02_multi4_tests.txt 2>&1; tail -3 gpurun_out/r02_multi4_tests.txt
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_r02_n2.json 2> gpurun_out/bench_r02_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_r02_n4.json 2> gpurun_out/bench_r02_n4.err
RAS_SETUP_TRACE=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus 4 --config c5 --steps 20 --warmup 5 > gpurun_out/bench_r02_n4_c5.json 2> gpurun_out/bench_r02_n4_c5.err
grep "ras setup" gpurun_out/bench_r02_n4_c5.err | head -4
for f in bench_r02_n2 bench_r02_n4 bench_r02_n4_c5; do python -c "
import json,sys; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], d['e2e'], d['setup_s'])"; done

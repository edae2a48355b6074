set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_final.json 2> gpurun_out/bench_r02_final.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_r02_final.json 2>&1
python bench.py --steps 5 --warmup 3 --tts --no-cpu-baseline --no-e2e --no-tts > gpurun_out/bench_r02_tts_c2.json 2> gpurun_out/bench_r02_tts_c2.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tts --no-e2e > gpurun_out/launch_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tts --no-e2e > gpurun_out/ncu_launch.log 2>&1
tail -c 300 gpurun_out/bench_r02_tts_c2.json

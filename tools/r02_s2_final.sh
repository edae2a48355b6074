#!/bin/bash
# Round 2, session 2, final single-GPU measurements on the final code: the full
# bench line (C2, TTS on the small configs, e2e, cpu_baseline), the reference
# (oracle) arm, the C2 time to 1e-8, and the ncu launch list of the bench command
# (each ncu pass only after the same command exited 0 without ncu).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/s2_final_bench.json 2> gpurun_out/s2_final_bench.err
tail -c 300 gpurun_out/s2_final_bench.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/s2_final_reference.json 2> gpurun_out/s2_final_reference.err
python bench.py --steps 5 --warmup 3 --tts --no-cpu-baseline --no-e2e --no-tts > gpurun_out/s2_final_tts_c2.json 2> gpurun_out/s2_final_tts_c2.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts --no-e2e > gpurun_out/s2_final_launch_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2_final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts --no-e2e > gpurun_out/s2_final_ncu.log 2>&1
tail -c 300 gpurun_out/s2_final_tts_c2.json

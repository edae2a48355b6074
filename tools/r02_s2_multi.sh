#!/bin/bash
# Round 2, session 2, multi-GPU runs on a 4-GPU box: C3 as specified (one 2^24-row
# subdomain per GPU, overlap 1/2/4/8, sync and async) at G = 1, 2, 4, and the
# C4 shape on 4 GPUs (one 256^3 subdomain each, IC(0)-PCG, sync and async) with
# the session-2 trisolve.
set -x
mkdir -p gpurun_out
for G in 1 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $((29620 + G)) \
    tools/c3_run.py >> gpurun_out/s2_c3.jsonl 2>> gpurun_out/s2_c3.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29630 \
  tools/c4_run.py --grid 512 512 256 --parts 2 2 1 --solvers ic0:10 --modes sync,async >> gpurun_out/s2_c4run4.jsonl 2>> gpurun_out/s2_c4run4.err
cut -c1-250 gpurun_out/s2_c3.jsonl gpurun_out/s2_c4run4.jsonl

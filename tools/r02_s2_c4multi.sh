#!/bin/bash
# C4 shape (one 256^3 subdomain per GPU, IC(0)-PCG m=10, sync and async) on 2 and 4
# GPUs with the final trisolve (k_trsv_pf with per-chunk dependency flags).
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 \
  tools/c4_run.py --grid 512 256 256 --parts 2 1 1 --solvers ic0:10 --modes sync,async >> gpurun_out/s2z_c4.jsonl 2>> gpurun_out/s2z_c4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 \
  tools/c4_run.py --grid 512 512 256 --parts 2 2 1 --solvers ic0:10 --modes sync,async >> gpurun_out/s2z_c4.jsonl 2>> gpurun_out/s2z_c4.err
cut -c1-250 gpurun_out/s2z_c4.jsonl

#!/bin/bash
# Exercise bench.py's N > 1 code on a one-GPU box: every rank on cuda:0,
# gloo host plumbing, communicator-less upir world (peer windows only).
# Numbers printed here are NOT bench values (ranks time-slice one GPU).
set -x
R=torch.distributed.run
for wl in reduce reduce34 jacobi32k; do
  UPIR_BENCH_SHARED_GPU=1 UPIR_C5A_LOG2=24 UPIR_C5B_N=2048 timeout 300 python -m $R --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --steps 3 --warmup 3 \
    --n-log2 24 --e2e-steps 1 --workload $wl
  echo "rc[$wl]=$?"
done

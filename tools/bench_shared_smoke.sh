#!/bin/bash
# Exercise bench.py's N > 1 code on a one-GPU box: every rank on cuda:0,
# gloo host plumbing, communicator-less upir world (peer windows only; the
# NCCL lines report "unavailable").  Numbers printed here are NOT bench
# values (the ranks time-slice one GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for n in 2 3; do
  UPIR_BENCH_SHARED_GPU=1 UPIR_C5A_LOG2=26 UPIR_C5B_N=4096 timeout 600 python bench.py --gpus $n --steps 3 \
    --warmup 3 --n-log2 26 --e2e-steps 1 --no-kernels > gpurun_out/shared_$n.json 2> gpurun_out/shared_$n.err
  echo "rc[N=$n]=$?"
done

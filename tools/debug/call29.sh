cd "$GRAFT_REPO_ROOT"
bash tools/bench_shared_smoke.sh > gpurun_out/shared_smoke.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29733 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/ref_n2.log 2>&1; echo "ref n2 rc=$?" >> gpurun_out/ref_n2.log
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final.log

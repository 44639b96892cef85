cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_gputest.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2a_bench.log

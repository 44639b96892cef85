cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/sweep_r2.py axpy reduce > gpurun_out/r2e_sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/r2e_sweep.log
timeout 1800 python -m pytest -x -q tests/test_gpu_fullsize_bench.py tests/test_gpu_peer.py tests/test_gpu_data.py -k "fullsize or multirank or block or graph_capture or pipelined" > gpurun_out/r2e_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e_tests.log

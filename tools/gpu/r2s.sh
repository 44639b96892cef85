cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q tests/test_gpu_data.py tests/test_gpu_peer.py tests/test_gpu_stream.py > gpurun_out/r2s_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2s_tests.log

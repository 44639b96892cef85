cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/sweep_r2.py axpy2 > gpurun_out/r2q_sweep.log 2>&1
UPIR_DVAR=10 timeout 900 python -m pytest -x -q tests/test_gpu_stream.py -k "axpy" >> gpurun_out/r2q_sweep.log 2>&1

cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests -m gpu -x -q -k "jacobi or halo or peer" > gpurun_out/pytest_jac.log 2>&1; echo rc=$? >> gpurun_out/pytest_jac.log
timeout 600 python tools/debug/jacobi_sweep.py > gpurun_out/jacobi_sweep.txt 2>&1
timeout 300 python tools/debug/axpy_geom.py > gpurun_out/axpy_geom2.txt 2>&1

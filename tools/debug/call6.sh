cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests -m gpu -x -q -k "jacobi or halo or peer or stencil" > gpurun_out/pytest_jac.log 2>&1; echo rc=$? >> gpurun_out/pytest_jac.log
TILES=16x256,32x128 TEAMS=296,444 NSTS=0,2,3 timeout 600 python tools/debug/jacobi_sweep.py > gpurun_out/jacobi_sweep3.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_k3.log 2>&1

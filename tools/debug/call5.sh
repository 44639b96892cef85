cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests -m gpu -x -q -k "jacobi or halo or peer" > gpurun_out/pytest_jac.log 2>&1; echo rc=$? >> gpurun_out/pytest_jac.log
TILES=16x256,32x256,32x128 TEAMS=296,444 NSTS=0,2 timeout 600 python tools/debug/jacobi_sweep.py > gpurun_out/jacobi_sweep2.txt 2>&1
export TILES=16x256 TEAMS=444 NSTS=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi5 -s 10 -c 1 -o gpurun_out/prof_jacobi_ring2 -f python tools/debug/jacobi_sweep.py > gpurun_out/ncu_jac.log 2>&1

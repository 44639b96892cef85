cd "$GRAFT_REPO_ROOT"
export TILES=16x256 TEAMS=444 NSTS=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi5 -s 10 -c 1 -o gpurun_out/prof_jacobi_ring -f python tools/debug/jacobi_sweep.py > gpurun_out/ncu_jac.log 2>&1

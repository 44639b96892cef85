cd "$GRAFT_REPO_ROOT"
TILES=16x256,16x256,16x256 TEAMS=444,296 NSTS=0 timeout 600 python tools/debug/jacobi_sweep.py > gpurun_out/jacobi_sweep4.txt 2>&1
timeout 600 python bench.py --workload jacobi32k --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_j32k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 55 -c 1 -o gpurun_out/prof_stencil7b -f python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1

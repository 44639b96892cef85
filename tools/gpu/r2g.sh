cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_jacobi.py tests/test_gpu_fullsize_bench.py -k "jacobi or c3 or c5b" > gpurun_out/r2g_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2g_tests.log
timeout 1500 python tools/sweep_r2.py jacobi c5b > gpurun_out/r2g_sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/r2g_sweep.log
timeout 600 ncu --set full --clock-control none -k regex:jacobi5 -s 1 -c 1 -o gpurun_out/r2g_jacobi_c5b_skew -f python tools/one_kernel.py jacobi_c5b > gpurun_out/r2g_ncu.log 2>&1

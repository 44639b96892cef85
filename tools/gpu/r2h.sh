cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_stencil.py > gpurun_out/r2h_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2h_tests.log
for w in 0 2 3; do
  UPIR_STENCIL_WARPRING=$w timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-scaling --lines stencil7 > gpurun_out/r2h_st$w.json 2> gpurun_out/r2h_st$w.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil -s 1 -c 1 -o gpurun_out/r2h_stencil_wr -f python tools/one_kernel.py stencil7 > gpurun_out/r2h_ncu.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_fullsize_bench.py -k c5b >> gpurun_out/r2h_tests.log 2>&1
echo "pytest2 rc=$?" >> gpurun_out/r2h_tests.log

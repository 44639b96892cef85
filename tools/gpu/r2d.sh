cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for l in var_libs/libupir_old.so paper_2209_10643_b200/libupir.so; do
  timeout 300 python tools/experiments/ab_lib.py $l >> gpurun_out/r2d_ab.log 2>&1
done
timeout 1500 python -m pytest -x -q tests/test_gpu_stream.py tests/test_gpu_data.py tests/test_gpu_peer.py tests/test_gpu_fullsize_bench.py tests/test_gpu_matvec.py > gpurun_out/r2d_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d_tests.log
UPIR_BENCH_SHARED_GPU=1 UPIR_C5A_LOG2=31 UPIR_C5B_N=8192 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-kernels > gpurun_out/r2d_shared2.json 2> gpurun_out/r2d_shared2.err
echo "shared2 rc=$?" >> gpurun_out/r2d_shared2.err
timeout 1200 python tools/sweep_r2.py axpy jacobi c5b > gpurun_out/r2d_sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/r2d_sweep.log

# round 2: new parity tests, then the reworked bench (N=1, shared-GPU N=2, --gpus 2 refusal, reference arm)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q tests/test_gpu_stream.py -k misaligned tests/test_gpu_data.py tests/test_gpu_peer.py tests/test_gpu_fullsize_bench.py tests/test_gpu_matvec.py > gpurun_out/r2b_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench rc=$?" >> gpurun_out/r2b_bench.err
timeout 300 python bench.py --gpus 2 > gpurun_out/r2b_g2.log 2>&1
echo "gpus2 rc=$?" >> gpurun_out/r2b_g2.log
UPIR_BENCH_SHARED_GPU=1 UPIR_C5A_LOG2=31 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-kernels > gpurun_out/r2b_shared2.json 2> gpurun_out/r2b_shared2.err
echo "shared2 rc=$?" >> gpurun_out/r2b_shared2.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
echo "ref rc=$?" >> gpurun_out/r2b_ref.err

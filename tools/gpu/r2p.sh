cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_jacobi.py tests/test_gpu_stencil.py tests/test_gpu_peer.py -k "not matmul and not block" > gpurun_out/r2p_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2p_tests.log
for p in 0 1 0 1; do
  UPIR_PDL=$p timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-scaling --lines jacobi,stencil7 > gpurun_out/r2p_$p.json 2> gpurun_out/r2p_$p.err
  grep -E "jacobi|stencil" gpurun_out/r2p_$p.err | sed "s/^/PDL=$p /" >> gpurun_out/r2p_sum.log
  UPIR_PDL=$p timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-kernels --lines c5b > gpurun_out/r2p_c5b_$p.json 2> gpurun_out/r2p_c5b_$p.err
  grep -E "c5b" gpurun_out/r2p_c5b_$p.err | sed "s/^/PDL=$p /" >> gpurun_out/r2p_sum.log
done

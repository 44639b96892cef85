cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for h in 4 8 2 4; do
  UPIR_STENCIL_H=$h UPIR_STENCIL_CFGS="444x128:8x512" timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-scaling --lines stencil7 > gpurun_out/r2o_h$h.json 2>> gpurun_out/r2o.err
  grep stencil7_8192 gpurun_out/r2o.err | tail -1 | sed "s/^/H=$h /" >> gpurun_out/r2o_sum.log
done
UPIR_STENCIL_H=8 timeout 600 python -m pytest -q -x tests/test_gpu_stencil.py -k "strip_tiles and 8-512" >> gpurun_out/r2o_sum.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in 0 2; do
  UPIR_STENCIL_WARPRING=$w UPIR_STENCIL_CFGS="444x128:8x512,740x128:4x512,592x128:4x512,888x64:4x256,1184x64:4x256,888x64:8x256" timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-scaling --lines stencil7 > gpurun_out/r2i_st$w.json 2> gpurun_out/r2i_st$w.err
done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/sweep_r2.py jacobi > gpurun_out/r2n_sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/r2n_sweep.log

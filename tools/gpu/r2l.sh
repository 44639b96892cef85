cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_stencil.py > gpurun_out/r2l_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2l_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-scaling --lines stencil7 > gpurun_out/r2l_st.json 2> gpurun_out/r2l_st.err
TAG=r02 bash tools/prof_all.sh > gpurun_out/r2l_prof.log 2>&1
du -sh gpurun_out

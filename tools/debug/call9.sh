cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests -m gpu -x -q -k "stencil" > gpurun_out/pytest_st.log 2>&1; echo rc=$? >> gpurun_out/pytest_st.log
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_k4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 55 -c 1 -o gpurun_out/prof_stencil7 -f python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1

cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py -x -q > gpurun_out/pytest_ring.log 2>&1; echo rc=$? >> gpurun_out/pytest_ring.log
timeout 1000 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
CS=/usr/local/cuda/bin/compute-sanitizer
J="ring_depths and 9-128 or ragged_team_sizes or interior_fast_path or strip_tiles"
timeout 400 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py -q -x -k "$J" > gpurun_out/san_race_ring.log 2>&1; echo racecheck ring rc=$? >> gpurun_out/san_ring.txt
timeout 300 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py -q -x -k "$J" > gpurun_out/san_sync_ring.log 2>&1; echo synccheck ring rc=$? >> gpurun_out/san_ring.txt
timeout 300 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py -q -x -k "$J" > gpurun_out/san_mem_ring.log 2>&1; echo memcheck ring rc=$? >> gpurun_out/san_ring.txt

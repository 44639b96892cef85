#!/bin/bash
# compute-sanitizer over a representative subset of the GPU tests (1 B200).
cd "$GRAFT_REPO_ROOT"
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="test_reduce_i64_parity and (148-256 or 3-37) and (direct or staged) or test_axpy_parity and 4-100 or test_trace_mapping_bit_exact and 9-33 or guided_reduce and 3-37"
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_stream.py -q -x -k "$SEL" > gpurun_out/san_mem_stream.log 2>&1; echo memcheck stream rc=$?
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_matvec.py tests/test_gpu_stencil.py -q -x -k "parity_tiles and 70-300 or matvec_parity and 148 or stencil_parity and 70-300 or strip_tiles" > gpurun_out/san_mem_tiled.log 2>&1; echo memcheck tiled rc=$?
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_matmul.py -q -x -k "matmul_parity and 256-512 or f32_parity and 200" > gpurun_out/san_mem_mm.log 2>&1; echo memcheck matmul rc=$?
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py tests/test_gpu_matvec.py -q -x -k "parity_tiles and 70-300 and 32-256 or stencil_parity and 70-300 and 7 or matvec_parity and 148 and 257" > gpurun_out/san_race.log 2>&1; echo racecheck rc=$?
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_stream.py tests/test_gpu_matvec.py -q -x -k "test_reduce_i64_parity and 3-37 and direct or matvec_parity and 5-96" > gpurun_out/san_sync.log 2>&1; echo synccheck rc=$?
# the Jacobi window ring (producer warp, 2-4 slots, ragged teams) and the stencil strip ring
J="ring_depths and 9-128 or ragged_team_sizes or interior_fast_path or strip_tiles"
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py -q -x -k "$J" > gpurun_out/san_race_ring.log 2>&1; echo racecheck ring rc=$?
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py -q -x -k "$J" > gpurun_out/san_sync_ring.log 2>&1; echo synccheck ring rc=$?
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_stencil.py -q -x -k "$J" > gpurun_out/san_mem_ring.log 2>&1; echo memcheck ring rc=$?
# round 2: address-aligned vector paths (misaligned adopted views), the 256-thread AXPY kernel with
# one team per SM, the chunk-pipelined map and the graph-captured async halo
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_stream.py -q -x -k "misaligned and direct or axpy_misaligned or axpy_parity and 148-256 and direct" > gpurun_out/san_mem_align.log 2>&1; echo memcheck align rc=$?
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_data.py -q -x -k "pipelined or graph_capture or async_halo" > gpurun_out/san_mem_data.log 2>&1; echo memcheck data rc=$?
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -m pytest tests/test_gpu_stencil.py -q -x -k "strip_tiles" > gpurun_out/san_race_stencil.log 2>&1; echo racecheck stencil rc=$?
# the reversed Jacobi tile order, the async allreduce, the world-1 communicator combine path
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py tests/test_gpu_data.py -q -x -k "reverse or alternating or async_allreduce or world_combine" > gpurun_out/san_mem_r2b.log 2>&1; echo memcheck r2b rc=$?
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py -q -x -k "reverse and 1-static" > gpurun_out/san_race_rev.log 2>&1; echo racecheck reverse rc=$?
for f in gpurun_out/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed" $f | tail -3; done

#!/bin/bash
# bench + launch list + ncu --set full of the top kernels (1 B200).
cd "$GRAFT_REPO_ROOT"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_loop -c 2 -o gpurun_out/prof_reduce -f python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-kernels > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi5 -s 10 -c 1 -o gpurun_out/prof_jacobi -f python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:matmul -s 3 -c 1 -o gpurun_out/prof_matmul -f python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out

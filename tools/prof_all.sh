#!/bin/bash
# bench + launch list + ncu --set full of every loop-body kernel (1 B200).
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r01}
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_loop -c 2 -o gpurun_out/prof_reduce -f $B --no-kernels > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_loop -s 2 -c 1 -o gpurun_out/prof_axpy -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi5 -s 10 -c 1 -o gpurun_out/prof_jacobi -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:matmul_kernel -s 3 -c 1 -o gpurun_out/prof_matmul -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:matmul_pair_kernel -s 3 -c 1 -o gpurun_out/prof_matmul_pair -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:matmul_kernel -s 6 -c 1 -o gpurun_out/prof_matmul_f32 -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:matmul_pair_f32 -s 2 -c 1 -o gpurun_out/prof_matmul_pair_f32 -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi5 -s 5 -c 1 -o gpurun_out/prof_jacobi32k -f python bench.py --workload jacobi32k --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:matvec -s 3 -c 1 -o gpurun_out/prof_matvec -f $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 55 -c 1 -o gpurun_out/prof_stencil7 -f $B > /dev/null 2>&1
UPIR_PROFILES_OUT=gpurun_out/profiles python tools/ncu_summary.py $TAG gpurun_out/prof_*.ncu-rep
mkdir -p /tmp/ncu_keep && mv gpurun_out/prof_*.ncu-rep /tmp/ncu_keep/
cp /tmp/ncu_keep/prof_jacobi.ncu-rep /tmp/ncu_keep/prof_stencil7.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out gpurun_out/profiles

#!/bin/bash
# Profile the reduction loop kernels on one B200 (run under gpurun).
set -x
cd "$GRAFT_REPO_ROOT"
for s in static static1 dynamic; do
  timeout 300 python bench.py --steps 10 --warmup 3 --sched $s --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$s.log 2>&1
  tail -1 gpurun_out/bench_$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$s', d['value'], d['kernel_ms'], d['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_loop -c 2 -o gpurun_out/prof_static -f python bench.py --steps 1 --warmup 0 --sched static --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_static.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_loop -c 2 -o gpurun_out/prof_static1 -f python bench.py --steps 1 --warmup 0 --sched static1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_static1.log 2>&1
ls -la gpurun_out

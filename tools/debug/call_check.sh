cd "$GRAFT_REPO_ROOT"
nvidia-smi -q -d CLOCK,PERFORMANCE,POWER | head -80 > gpurun_out/smi_q.txt
./tools/debug/ffma_rate > gpurun_out/ffma.txt 2>&1
timeout 300 python tools/debug/axpy_geom.py > gpurun_out/axpy_geom.txt 2>&1
for i in 1 2; do
 (nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 500 > gpurun_out/smi_loop_$i.csv &  echo $! > /tmp/smipid)
 timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_k$i.log 2>&1
 kill $(cat /tmp/smipid)
done

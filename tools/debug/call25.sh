cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_jacobi.py -x -q > gpurun_out/pytest_jac3.log 2>&1; echo rc=$? >> gpurun_out/pytest_jac3.log
for cfg in "1 row" "0 col" "1 col" "0 row"; do
  set -- $cfg
  UPIR_JACOBI_CHUNK=$1 UPIR_JACOBI_ORDER=$2 TILES=16x256 TEAMS=444,296 NSTS=0 timeout 300 python tools/debug/jacobi_sweep.py | sed "s/^/C3 chunk $1 $2 /" >> gpurun_out/jac_order.txt 2>&1
  UPIR_JACOBI_CHUNK=$1 UPIR_JACOBI_ORDER=$2 timeout 600 python bench.py --workload jacobi32k --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5b chunk $1 $2', round(d['glups'],1), round(d['roofline']['frac'],3))" >> gpurun_out/jac_order.txt 2>&1
done
M=dram__bytes_read.sum,gpu__time_duration.sum
UPIR_JACOBI_CHUNK=0 UPIR_JACOBI_ORDER=col timeout 600 ncu --metrics $M --clock-control none -k regex:jacobi5 -s 4 -c 1 --csv python bench.py --workload jacobi32k --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/ncu C5b static col /" >> gpurun_out/jac_order.txt

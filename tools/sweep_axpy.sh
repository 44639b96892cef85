#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for v in 2 2 7 8 9; do
UPIR_DVAR=$v timeout 300 python bench.py --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --n-log2 24 > gpurun_out/sa.log 2>&1
tail -1 gpurun_out/sa.log | python -c "import json,sys
d=json.loads(sys.stdin.read())['kernels']['axpy']
print('dvar $v', {k:round(v['GB/s']) for k,v in d.items() if isinstance(v,dict)})"
done

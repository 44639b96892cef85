#!/bin/bash
cd "$GRAFT_REPO_ROOT"
j() { env "$@" timeout 300 python bench.py --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --n-log2 24 > gpurun_out/sj.log 2>&1
  tail -1 gpurun_out/sj.log | python -c "import json,sys
d=json.loads(sys.stdin.read())['kernels']
print('$*', 'jacobi', round(d['jacobi'].get('GLUP/s',0),1), 'axpy', {k:round(v['GB/s']) for k,v in d['axpy'].items() if isinstance(v,dict)})"; }
j UPIR_JACOBI_TEAMS=296
j UPIR_JACOBI_TEAMS=444
j UPIR_JACOBI_TEAMS=148
j UPIR_JACOBI_TEAMS=740 UPIR_JACOBI_TILE=16x256
j UPIR_JACOBI_TEAMS=444 UPIR_JACOBI_TILE=16x256
j UPIR_JACOBI_TEAMS=592 UPIR_JACOBI_TILE=32x128
j UPIR_JACOBI_TEAMS=296 UPIR_JACOBI_TILE=64x128
for v in 0 1 2 3; do j UPIR_DVAR=$v UPIR_JACOBI_TEAMS=296; done
j UPIR_PATH=staged UPIR_STAGE=8,2
j UPIR_PATH=staged UPIR_STAGE=4,2

#!/bin/bash
# Sweep memory paths / configs of the static-block reduction (1 B200).
cd "$GRAFT_REPO_ROOT"
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 2 --sched ${SCHED:-static} --e2e-steps 0 --no-cpu-baseline > gpurun_out/sw_$label.log 2>&1
  tail -1 gpurun_out/sw_$label.log | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$label', round(d['value']), {k: round(v,3) for k,v in d['kernel_ms'].items()})
except Exception as e: print('$label', 'FAILED', e)"
}
for v in 0 1 2 3; do run direct_v$v UPIR_PATH=direct UPIR_DVAR=$v; done
for cfg in 16,2 8,2; do run staged_$cfg UPIR_PATH=staged UPIR_STAGE=$cfg; done
SCHED=static1 run static1 X=1
SCHED=dynamic run dynamic X=1

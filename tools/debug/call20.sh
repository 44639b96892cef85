cd "$GRAFT_REPO_ROOT"
for v in base axb base axb; do
  cp build/var/libupir_$v.so paper_2209_10643_b200/libupir.so
  GEOMS=592x256,296x256 DVARS=8 timeout 300 python tools/debug/axpy_geom.py | sed "s/^/$v static /" >> gpurun_out/axpy_ab.txt 2>&1
  TAG=$v timeout 300 python - >> gpurun_out/axpy_ab.txt 2>&1 <<'PY'
import os, sys, types
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2209_10643_b200 as U
ctx = U.upir_init(0)
stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
peaks, src = bench.measured_peaks()
r = bench.bench_axpy(types.SimpleNamespace(steps=5), U, ctx, stream, peaks, src)
print(os.environ["TAG"], "bench_axpy", {k: round(v["frac"], 3) for k, v in r.items() if isinstance(v, dict)}, flush=True)
U.upir_finalize(ctx)
PY
done
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -1 >> gpurun_out/axpy_ab.txt

"""bench.py's stencil7 line alone (GLUP/s per tile / geometry).  Run on the GPU box."""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2209_10643_b200 as U  # noqa: E402

ctx = U.upir_init(0)
stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
peaks, src = bench.measured_peaks()
r = bench.bench_stencil7(types.SimpleNamespace(steps=5), U, ctx, stream, peaks, src)
print(os.environ.get("TAG", ""), {k: round(v["GLUP/s"]) for k, v in r.items() if isinstance(v, dict) and "GLUP/s" in v},
      round(r["roofline"]["frac"], 3), flush=True)
U.upir_finalize(ctx)

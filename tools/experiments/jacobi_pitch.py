"""C5b-size Jacobi (32768^2 interior space) with a padded row pitch: does a
non-power-of-2 pitch remove the L2 set conflicts of 128 KiB rows?  (Fill
treats the padded row as the grid row: a perf experiment, not a parity run.)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2209_10643_b200 as U  # noqa: E402

n, S = 32768, 20
ctx = U.upir_init(0)
stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
for pad in [int(p) for p in os.environ.get("PADS", "0,32,64,128,1024").split(",")]:
    ld = n + pad
    a_t = torch.empty(n * ld, dtype=torch.float32, device="cuda")
    b_t = torch.empty(n * ld, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma, mb = U.upir_data_adopt(ctx, a_t), U.upir_data_adopt(ctx, b_t)
    U.upir_synth_fill(ctx, ma, 4, 5, 0, n, ld)
    U.upir_synth_fill(ctx, mb, 4, 5, 0, n, ld)
    loop = U.loop_desc([1, 1], [n - 1, n - 1], tile=[16, 256], policy=U.SCHED_STATIC, chunk=1,
                       distribute=U.DIST_TEAMS, inner_chunk=4)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(int(os.environ.get("TEAMS", 444)), 256))
    bodies = [U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(ld, 0, 0), dims=(n, 0, 0)),
              U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(ld, 0, 0), dims=(n, 0, 0))]
    U.upir_graph_begin(ctx)
    for k in range(S):
        U.upir_loop_exec(s, loop, bodies[k % 2])
    g = U.upir_graph_end(ctx)
    U.upir_graph_launch(ctx, g)
    U.upir_sync(ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        U.upir_graph_launch(ctx, g)
    e1.record(stream)
    U.upir_sync(ctx)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    lups = (n - 2) ** 2 * S
    print(f"pad {pad}: {lups / ms / 1e6:.1f} GLUP/s  {8 * lups / ms / 1e6:.0f} GB/s", flush=True)
    U.upir_graph_destroy(g)
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, ma)
    U.upir_data_unmap(ctx, mb)
    U.upir_sync(ctx)
    del a_t, b_t
    torch.cuda.empty_cache()
U.upir_finalize(ctx)

"""Run one STENCIL2D sweep configuration (for ncu): n, teams, units, BM, BN, reps."""
import sys

import torch

import paper_2209_10643_b200 as U

n, teams, units, bm, bn, reps = (int(v) for v in sys.argv[1:7])
ctx = U.upir_init(0)
v = torch.tensor([1, 2, 3, 4, 3, 2, 1], dtype=torch.float64)
w = (torch.outer(v, v) / 256.0).float().cuda()
a_t = torch.empty(n * n, dtype=torch.float32, device="cuda")
b_t = torch.empty(n * n, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
ma, mb, mw = U.upir_data_adopt(ctx, a_t), U.upir_data_adopt(ctx, b_t), U.upir_data_adopt(ctx, w)
U.upir_synth_fill(ctx, ma, 4, 5, 0, n, n)
s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
loop = U.loop_desc([3, 3], [n - 3, n - 3], tile=[bm, bn], chunk=1, distribute=U.DIST_TEAMS, inner_chunk=4)
body = U.body(U.BODY_STENCIL2D, U.F32, in0=ma, in1=mw, out=mb, ld=(n, 0, 0), dims=(n, 7, 0))
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
for k in range(reps):
    if k == reps - 1:
        st.record(stream)
    U.upir_loop_exec(s, loop, body)
en.record(stream)
U.upir_sync(ctx)
torch.cuda.synchronize()
ms = st.elapsed_time(en)
print(f"n={n} {teams}x{units} tile {bm}x{bn}: {ms:.4f} ms, {(n - 6) ** 2 / ms / 1e6:.1f} GLUP/s")
U.upir_spmd_end(s)
for m in (mw, mb, ma):
    U.upir_data_unmap(ctx, m)
U.upir_sync(ctx)
U.upir_finalize(ctx)

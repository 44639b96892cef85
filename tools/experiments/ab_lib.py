"""A/B of two libupir.so builds on the C2 reduce and axpy loops (one GPU).

    python tools/experiments/ab_lib.py <path/to/libupir.so>
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2209_10643_b200._abi as A  # noqa: E402

A.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402
import paper_2209_10643_b200 as U  # noqa: E402

ctx = U.upir_init(0)
stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
n = 1 << 30
x = torch.empty(n, dtype=torch.int64, device="cuda")
y = torch.empty(n // 4, dtype=torch.float32, device="cuda")
z = torch.empty(n // 4, dtype=torch.float32, device="cuda")
r = torch.zeros(4, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
mx, my, mz = U.upir_data_adopt(ctx, x), U.upir_data_adopt(ctx, y), U.upir_data_adopt(ctx, z)
U.upir_synth_fill(ctx, mx, 2, 6)
U.upir_synth_fill(ctx, my, 0, 1)
U.upir_synth_fill(ctx, mz, 0, 2)
s = U.upir_spmd_launch(ctx, U.spmd_desc(592, 256))
b = r.data_ptr()
for label, loop, body, reds, nbytes in (
        ("reduce_i64_static", U.loop_desc(0, n), U.body(U.BODY_REDUCE, U.I64, in0=mx),
         [U.reduction(U.OP_SUM, U.I64, b), U.reduction(U.OP_MAX, U.I64, b + 8)], 8 * n),
        ("axpy_static", U.loop_desc(0, n // 4), U.body(U.BODY_AXPY, U.F32, in0=my, out=mz, alpha=2.0),
         [U.reduction(U.OP_SUM, U.F32, b + 16)], 12 * (n // 4)),
        ("axpy_static4", U.loop_desc(0, n // 4, chunk=4), U.body(U.BODY_AXPY, U.F32, in0=my, out=mz, alpha=2.0),
         [U.reduction(U.OP_SUM, U.F32, b + 16)], 12 * (n // 4))):
    for _ in range(3):
        U.upir_loop_exec(s, loop, body, reds)
    U.upir_sync(ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        U.upir_loop_exec(s, loop, body, reds)
    e1.record(stream)
    U.upir_sync(ctx)
    ms = e0.elapsed_time(e1) / 10
    print(f"{os.path.basename(sys.argv[1])} {label}: {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)
U.upir_spmd_end(s)

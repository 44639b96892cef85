"""Sweep: AXPY (fused fp32 sum) under schedule(static) block vs. SPMD geometry
and long-chunk variant (UPIR_DVAR).  Prints GB/s per (teams, units, dvar).
Run on the GPU box: python tools/experiments/axpy_geom.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2209_10643_b200 as U  # noqa: E402


def main():
    n = 1 << 28
    ctx = U.upir_init(0)
    stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    r = torch.zeros(1, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    mx, my = U.upir_data_adopt(ctx, x), U.upir_data_adopt(ctx, y)
    U.upir_synth_fill(ctx, mx, 0, 1)
    U.upir_synth_fill(ctx, my, 0, 2)
    geoms = [tuple(int(v) for v in g.split("x"))
             for g in os.environ.get("GEOMS", "148x256,296x128,296x256,444x256,592x256,148x1024").split(",")]
    # "8" = direct path variant 8 (UPIR_DVAR), "s" = the staged (per-unit TMA bulk) path
    dvars = os.environ.get("DVARS", "1,7,8,s").split(",")
    for t, u in geoms:
        s = U.upir_spmd_launch(ctx, U.spmd_desc(t, u))
        for dv in dvars:
            if dv == "s":
                os.environ["UPIR_PATH"] = "staged"
            else:
                os.environ.pop("UPIR_PATH", None)
                os.environ["UPIR_DVAR"] = dv
            loop = U.loop_desc(0, n, policy=U.SCHED_STATIC, chunk=0)
            body = U.body(U.BODY_AXPY, U.F32, in0=mx, out=my, alpha=2.0)
            red = [U.reduction(U.OP_SUM, U.F32, r)]
            for _ in range(3):
                U.upir_loop_exec(s, loop, body, red)
            U.upir_sync(ctx)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                U.upir_loop_exec(s, loop, body, red)
            e1.record(stream)
            U.upir_sync(ctx)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            print(f"teams {t:5d} units {u:5d} dvar {dv}: {12 * n / ms / 1e6:8.1f} GB/s", flush=True)
        U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, mx)
    U.upir_data_unmap(ctx, my)
    U.upir_sync(ctx)
    U.upir_finalize(ctx)


if __name__ == "__main__":
    main()

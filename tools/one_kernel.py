"""Run ONE loop-body configuration twice (warm-up + the launch ncu captures
with `-s 1 -c 1 -k regex:<kernel>`), inputs from the on-device generator.

    python tools/one_kernel.py axpy_static|axpy_static4|reduce_i64|reduce_f32|
                               jacobi_c3|jacobi_c5b|stencil7|matvec|matmul_pair|matmul_f32_pair
Env hooks of the runtime (UPIR_*) apply as in bench.py."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2209_10643_b200 as U  # noqa: E402


def main():
    what = sys.argv[1]
    ctx = U.upir_init(0)
    keep = []

    def adopt(n, dt, dist_code=None, stream=0, rows=0, cols=0, d=None):
        t = torch.empty(n, dtype=dt, device="cuda")
        torch.cuda.synchronize()
        keep.append(t)
        m = U.upir_data_adopt(ctx, t, d) if d else U.upir_data_adopt(ctx, t)
        if dist_code is not None:
            U.upir_synth_fill(ctx, m, dist_code, stream, 0, rows, cols)
        return m

    r = torch.zeros(4, dtype=torch.int64, device="cuda")
    b = r.data_ptr()
    if what.startswith("axpy"):
        n = 1 << 28
        mx, my = adopt(n, torch.float32, 0, 1), adopt(n, torch.float32, 0, 2)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(592, 256))
        loop = U.loop_desc(0, n, chunk=4 if what == "axpy_static4" else 0)
        run = lambda: U.upir_loop_exec(s, loop, U.body(U.BODY_AXPY, U.F32, in0=mx, out=my, alpha=2.0),  # noqa: E731
                                       [U.reduction(U.OP_SUM, U.F32, b)])
    elif what.startswith("reduce"):
        n = 1 << 30
        dt, code, st = (U.I64, 2, 6) if what == "reduce_i64" else (U.F32, 0, 7)
        m = adopt(n, torch.int64 if dt == U.I64 else torch.float32, code, st)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(592, 256))
        ch = int(os.environ.get("UPIR_C2_CHUNK", 2 if dt == U.I64 else 4))   # bench's C2 schedule: one 16-B vector
        run = lambda: U.upir_loop_exec(s, U.loop_desc(0, n, chunk=ch), U.body(U.BODY_REDUCE, dt, in0=m),  # noqa: E731
                                       [U.reduction(U.OP_SUM, dt, b), U.reduction(U.OP_MAX, dt, b + 8)])
    elif what.startswith("jacobi"):
        n = 8192 if what == "jacobi_c3" else 32768
        ma, mb = adopt(n * n, torch.float32, 4, 5, n, n), adopt(n * n, torch.float32, 4, 5, n, n)
        teams = int(os.environ.get("UPIR_JACOBI_TEAMS", 444))
        pol = U.SCHED_DYNAMIC if os.environ.get("UPIR_JACOBI_POLICY") == "dynamic" else U.SCHED_STATIC
        s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, 256))
        loop = U.loop_desc([1, 1], [n - 1, n - 1], tile=[16, 256], policy=pol,
                           chunk=int(os.environ.get("UPIR_JACOBI_CHUNK", 1)), distribute=U.DIST_TEAMS, inner_chunk=4)
        run = lambda: U.upir_loop_exec(s, loop, U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb,  # noqa: E731
                                                       ld=(n, 0, 0), dims=(n, 0, 0)))
    elif what == "stencil7":
        n = 8192
        ma, mb = adopt(n * n, torch.float32, 4, 5, n, n), adopt(n * n, torch.float32, 4, 5, n, n)
        v = torch.tensor([1, 2, 3, 4, 3, 2, 1], dtype=torch.float64)
        w = (torch.outer(v, v) / 256.0).float().cuda()
        keep.append(w)
        mw = U.upir_data_adopt(ctx, w)
        teams, units = (int(x) for x in os.environ.get("UPIR_STENCIL_GEOM", "444x128").split("x"))
        bm, bn = (int(x) for x in os.environ.get("UPIR_STENCIL_TILE", "8x512").split("x"))
        s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
        loop = U.loop_desc([3, 3], [n - 3, n - 3], tile=[bm, bn], chunk=1, distribute=U.DIST_TEAMS, inner_chunk=4)
        run = lambda: U.upir_loop_exec(s, loop, U.body(U.BODY_STENCIL2D, U.F32, in0=ma, in1=mw, out=mb,  # noqa: E731
                                                       ld=(n, 0, 0), dims=(n, 7, 0)))
    elif what == "matvec":
        n = 16384
        ma, mx, my = adopt(n * n, torch.float32, 1, 3), adopt(n, torch.float32, 1, 1), adopt(n, torch.float32)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(592, 256))
        run = lambda: U.upir_loop_exec(s, U.loop_desc(0, n, chunk=1, distribute=U.DIST_TEAMS, inner_chunk=4),  # noqa: E731
                                       U.body(U.BODY_MATVEC, U.F32, in0=ma, in1=mx, out=my, ld=(n, 0, 0), dims=(n, n, 0)))
    elif what.startswith("matmul"):
        n = 8192
        f32 = "f32" in what
        tdt, dt, code = (torch.float32, U.F32, 1) if f32 else (torch.bfloat16, U.BF16, 3)
        ma, mb, mc = adopt(n * n, tdt, code, 3), adopt(n * n, tdt, code, 4), adopt(n * n, torch.float32)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(74, 768 if f32 else 512))
        run = lambda: U.upir_loop_exec(s, U.loop_desc([0, 0], [n, n], chunk=1, distribute=U.DIST_TEAMS),  # noqa: E731
                                       U.body(U.BODY_MATMUL, dt, in0=ma, in1=mb, out=mc, ld=(n, n, n), dims=(n, n, n)))
    else:
        raise SystemExit("unknown kernel " + what)
    run()
    U.upir_sync(ctx)
    run()
    U.upir_sync(ctx)
    U.upir_spmd_end(s)
    print("ok", what)


if __name__ == "__main__":
    main()

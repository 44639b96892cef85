"""Shared helpers for the -m gpu parity tests (test harness only)."""
import contextlib
import os

import numpy as np
import torch

import paper_2209_10643_b200 as U


@contextlib.contextmanager
def upir_path(p):
    """Force the streaming kernels' memory path ('direct' / 'staged')."""
    old = os.environ.get("UPIR_PATH")
    os.environ["UPIR_PATH"] = p
    try:
        yield
    finally:
        if old is None:
            os.environ.pop("UPIR_PATH", None)
        else:
            os.environ["UPIR_PATH"] = old


def dev_scalar(dtype):
    t = torch.zeros(1, dtype=torch.int64 if dtype == U.I64 else torch.float32, device="cuda")
    torch.cuda.synchronize()
    return t


def run_reduce(ctx, x, ops, teams, units, policy=U.SCHED_STATIC, chunk=0, distribute=U.DIST_TEAMS_UNITS,
               lb=0, ub=None, step=1, inits=None, trace=False, simdlen=0):
    """Map x (host numpy int64/float32) TO the device, run a REDUCE loop with the
    given reductions, return (results, trace arrays or None)."""
    dtype = U.I64 if x.dtype == np.int64 else U.F32
    ub = len(x) if ub is None else ub
    m = U.upir_data_map(ctx, x, U.MAP_TO)
    outs = [dev_scalar(dtype) for _ in ops]
    inits = inits or [None] * len(ops)
    reds = [U.reduction(op, dtype, o, init=i) for op, o, i in zip(ops, outs, inits)]
    loop = U.loop_desc(lb, ub, step, policy=policy, chunk=chunk, distribute=distribute, simdlen=simdlen)
    T, _ = U.upir_loop_normalize(loop)
    tr = tm = None
    if trace:
        tr = np.zeros(3 * max(T, 1), dtype=np.int32)
        tm = U.upir_data_map(ctx, tr, U.MAP_TOFROM)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
    U.upir_loop_exec(s, loop, U.body(U.BODY_REDUCE, dtype, in0=m), reds, trace=tm)
    U.upir_spmd_end(s)
    if tm is not None:
        U.upir_data_unmap(ctx, tm)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    res = [o.item() for o in outs]
    trs = None
    if trace:
        trs = (tr[:T].copy(), tr[T:2 * T].copy(), tr[2 * T:3 * T].copy())
    return res, trs


def run_axpy(ctx, a, x, y, teams, units, policy=U.SCHED_STATIC, chunk=0, distribute=U.DIST_TEAMS_UNITS,
             lb=0, ub=None, step=1, sum_=False, trace=False, simdlen=0):
    ub = len(y) if ub is None else ub
    yy = y.copy()
    mx = U.upir_data_map(ctx, x, U.MAP_TO)
    my = U.upir_data_map(ctx, yy, U.MAP_TOFROM)
    out = dev_scalar(U.F32)
    reds = [U.reduction(U.OP_SUM, U.F32, out)] if sum_ else None
    loop = U.loop_desc(lb, ub, step, policy=policy, chunk=chunk, distribute=distribute, simdlen=simdlen)
    T, _ = U.upir_loop_normalize(loop)
    tr = tm = None
    if trace:
        tr = np.zeros(3 * max(T, 1), dtype=np.int32)
        tm = U.upir_data_map(ctx, tr, U.MAP_TOFROM)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
    U.upir_loop_exec(s, loop, U.body(U.BODY_AXPY, U.F32, in0=mx, out=my, alpha=a), reds, trace=tm)
    U.upir_spmd_end(s)
    if tm is not None:
        U.upir_data_unmap(ctx, tm)
    U.upir_data_unmap(ctx, my)
    U.upir_data_unmap(ctx, mx)
    U.upir_sync(ctx)
    trs = (tr[:T].copy(), tr[T:2 * T].copy(), tr[2 * T:3 * T].copy()) if trace else None
    return yy, (out.item() if sum_ else None), trs


def flat_unit(team, unit, units, distribute):
    """Schedule-unit id g of an executor (team, unit) (readings c5-c7)."""
    if distribute == U.DIST_TEAMS:
        return team
    if distribute == U.DIST_UNITS:
        return unit
    return team.astype(np.int64) * units + unit

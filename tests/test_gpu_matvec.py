"""GPU parity of the MATVEC loop body (NEXT #2: the paper's fourth kernel,
PAPER.md:1217) against the fp64 oracle.  Tolerance: |dy_i| / sum_k |A_ik x_k|
<= 1e-5 (reading c22 applied per row); the row -> team / unit mapping of the
static schedules is bit-exact."""
import numpy as np
import pytest

import oracle
import paper_2209_10643_b200 as U
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(upir):
    c = U.upir_init(0)
    yield c
    U.upir_finalize(c)


def matvec_gpu(ctx, A, x, teams, units, distribute=U.DIST_TEAMS, policy=U.SCHED_STATIC, chunk=0, ic=4,
               lb=0, ub=None, trace=False, simdlen=0):
    M, K = A.shape
    ub = M if ub is None else ub
    y = np.full(M, -3.0, np.float32)
    ma, mx, my = U.upir_data_map(ctx, A, U.MAP_TO), U.upir_data_map(ctx, x, U.MAP_TO), \
        U.upir_data_map(ctx, y, U.MAP_TOFROM)
    T = max(0, ub - lb)
    tr = np.zeros(3 * max(T, 1), np.int32) if trace else None
    tm = U.upir_data_map(ctx, tr, U.MAP_TOFROM) if trace else None
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
    try:
        U.upir_loop_exec(s, U.loop_desc(lb, ub, policy=policy, chunk=chunk, distribute=distribute, inner_chunk=ic, simdlen=simdlen),
                         U.body(U.BODY_MATVEC, U.F32, in0=ma, in1=mx, out=my, ld=(K, 0, 0), dims=(K, M, 0)),
                         trace=tm)
    finally:
        U.upir_spmd_end(s)
        for m in ([tm] if trace else []) + [my, mx, ma]:
            U.upir_data_unmap(ctx, m)
        U.upir_sync(ctx)
    return y, (tr[:T], tr[T:2 * T], tr[2 * T:3 * T]) if trace else None


def check(y, A, x, lb=0, ub=None):
    ub = len(y) if ub is None else ub
    ref = oracle.matvec(A, x, lb, ub, y_in=np.full(len(y), -3.0))
    scale = np.abs(A.astype(np.float64)) @ np.abs(x.astype(np.float64))
    scale[scale == 0] = 1
    assert (np.abs(y - ref) / scale).max() <= 1e-5
    assert (y[:lb] == -3).all() and (y[ub:] == -3).all()


@pytest.mark.parametrize("M,K", [(100, 300), (257, 1000), (64, 4096), (1, 7), (130, 1001), (33, 1)])
@pytest.mark.parametrize("distribute,teams,units", [(U.DIST_TEAMS, 148, 256), (U.DIST_TEAMS, 5, 96),
                                                    (U.DIST_TEAMS_UNITS, 4, 64), (U.DIST_UNITS, 1, 32)])
def test_matvec_parity(ctx, M, K, distribute, teams, units):
    A = synth.f32_sym(3, 0, M * K).reshape(M, K)
    x = synth.f32_sym(1, 0, K)
    y, _ = matvec_gpu(ctx, A, x, teams, units, distribute)
    check(y, A, x)


@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 1), (U.SCHED_STATIC, 3),
                                          (U.SCHED_DYNAMIC, 1), (U.SCHED_DYNAMIC, 4)])
@pytest.mark.parametrize("ic", [4, 1, 7])
def test_matvec_schedules_inner_chunks_subrange(ctx, policy, chunk, ic):
    M, K = 300, 520
    A = synth.f32_sym(3, 0, M * K).reshape(M, K)
    x = synth.f32_sym(1, 0, K)
    y, _ = matvec_gpu(ctx, A, x, 7, 128, policy=policy, chunk=chunk, ic=ic, lb=11, ub=290)
    check(y, A, x, 11, 290)


@pytest.mark.parametrize("distribute,teams,units,chunk", [(U.DIST_TEAMS, 9, 64, 0), (U.DIST_TEAMS, 9, 64, 2),
                                                          (U.DIST_TEAMS_UNITS, 3, 32, 0),
                                                          (U.DIST_TEAMS_UNITS, 3, 32, 5)])
def test_matvec_trace_mapping(ctx, distribute, teams, units, chunk):
    M, K = 200, 64
    A = synth.f32_sym(3, 0, M * K).reshape(M, K)
    x = synth.f32_sym(1, 0, K)
    y, (team, unit, hits) = matvec_gpu(ctx, A, x, teams, units, distribute, chunk=chunk, trace=True)
    assert (hits == 1).all()
    if distribute == U.DIST_TEAMS:
        assert (team == oracle.owner_map(oracle.STATIC, chunk, M, teams)).all()
    else:
        g = team.astype(np.int64) * units + unit
        assert (g == oracle.owner_map(oracle.STATIC, chunk, M, teams * units)).all()


def test_matvec_small_integers_exact(ctx):
    rng = np.random.default_rng(4)
    A = rng.integers(-3, 4, (128, 2048)).astype(np.float32)
    x = rng.integers(-3, 4, 2048).astype(np.float32)
    y, _ = matvec_gpu(ctx, A, x, 16, 256)
    assert (y == (A.astype(np.int64) @ x.astype(np.int64))).all()


@pytest.mark.slow
def test_matvec_full_size_16384_sampled(ctx):
    """The paper's largest matvec size N = 16384."""
    import torch
    n = 16384
    A = torch.empty(n * n, dtype=torch.float32, device="cuda")
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma, mx, my = U.upir_data_adopt(ctx, A), U.upir_data_adopt(ctx, x), U.upir_data_adopt(ctx, y)
    U.upir_synth_fill(ctx, ma, 1, 3)
    U.upir_synth_fill(ctx, mx, 1, 1)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(592, 256))
    U.upir_loop_exec(s, U.loop_desc(0, n, chunk=1, distribute=U.DIST_TEAMS, inner_chunk=4),
                     U.body(U.BODY_MATVEC, U.F32, in0=ma, in1=mx, out=my, ld=(n, 0, 0), dims=(n, n, 0)))
    U.upir_spmd_end(s)
    U.upir_sync(ctx)
    rows = np.array([0, 1, 777, 8191, 16383])
    xh = synth.f32_sym(1, 0, n)
    got = y.cpu().numpy()[rows]
    Ar = np.stack([synth.f32_sym(3, int(r) * n, n) for r in rows])   # the sampled rows of A
    ref = oracle.matvec(Ar, xh)
    scale = np.abs(Ar.astype(np.float64)) @ np.abs(xh.astype(np.float64))
    assert (np.abs(got - ref) <= 1e-5 * scale).all()
    for m in (my, mx, ma):
        U.upir_data_unmap(ctx, m)

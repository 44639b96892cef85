"""GPU parity of the streaming loop bodies (axpy, sum/max reductions) against
the CPU oracle, through the C-ABI.

Tolerances (north_star, reading c22): int64 results and schedule mappings
bit-exact; fp32 max bit-exact; fp32 axpy max|d|/max|ref| <= 1e-5; fp32 sums
|d| / sum|x| <= 1e-5 at these sizes (1e-4 is the bar at >= 1e8 elements).
"""
import numpy as np
import pytest

import oracle
import paper_2209_10643_b200 as U
import synth
from gpu_helpers import flat_unit, run_axpy, run_reduce, upir_path

pytestmark = pytest.mark.gpu

PATHS = ["direct", "staged"]
GEOMS = [(1, 1), (3, 37), (7, 64), (148, 256), (5, 1024)]
SCHEDS = [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 1), (U.SCHED_STATIC, 2), (U.SCHED_STATIC, 3),
          (U.SCHED_STATIC, 64), (U.SCHED_DYNAMIC, 0), (U.SCHED_DYNAMIC, 5), (U.SCHED_DYNAMIC, 100),
          (U.SCHED_RUNTIME, 0)]
OPOL = {U.SCHED_STATIC: oracle.STATIC, U.SCHED_DYNAMIC: oracle.DYNAMIC, U.SCHED_RUNTIME: oracle.RUNTIME,
        U.SCHED_GUIDED: oracle.GUIDED}


@pytest.fixture(scope="module")
def ctx(upir):
    c = U.upir_init(0)
    yield c
    U.upir_finalize(c)


def _p(teams, units, distribute):
    return {U.DIST_TEAMS_UNITS: teams * units, U.DIST_TEAMS: teams, U.DIST_UNITS: units}[distribute]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("teams,units", GEOMS)
@pytest.mark.parametrize("policy,chunk", SCHEDS)
def test_reduce_i64_parity(ctx, path, teams, units, policy, chunk):
    n = 100_003                                     # several tiles + a ragged tail
    x = synth.i64_sym(6, 0, n)
    with upir_path(path):
        (s, mx), _ = run_reduce(ctx, x, [U.OP_SUM, U.OP_MAX], teams, units, policy, chunk)
    p = teams * units
    assert s == oracle.reduce_i64(oracle.SUM, x, policy=OPOL[policy], chunk=chunk, p=p)
    assert mx == oracle.reduce_i64(oracle.MAX, x, policy=OPOL[policy], chunk=chunk, p=p)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("teams,units", [(3, 37), (148, 256)])
@pytest.mark.parametrize("policy,chunk", SCHEDS)
def test_reduce_f32_parity(ctx, path, teams, units, policy, chunk):
    n = 77_777
    x = synth.f32_sym(7, 0, n)
    with upir_path(path):
        (s, mx), _ = run_reduce(ctx, x, [U.OP_SUM, U.OP_MAX], teams, units, policy, chunk)
    p = teams * units
    ref = oracle.reduce_f32(oracle.SUM, x, policy=OPOL[policy], chunk=chunk, p=p)
    assert abs(s - ref) <= 1e-5 * np.abs(x.astype(np.float64)).sum()
    assert mx == oracle.reduce_f32(oracle.MAX, x, policy=OPOL[policy], chunk=chunk, p=p)


@pytest.mark.parametrize("path", PATHS)
def test_reduce_min_and_init(ctx, path):
    x = synth.i64_sym(6, 0, 5000)
    with upir_path(path):
        (mn, s), _ = run_reduce(ctx, x, [U.OP_MIN, U.OP_SUM], 4, 128, inits=[-(1 << 40), 1000])
    assert mn == -(1 << 40)
    assert s == 1000 + int(x.sum())
    xf = synth.f32_unit(7, 0, 3000)
    with upir_path(path):
        (mnf, sf), _ = run_reduce(ctx, xf, [U.OP_MIN, U.OP_SUM], 2, 96, inits=[0.5, 2.5])
    assert mnf == min(0.5, float(xf.min()))
    assert abs(sf - oracle.reduce_f32(oracle.SUM, xf, init=2.5)) <= 1e-6 * (2.5 + xf.sum())


@pytest.mark.parametrize("path", PATHS)
def test_reduce_spec_example_and_closed_forms(ctx, path):
    # SPEC.md:405 reduction(+:sum) over 1..10 with p=3 static -> 55
    x = np.arange(1, 11, dtype=np.int64)
    with upir_path(path):
        assert run_reduce(ctx, x, [U.OP_SUM], 1, 3)[0] == [55]
        n = 1 << 20
        assert run_reduce(ctx, np.arange(1, n + 1, dtype=np.int64), [U.OP_SUM], 148, 256)[0] == [n * (n + 1) // 2]
        y = synth.f32_unit(7, 0, 1 << 20)
        y[777_777] = 2.0
        assert run_reduce(ctx, y, [U.OP_MAX], 148, 256, U.SCHED_DYNAMIC, 3)[0] == [2.0]


@pytest.mark.parametrize("path", PATHS)
def test_empty_and_offsets(ctx, path):
    x = synth.i64_sym(6, 0, 1000)
    with upir_path(path):
        assert run_reduce(ctx, x, [U.OP_SUM], 8, 64, lb=5, ub=5, inits=[7])[0] == [7]
        for lb, ub, step in ((3, 997, 1), (999, 0, -1), (1, 1000, 3), (998, 2, -7)):
            for pol, c in ((U.SCHED_STATIC, 0), (U.SCHED_STATIC, 5), (U.SCHED_DYNAMIC, 2)):
                got = run_reduce(ctx, x, [U.OP_SUM], 3, 32, pol, c, lb=lb, ub=ub, step=step)[0][0]
                exp = oracle.reduce_i64(oracle.SUM, x, lb=lb, ub=ub, step=step, policy=OPOL[pol], chunk=c, p=96)
                assert got == exp, (lb, ub, step, pol, c)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("distribute,teams,units", [(U.DIST_TEAMS, 37, 64), (U.DIST_UNITS, 1, 200),
                                                    (U.DIST_TEAMS_UNITS, 9, 33)])
@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 4), (U.SCHED_STATIC, 50)])
def test_trace_mapping_bit_exact(ctx, path, distribute, teams, units, policy, chunk):
    """Executor of every iteration == the oracle's schedule (static: bit-exact)."""
    n = 20_011
    x = synth.i64_sym(6, 0, n)
    with upir_path(path):
        (s,), (team, unit, hits) = run_reduce(ctx, x, [U.OP_SUM], teams, units, policy, chunk,
                                              distribute=distribute, trace=True)
    p = _p(teams, units, distribute)
    assert (hits == 1).all()                         # exactly once
    g = flat_unit(team, unit, units, distribute)
    assert (g == oracle.owner_map(oracle.STATIC, chunk, n, p)).all()
    if distribute == U.DIST_TEAMS:
        assert (unit == 0).all()                     # reading c6
    assert s == oracle.reduce_i64(oracle.SUM, x, chunk=chunk, p=p)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("chunk", [1, 3, 64, 1000])
def test_trace_dynamic_valid(ctx, path, chunk):
    """dynamic: chunk partition exact, each chunk run by one unit, exactly once
    (reading c8: the unit assignment itself has several correct answers)."""
    n = 50_001
    teams, units = 11, 96
    x = synth.i64_sym(6, 0, n)
    with upir_path(path):
        (s,), (team, unit, hits) = run_reduce(ctx, x, [U.OP_SUM], teams, units, U.SCHED_DYNAMIC, chunk, trace=True)
    assert (hits == 1).all()
    g = flat_unit(team, unit, units, U.DIST_TEAMS_UNITS)
    assert g.min() >= 0 and g.max() < teams * units
    for k in range(0, n, chunk):
        blk = g[k:k + chunk]
        assert (blk == blk[0]).all()
    assert s == int(x.sum())


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("teams,units", [(1, 1), (4, 100), (148, 256)])
@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 4), (U.SCHED_STATIC, 33),
                                          (U.SCHED_DYNAMIC, 1), (U.SCHED_DYNAMIC, 16)])
def test_axpy_parity(ctx, path, teams, units, policy, chunk):
    n = 65_537
    x = synth.f32_unit(1, 0, n)
    y = synth.f32_unit(2, 0, n)
    with upir_path(path):
        yy, s, _ = run_axpy(ctx, 2.0, x, y, teams, units, policy, chunk, sum_=True)
    ref = oracle.axpy(2.0, x, y)
    assert np.abs(yy - ref).max() / np.abs(ref).max() <= 1e-5
    # x, y on the 2^-24 grid: a*x + y is exact in fp32 here -> bit-exact
    assert (yy == ref.astype(np.float32)).all()
    rs = oracle.reduce_f32(oracle.SUM, yy)
    assert abs(s - rs) <= 1e-5 * abs(rs)


@pytest.mark.parametrize("path", PATHS)
def test_axpy_spec_example_and_ranges(ctx, path):
    with upir_path(path):
        yy, _, _ = run_axpy(ctx, 2.0, np.array([1, 2, 3, 4], np.float32), np.ones(4, np.float32), 1, 4)
        assert yy.tolist() == [3, 5, 7, 9]
        x = synth.f32_sym(1, 0, 10_000)
        y = synth.f32_sym(2, 0, 10_000)
        for lb, ub, step in ((13, 9_990, 1), (9_999, 0, -1), (5, 9_000, 7)):
            yy, _, (team, unit, hits) = run_axpy(ctx, -1.5, x, y, 6, 70, lb=lb, ub=ub, step=step, trace=True)
            ref = oracle.axpy(-1.5, x, y, lb=lb, ub=ub, step=step)
            assert np.abs(yy - ref).max() <= 1e-5 * np.abs(ref).max()
            assert (hits == 1).all()
            T = oracle.trip_count(lb, ub, step)
            assert (flat_unit(team, unit, 70, U.DIST_TEAMS_UNITS) == oracle.owner_map(oracle.STATIC, 0, T, 420)).all()


def test_geometry_honoured_exactly(ctx):
    # the paper's CUDA geometry <<<(n+255)/256, 256>>> with the
    # flat index team*units + unit
    n = 10_240
    x = synth.i64_sym(6, 0, n)
    (s,), (team, unit, hits) = run_reduce(ctx, x, [U.OP_SUM], (n + 255) // 256, 256, trace=True)
    assert (team.astype(np.int64) * 256 + unit == np.arange(n)).all()
    with pytest.raises(U.UpirError):
        U.upir_spmd_launch(ctx, U.spmd_desc(1, 1025))


def test_synth_fill_matches_host_generator(ctx):
    import torch
    n = 100_000
    cases = [(0, 7, np.float32, lambda: synth.f32_unit(7, 0, n)),
             (1, 1, np.float32, lambda: synth.f32_sym(1, 0, n)),
             (2, 6, np.int64, lambda: synth.i64_sym(6, 0, n)),
             (3, 3, np.uint16, lambda: (synth.bf16_sym_as_f32(3, 0, n).view(np.uint32) >> 16).astype(np.uint16))]
    for dist, stream, dt, ref in cases:
        h = np.zeros(n, dtype=dt)
        m = U.upir_data_map(ctx, h, U.MAP_FROM)
        U.upir_synth_fill(ctx, m, dist, stream)
        U.upir_data_unmap(ctx, m)
        U.upir_sync(ctx)
        assert (h == ref()).all(), dist
    g = np.zeros((37, 53), np.float32)
    m = U.upir_data_map(ctx, g, U.MAP_FROM)
    U.upir_synth_fill(ctx, m, 4, 5, 0, 37, 53)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    assert (g == synth.jacobi_init(37, 53)).all()
    # golden vectors of the recipe
    h = np.zeros(4, np.int64)
    m = U.upir_data_map(ctx, h, U.MAP_FROM)
    U.upir_synth_fill(ctx, m, 2, 6)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    assert h.tolist() == synth.GOLDEN[(6, "i64")]


# ---- guided ------------------------------------------------
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("teams,units", [(1, 32), (3, 37), (148, 256)])
@pytest.mark.parametrize("chunk", [0, 1, 5, 1000])
def test_guided_reduce_parity_and_chunks(ctx, path, teams, units, chunk):
    n = 60_013
    x = synth.i64_sym(6, 0, n)
    with upir_path(path):
        (s, mx), (team, unit, hits) = run_reduce(ctx, x, [U.OP_SUM, U.OP_MAX], teams, units,
                                                 U.SCHED_GUIDED, chunk, trace=True)
    p = teams * units
    assert s == oracle.reduce_i64(oracle.SUM, x, policy=oracle.GUIDED, chunk=chunk, p=p)
    assert mx == int(x.max())
    assert (hits == 1).all()
    # chunk boundaries are the oracle's guided sequence: every oracle chunk is
    # executed by one unit (reading c8: the assignment itself is decided at run time)
    g = flat_unit(team, unit, units, U.DIST_TEAMS_UNITS)
    bounds = sorted(lo for u in range(p) for lo, hi in oracle.schedule_chunks(oracle.GUIDED, chunk, n, p, u)
                    ) + [n] if p <= 4096 else None
    if bounds is not None:
        for a_, b_ in zip(bounds[:-1], bounds[1:]):
            assert (g[a_:b_] == g[a_]).all()


@pytest.mark.parametrize("path", PATHS)
def test_guided_axpy_f32(ctx, path):
    n = 40_000
    x = synth.f32_sym(1, 0, n)
    y = synth.f32_sym(2, 0, n)
    with upir_path(path):
        yy, s, _ = run_axpy(ctx, 0.5, x, y, 8, 128, U.SCHED_GUIDED, 3, sum_=True)
    ref = oracle.axpy(0.5, x, y)
    assert np.abs(yy - ref).max() <= 1e-5 * np.abs(ref).max()
    assert abs(s - oracle.reduce_f32(oracle.SUM, yy)) <= 1e-5 * np.abs(yy).sum()


# ---- address alignment: an adopted view with a storage
# offset is not 16/32-B aligned by element index; the vector paths must align
# by address (or fall back to scalar accesses when x and y disagree)
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("off", [1, 2, 3, 5])
@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 2), (U.SCHED_STATIC, 4),
                                          (U.SCHED_DYNAMIC, 4)])
def test_reduce_misaligned_adopted_view(ctx, path, off, policy, chunk):
    import torch
    n = 200_003
    xi = synth.i64_sym(6, 0, n + off)
    xf = synth.f32_unit(7, 0, n + off)
    ti = torch.from_numpy(xi).cuda()[off:]
    tf = torch.from_numpy(xf).cuda()[off:]
    r = torch.zeros(4, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    mi, mf = U.upir_data_adopt(ctx, ti), U.upir_data_adopt(ctx, tf)
    b = r.data_ptr()
    with upir_path(path):
        s = U.upir_spmd_launch(ctx, U.spmd_desc(37, 128))
        U.upir_loop_exec(s, U.loop_desc(0, n, policy=policy, chunk=chunk), U.body(U.BODY_REDUCE, U.I64, in0=mi),
                         [U.reduction(U.OP_SUM, U.I64, b), U.reduction(U.OP_MAX, U.I64, b + 8)])
        U.upir_loop_exec(s, U.loop_desc(0, n, policy=policy, chunk=chunk), U.body(U.BODY_REDUCE, U.F32, in0=mf),
                         [U.reduction(U.OP_SUM, U.F32, b + 16), U.reduction(U.OP_MAX, U.F32, b + 24)])
        U.upir_spmd_end(s)
    U.upir_sync(ctx)
    got = r.cpu().numpy()
    assert int(got[0]) == oracle.reduce_i64(oracle.SUM, xi[off:])
    assert int(got[1]) == oracle.reduce_i64(oracle.MAX, xi[off:])
    fs, fm = np.frombuffer(got[2:].tobytes(), np.float32)[[0, 2]]
    rs = oracle.reduce_f32(oracle.SUM, xf[off:])
    assert abs(float(fs) - rs) <= 1e-5 * rs
    assert float(fm) == oracle.reduce_f32(oracle.MAX, xf[off:])
    U.upir_data_unmap(ctx, mf)
    U.upir_data_unmap(ctx, mi)
    U.upir_sync(ctx)


@pytest.mark.parametrize("xoff,yoff", [(1, 1), (1, 2), (0, 3), (5, 5)])
@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 4), (U.SCHED_DYNAMIC, 4)])
def test_axpy_misaligned_adopted_views(ctx, xoff, yoff, policy, chunk):
    import torch
    n = 100_001
    x = synth.f32_unit(1, 0, n + 8)
    y = synth.f32_unit(2, 0, n + 8)
    tx = torch.from_numpy(x).cuda()[xoff:xoff + n]
    ty_base = torch.from_numpy(y).cuda()
    ty = ty_base[yoff:yoff + n]
    r = torch.zeros(1, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    mx, my = U.upir_data_adopt(ctx, tx), U.upir_data_adopt(ctx, ty)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(148, 256))
    U.upir_loop_exec(s, U.loop_desc(0, n, policy=policy, chunk=chunk),
                     U.body(U.BODY_AXPY, U.F32, in0=mx, out=my, alpha=2.0), [U.reduction(U.OP_SUM, U.F32, r)])
    U.upir_spmd_end(s)
    U.upir_sync(ctx)
    full = ty_base.cpu().numpy()
    ref = oracle.axpy(2.0, x[xoff:xoff + n], y[yoff:yoff + n])
    assert (full[yoff:yoff + n] == ref.astype(np.float32)).all()      # 2^-24 grid: exact
    assert (full[:yoff] == y[:yoff]).all() and (full[yoff + n:] == y[yoff + n:]).all()   # nothing else written
    rs = oracle.reduce_f32(oracle.SUM, full[yoff:yoff + n])
    assert abs(r.item() - rs) <= 1e-5 * rs
    U.upir_data_unmap(ctx, my)
    U.upir_data_unmap(ctx, mx)
    U.upir_sync(ctx)

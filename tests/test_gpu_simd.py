"""simd(simdlen) with worksharing (reading c33) on the GPU, through the C-ABI:
the executor of every iteration equals the oracle's strip-mined schedule
(static: bit-exact), dynamic / guided runs keep SIMD groups whole and exact
chunk boundaries, results match the oracle, and the intra-tile / matvec
loops use SIMD groups of positions / rows.
"""
import math

import numpy as np
import pytest

import oracle
import paper_2209_10643_b200 as U
import synth
from gpu_helpers import flat_unit, run_axpy, run_reduce, upir_path
from test_gpu_jacobi import jacobi_gpu
from test_gpu_matvec import check as matvec_check
from test_gpu_matvec import matvec_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(upir):
    c = U.upir_init(0)
    yield c
    U.upir_finalize(c)


def _p(teams, units, distribute):
    return {U.DIST_TEAMS_UNITS: teams * units, U.DIST_TEAMS: teams, U.DIST_UNITS: units}[distribute]


@pytest.mark.parametrize("path", ["direct", "staged"])
@pytest.mark.parametrize("distribute,teams,units", [(U.DIST_TEAMS_UNITS, 9, 33), (U.DIST_TEAMS, 37, 64),
                                                    (U.DIST_UNITS, 1, 200), (U.DIST_TEAMS_UNITS, 148, 256)])
@pytest.mark.parametrize("chunk", [0, 1, 5, 64])
@pytest.mark.parametrize("s", [2, 4, 8])
def test_simd_static_mapping_bit_exact(ctx, path, distribute, teams, units, chunk, s):
    n = 20_011
    x = synth.i64_sym(6, 0, n)
    with upir_path(path):
        (sm,), (team, unit, hits) = run_reduce(ctx, x, [U.OP_SUM], teams, units, U.SCHED_STATIC, chunk,
                                               distribute=distribute, trace=True, simdlen=s)
    p = _p(teams, units, distribute)
    assert (hits == 1).all()
    g = flat_unit(team, unit, units, distribute)
    assert (g == oracle.owner_map(oracle.STATIC, chunk, n, p, simdlen=s)).all()
    assert sm == oracle.reduce_i64(oracle.SUM, x)      # int64: exact in any order


@pytest.mark.parametrize("policy", [U.SCHED_DYNAMIC, U.SCHED_GUIDED])
@pytest.mark.parametrize("chunk", [0, 3, 40])
@pytest.mark.parametrize("s", [4, 16])
def test_simd_dynamic_guided_groups(ctx, policy, chunk, s):
    n = 50_003
    teams, units = 11, 96
    p = teams * units
    x = synth.i64_sym(6, 0, n)
    (sm,), (team, unit, hits) = run_reduce(ctx, x, [U.OP_SUM], teams, units, policy, chunk, trace=True, simdlen=s)
    assert (hits == 1).all()
    assert sm == int(x.sum())
    g = flat_unit(team, unit, units, U.DIST_TEAMS_UNITS)
    opol = oracle.DYNAMIC if policy == U.SCHED_DYNAMIC else oracle.GUIDED
    # the oracle's chunk partition (unit assignment decided at run time, c8)
    chunks = sorted(ch for u in range(p) for ch in oracle.schedule_chunks(opol, chunk, n, p, u, simdlen=s))
    for lo, hi in chunks:
        assert (g[lo:hi] == g[lo]).all()      # a chunk (whole SIMD groups) runs on one unit
    # and runs of one unit start at chunk starts only
    starts = {lo for lo, _ in chunks}
    change = np.flatnonzero(np.diff(g)) + 1
    assert set(change.tolist()) <= starts


@pytest.mark.parametrize("s", [4, 8])
def test_simd_axpy_and_f32(ctx, s):
    n = 65_537
    x = synth.f32_unit(1, 0, n)
    y = synth.f32_unit(2, 0, n)
    yy, ysum, _ = run_axpy(ctx, 2.0, x, y, 148, 256, U.SCHED_STATIC, 0, sum_=True, simdlen=s)
    ref = oracle.axpy(2.0, x, y)
    assert np.abs(yy - ref).max() <= 1e-5 * np.abs(ref).max()
    assert abs(ysum - ref.sum()) <= 1e-5 * np.abs(ref).sum()
    xf = synth.f32_sym(7, 0, 77_777)
    (sm, mx), _ = run_reduce(ctx, xf, [U.OP_SUM, U.OP_MAX], 148, 256, U.SCHED_STATIC, 3, simdlen=s)
    assert abs(sm - oracle.reduce_f32(oracle.SUM, xf)) <= 1e-5 * np.abs(xf.astype(np.float64)).sum()
    assert mx == float(xf.max())


@pytest.mark.parametrize("ic,s", [(1, 4), (4, 8), (3, 2)])
def test_simd_intra_tile_groups(ctx, ic, s):
    # JACOBI5: the intra-tile position loop uses SIMD groups: static,ic
    # becomes static,s*ceil(ic/s) (the oracle rule pinned in test_oracle_schedule)
    g = synth.jacobi_init(75, 300)
    teams, units, tile = 5, 96, (32, 128)
    out, tr = jacobi_gpu(ctx, g, 1, teams=teams, units=units, tile=tile, ic=ic, trace=True, simdlen=s)
    n = len(tr) // 3
    team, unit, hits = tr[:n], tr[n:2 * n], tr[2 * n:]
    ot, ou = oracle.tiled_owner(1, 74, 1, 299, tile[0], tile[1], oracle.STATIC, 1, teams, s * math.ceil(ic / s),
                                units)
    it = ot >= 0
    assert (hits[it] == 1).all() and (team[it] == ot[it]).all() and (unit[it] == ou[it]).all()
    ref = oracle.jacobi5(g, 1)
    assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 3)])
def test_simd_matvec_rows(ctx, policy, chunk):
    M, K, s = 301, 77, 4
    A = synth.f32_sym(3, 0, M * K).reshape(M, K)
    x = synth.f32_sym(1, 0, K)
    y, (team, unit, hits) = matvec_gpu(ctx, A, x, 3, 32, distribute=U.DIST_TEAMS_UNITS, policy=policy,
                                       chunk=chunk, trace=True, simdlen=s)
    matvec_check(y, A, x)
    assert (hits == 1).all()
    g = team.astype(np.int64) * 32 + unit
    assert (g == oracle.owner_map(oracle.STATIC, chunk, M, 96, simdlen=s)).all()
    # distribute(teams): SIMD groups of the k-loop (values only)
    y2, _ = matvec_gpu(ctx, A, x, 7, 64, distribute=U.DIST_TEAMS, ic=3, simdlen=8)
    matvec_check(y2, A, x)

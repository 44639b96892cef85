"""GPU parity of the JACOBI5 loop body (tiled collapse(2) upir.loop with TMA
staging) against the fp64 oracle, through the C-ABI.

Tolerance (north_star; reading c22): max|d| / max|ref| <= 1e-5 for fp32
Jacobi against fp64.  Invariants hold bit-exactly (harmonic fixed points,
boundary unchanged); the tile -> team and position -> unit mapping of the
static schedules is bit-exact; full size (8192^2 x 100 sweeps) is checked on
light-cone windows (reading c16, c25).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2209_10643_b200 as U
import synth

pytestmark = pytest.mark.gpu

OPOL = {U.SCHED_STATIC: oracle.STATIC, U.SCHED_DYNAMIC: oracle.DYNAMIC}


@pytest.fixture(scope="module")
def ctx(upir):
    c = U.upir_init(0)
    yield c
    U.upir_finalize(c)


def jacobi_gpu(ctx, g, S, teams=8, units=256, tile=(32, 256), policy=U.SCHED_STATIC, chunk=1, ic=4,
               space=None, graph=False, trace=False, simdlen=0, flags=0):
    """Run S ping-pong sweeps; returns (grid after S sweeps, trace or None)."""
    ny, nx = g.shape
    a, b = g.copy(), g.copy()
    ma = U.upir_data_map(ctx, a, U.MAP_TOFROM)
    mb = U.upir_data_map(ctx, b, U.MAP_TOFROM)
    (lb0, ub0, lb1, ub1) = space or (1, ny - 1, 1, nx - 1)
    loop = U.loop_desc([lb0, lb1], [ub0, ub1], tile=list(tile), policy=policy, chunk=chunk,
                       distribute=U.DIST_TEAMS, inner_chunk=ic, simdlen=simdlen, flags=flags)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
    tr = tm = None
    if trace:
        nt = (((ub0 + tile[0] - 1) // tile[0]) - lb0 // tile[0]) * (((ub1 + tile[1] - 1) // tile[1]) - lb1 // tile[1])
        tr = np.zeros(3 * nt * tile[0] * tile[1], np.int32)
        tm = U.upir_data_map(ctx, tr, U.MAP_TOFROM)
    bodies = [U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(nx, 0, 0), dims=(ny, 0, 0)),
              U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(nx, 0, 0), dims=(ny, 0, 0))]
    gr = None
    try:
        if graph:
            U.upir_graph_begin(ctx)
        for k in range(S):
            U.upir_loop_exec(s, loop, bodies[k % 2], trace=tm if k == 0 else None)
        if graph:
            gr = U.upir_graph_end(ctx)
            U.upir_graph_launch(ctx, gr)
    finally:
        U.upir_spmd_end(s)
        if tm is not None:
            U.upir_data_unmap(ctx, tm)
        U.upir_data_unmap(ctx, mb)
        U.upir_data_unmap(ctx, ma)
        U.upir_sync(ctx)
    if gr is not None:
        U.upir_graph_destroy(gr)
    return (b if S % 2 else a), tr


def rel(x, ref):
    return np.abs(x.astype(np.float64) - ref).max() / np.abs(ref).max()


@pytest.mark.parametrize("tile", [(32, 256), (32, 128), (16, 256), (64, 128), (8, 64)])
@pytest.mark.parametrize("shape", [(70, 300), (33, 68), (129, 516)])
def test_jacobi_parity_tiles(ctx, tile, shape):
    g = synth.jacobi_init(*shape)
    out, _ = jacobi_gpu(ctx, g, 5, tile=tile)
    ref = oracle.jacobi5(g, 5)
    assert rel(out, ref) <= 1e-5
    for sl in (np.s_[0, :], np.s_[-1, :], np.s_[:, 0], np.s_[:, -1]):
        assert (out[sl] == g[sl]).all()          # Dirichlet boundary unchanged


@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 1), (U.SCHED_STATIC, 3),
                                          (U.SCHED_DYNAMIC, 1), (U.SCHED_DYNAMIC, 2)])
@pytest.mark.parametrize("teams,units", [(1, 32), (7, 256), (148, 128), (3, 1024)])
def test_jacobi_parity_schedules(ctx, policy, chunk, teams, units):
    g = synth.jacobi_init(100, 520)
    out, _ = jacobi_gpu(ctx, g, 3, teams=teams, units=units, policy=policy, chunk=chunk)
    assert rel(out, oracle.jacobi5(g, 3)) <= 1e-5


@pytest.mark.parametrize("ic", [1, 3, 4, 64])
def test_jacobi_inner_chunks_and_subspace(ctx, ic):
    g = synth.jacobi_init(90, 200)
    space = (5, 77, 9, 190)           # a sub-rectangle of the interior
    out, _ = jacobi_gpu(ctx, g, 1, ic=ic, space=space)
    ref = g.astype(np.float64).copy()
    full = oracle.jacobi5(g, 1)
    ref[5:77, 9:190] = full[5:77, 9:190]
    assert rel(out, ref) <= 1e-5
    mask = np.ones_like(g, bool)
    mask[5:77, 9:190] = False
    assert (out[mask] == g[mask]).all()


@pytest.mark.parametrize("name", ["constant", "linear", "bilinear"])
def test_jacobi_fixed_points_bit_exact(ctx, name):
    n = 160
    i = np.arange(n)[:, None].astype(np.float64)
    j = np.arange(n)[None, :].astype(np.float64)
    f = {"constant": np.full((n, n), 0.75), "linear": 3 * i + 5 * j + 7,
         "bilinear": (i - 80) * (j - 80)}[name].astype(np.float32)
    out, _ = jacobi_gpu(ctx, f, 4, tile=(32, 128))
    assert (out == f).all()


def test_jacobi_eigenmode(ctx):
    N, k, l, S = 260, 9, 5, 60
    ii = np.arange(N)[:, None]
    jj = np.arange(N)[None, :]
    g = (np.sin(k * np.pi * ii / (N - 1)) * np.sin(l * np.pi * jj / (N - 1))).astype(np.float32)
    out, _ = jacobi_gpu(ctx, g, S, tile=(32, 128))
    lam = (np.cos(k * np.pi / (N - 1)) + np.cos(l * np.pi / (N - 1))) / 2
    assert np.abs(out - g.astype(np.float64) * lam ** S).max() <= 1e-5


@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 1), (U.SCHED_STATIC, 0), (U.SCHED_STATIC, 2)])
@pytest.mark.parametrize("ic", [4, 3])
def test_jacobi_trace_mapping(ctx, policy, chunk, ic):
    g = synth.jacobi_init(75, 300)
    teams, units, tile = 5, 96, (32, 128)
    _, tr = jacobi_gpu(ctx, g, 1, teams=teams, units=units, tile=tile, policy=policy, chunk=chunk, ic=ic,
                       trace=True)
    n = len(tr) // 3
    team, unit, hits = tr[:n], tr[n:2 * n], tr[2 * n:]
    ot, ou = oracle.tiled_owner(1, 74, 1, 299, tile[0], tile[1], OPOL[policy], chunk, teams, ic, units)
    it = ot >= 0
    assert (hits[it] == 1).all() and (hits[~it] == 0).all()
    assert (team[it] == ot[it]).all()
    assert (unit[it] == ou[it]).all()


def test_jacobi_graph_equals_eager(ctx):
    g = synth.jacobi_init(300, 600)
    a, _ = jacobi_gpu(ctx, g, 20)
    b, _ = jacobi_gpu(ctx, g, 20, graph=True)
    assert (a == b).all()


def test_jacobi_rejects_bad_space(ctx):
    g = synth.jacobi_init(40, 64)
    with pytest.raises(U.UpirError):
        jacobi_gpu(ctx, g, 1, space=(0, 39, 1, 63))      # row 0 has no north neighbour
    with pytest.raises(U.UpirError):
        jacobi_gpu(ctx, g, 1, tile=(24, 100))            # tile not built


@pytest.mark.slow
def test_jacobi_full_size_windows(ctx):
    """C3 at full size: 8192^2, 100 sweeps (graph), static,1 tiles over 296
    teams -- checked against the oracle on light-cone windows."""
    import torch
    ny = nx = 8192
    S = 100
    a_t = torch.empty(ny * nx, dtype=torch.float32, device="cuda")
    b_t = torch.empty(ny * nx, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma = U.upir_data_adopt(ctx, a_t)
    mb = U.upir_data_adopt(ctx, b_t)
    U.upir_synth_fill(ctx, ma, 4, 5, 0, ny, nx)
    U.upir_synth_fill(ctx, mb, 4, 5, 0, ny, nx)
    loop = U.loop_desc([1, 1], [ny - 1, nx - 1], tile=[32, 256], policy=U.SCHED_STATIC, chunk=1,
                       distribute=U.DIST_TEAMS, inner_chunk=4)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(296, 256))
    bodies = [U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(nx, 0, 0), dims=(ny, 0, 0)),
              U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(nx, 0, 0), dims=(ny, 0, 0))]
    for k in range(S):
        U.upir_loop_exec(s, loop, bodies[k % 2])
    U.upir_spmd_end(s)
    U.upir_sync(ctx)
    res = a_t.view(ny, nx)
    for (r0, c0) in ((0, 0), (4000, 4093), (8192 - 16, 8192 - 16), (31, 255), (1000, 7000)):
        r1, c1 = r0 + 16, c0 + 16
        wr0, wr1 = max(0, r0 - S), min(ny, r1 + S)
        wc0, wc1 = max(0, c0 - S), min(nx, c1 + S)
        win = synth.jacobi_init_rows(ny, nx, wr0, wr1)[:, wc0:wc1]
        ref = oracle.jacobi5_window(ny, nx, S, wr0, wc0, win)[r0 - wr0:r1 - wr0, c0 - wc0:c1 - wc0]
        got = res[r0:r1, c0:c1].cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max()), (r0, c0)
    U.upir_data_unmap(ctx, mb)
    U.upir_data_unmap(ctx, ma)


@pytest.mark.parametrize("teams,units,tile", [(148, 256, (16, 256)), (444, 256, (16, 256)), (9, 128, (32, 128))])
def test_jacobi_ring_depths_identical(ctx, monkeypatch, teams, units, tile):
    """The window ring depth (2, 3, 4 slots; launcher's choice = 0) is a
    staging choice only: results are bit-identical and match the oracle."""
    g = synth.jacobi_init(203, 1028)
    outs = []
    for nst in ("0", "2", "3", "4"):
        monkeypatch.setenv("UPIR_JACOBI_NST", nst)
        out, _ = jacobi_gpu(ctx, g, 4, teams=teams, units=units, tile=tile)
        outs.append(out)
    assert rel(outs[0], oracle.jacobi5(g, 4)) <= 1e-5
    for o in outs[1:]:
        assert (o == outs[0]).all()


@pytest.mark.parametrize("teams,units", [(5, 100), (3, 33), (2, 1000)])
def test_jacobi_ragged_team_sizes(ctx, teams, units):
    """Team sizes that are not a multiple of the warp (the producer warp sits
    after the last partial warp; the units' interior fast path needs whole
    warps, so these run the checked path) -- and > 992 units (no producer
    warp: thread 0 produces between its own tiles)."""
    g = synth.jacobi_init(97, 516)
    out, tr = jacobi_gpu(ctx, g, 2, teams=teams, units=units, tile=(16, 256), trace=True)
    assert rel(out, oracle.jacobi5(g, 2)) <= 1e-5
    team, unit, hits = tr.reshape(3, -1)
    assert (unit[hits > 0] < units).all() and (team[hits > 0] < teams).all()


def test_jacobi_interior_fast_path_matches_checked(ctx):
    """Interior tiles (lean path: shuffled west / east neighbours) and the
    checked path (forced by a trace run) give bit-identical grids."""
    g = synth.jacobi_init(300, 1100)
    fast, _ = jacobi_gpu(ctx, g, 1, teams=37, units=256, tile=(16, 256))
    checked, _ = jacobi_gpu(ctx, g, 1, teams=37, units=256, tile=(16, 256), trace=True)
    assert (fast == checked).all()
    assert rel(fast, oracle.jacobi5(g, 1)) <= 1e-5


# ---- reading c35: column-major tile ids (UPIR_TILE_COLMAJOR) --------------------
@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 1), (U.SCHED_STATIC, 3),
                                          (U.SCHED_DYNAMIC, 2)])
def test_jacobi_colmajor_parity_and_trace(ctx, policy, chunk):
    """Column-major tile ids: same grid as the row-major order (bit-exact: the
    order only moves work between teams), tile -> team / position -> unit
    map bit-exact against the oracle's column-major enumeration (dynamic:
    the position -> unit map and coverage)."""
    g = synth.jacobi_init(150, 520)
    teams, units, tile = 7, 128, (16, 256)
    rowm, _ = jacobi_gpu(ctx, g, 3, teams=teams, units=units, tile=tile, policy=policy, chunk=chunk)
    colm, _ = jacobi_gpu(ctx, g, 3, teams=teams, units=units, tile=tile, policy=policy, chunk=chunk,
                         flags=U.TILE_COLMAJOR)
    assert (colm == rowm).all()
    assert rel(colm, oracle.jacobi5(g, 3)) <= 1e-5
    _, tr = jacobi_gpu(ctx, g, 1, teams=teams, units=units, tile=tile, policy=policy, chunk=chunk,
                       trace=True, flags=U.TILE_COLMAJOR)
    n = len(tr) // 3
    team, unit, hits = tr[:n], tr[n:2 * n], tr[2 * n:]
    ot, ou = oracle.tiled_owner(1, 149, 1, 519, tile[0], tile[1], OPOL[policy], chunk, teams, 4, units,
                                colmajor=True)
    it = ot >= 0
    assert (hits[it] == 1).all() and (hits[~it] == 0).all()
    assert (unit[it] == ou[it]).all()
    if policy == U.SCHED_STATIC:
        assert (team[it] == ot[it]).all()


def test_colmajor_rejected_for_other_bodies(ctx):
    x = np.zeros(1024, np.float32)
    m = U.upir_data_map(ctx, x, U.MAP_TO)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(4, 128))
    r = torch.zeros(1, dtype=torch.float32, device="cuda")
    with pytest.raises(U.UpirError):
        U.upir_loop_exec(s, U.loop_desc(0, 1024, flags=U.TILE_COLMAJOR), U.body(U.BODY_REDUCE, U.F32, in0=m),
                         [U.reduction(U.OP_SUM, U.F32, r)])
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)


@pytest.mark.parametrize("colmajor", [False, True])
@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 1), (U.SCHED_STATIC, 0), (U.SCHED_DYNAMIC, 1)])
def test_jacobi_reverse_order_parity_and_trace(ctx, colmajor, policy, chunk):
    """UPIR_TILE_REVERSE (reading c38): the same grid as the plain order, bit
    for bit (the order only moves work in time / between teams); the tile ->
    team and position -> unit maps bit-exact against the oracle's reversed
    enumeration (dynamic: position -> unit and coverage)."""
    g = synth.jacobi_init(150, 520)
    teams, units, tile = 7, 128, (16, 256)
    base = U.TILE_COLMAJOR if colmajor else 0
    plain, _ = jacobi_gpu(ctx, g, 3, teams=teams, units=units, tile=tile, policy=policy, chunk=chunk, flags=base)
    rev, _ = jacobi_gpu(ctx, g, 3, teams=teams, units=units, tile=tile, policy=policy, chunk=chunk,
                        flags=base | U.TILE_REVERSE)
    assert (rev == plain).all()
    assert rel(rev, oracle.jacobi5(g, 3)) <= 1e-5
    _, tr = jacobi_gpu(ctx, g, 1, teams=teams, units=units, tile=tile, policy=policy, chunk=chunk,
                       trace=True, flags=base | U.TILE_REVERSE)
    n = len(tr) // 3
    team, unit, hits = tr[:n], tr[n:2 * n], tr[2 * n:]
    ot, ou = oracle.tiled_owner(1, 149, 1, 519, tile[0], tile[1], OPOL[policy], chunk, teams, 4, units,
                                colmajor=colmajor, reverse=True)
    it = ot >= 0
    assert (hits[it] == 1).all() and (hits[~it] == 0).all()
    assert (unit[it] == ou[it]).all()
    if policy == U.SCHED_STATIC:
        assert (team[it] == ot[it]).all()


def test_jacobi_alternating_order_sweeps_equal_plain(ctx):
    """bench.py's C3 form: sweeps alternating the plain and the reversed tile
    order in one CUDA graph give the plain sweeps' grid bit for bit."""
    g = synth.jacobi_init(203, 1028)
    ny, nx = g.shape
    outs = []
    for alternate in (False, True):
        a, b = g.copy(), g.copy()
        ma, mb = U.upir_data_map(ctx, a, U.MAP_TOFROM), U.upir_data_map(ctx, b, U.MAP_TOFROM)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(9, 256))
        loops = [U.loop_desc([1, 1], [ny - 1, nx - 1], tile=[16, 256], chunk=1, distribute=U.DIST_TEAMS,
                             inner_chunk=4, flags=f) for f in (0, U.TILE_REVERSE)]
        bodies = [U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(nx, 0, 0), dims=(ny, 0, 0)),
                  U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(nx, 0, 0), dims=(ny, 0, 0))]
        U.upir_graph_begin(ctx)
        for k in range(10):
            U.upir_loop_exec(s, loops[k % 2] if alternate else loops[0], bodies[k % 2])
        gr = U.upir_graph_end(ctx)
        U.upir_graph_launch(ctx, gr)
        U.upir_sync(ctx)
        U.upir_graph_destroy(gr)
        U.upir_spmd_end(s)
        U.upir_data_unmap(ctx, mb)
        U.upir_data_unmap(ctx, ma)
        U.upir_sync(ctx)
        outs.append(a)
    assert (outs[0] == outs[1]).all()
    assert rel(outs[1], oracle.jacobi5(g, 10)) <= 1e-5


def test_reverse_rejected_for_other_bodies_and_subspace_parity(ctx):
    """UPIR_TILE_REVERSE is a JACOBI5 tile order: other bodies reject it
    (UPIR_E_UNSUPPORTED, no side effect); on a sub-space that starts and ends
    mid-tile the reversed order writes exactly the iterations of the plain
    order."""
    x = np.zeros(1024, np.float32)
    m = U.upir_data_map(ctx, x, U.MAP_TO)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(4, 128))
    r = torch.zeros(1, dtype=torch.float32, device="cuda")
    with pytest.raises(U.UpirError) as ei:
        U.upir_loop_exec(s, U.loop_desc(0, 1024, flags=U.TILE_REVERSE), U.body(U.BODY_REDUCE, U.F32, in0=m),
                         [U.reduction(U.OP_SUM, U.F32, r)])
    assert ei.value.status == U.E_UNSUPPORTED
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    g = synth.jacobi_init(120, 700)
    space = (7, 101, 13, 650)
    plain, _ = jacobi_gpu(ctx, g, 2, teams=5, units=256, tile=(16, 256), space=space)
    rev, _ = jacobi_gpu(ctx, g, 2, teams=5, units=256, tile=(16, 256), space=space, flags=U.TILE_REVERSE)
    assert (rev == plain).all()

"""GPU parity of upir.data map semantics (o9, reading c18/c19) and of the
CLUSTER-target code paths at world size 1, through the C-ABI."""
import numpy as np
import pytest
import torch

import oracle
import paper_2209_10643_b200 as U
import synth
from oracle.mapspace import MapSpace

pytestmark = pytest.mark.gpu


@pytest.fixture()
def ctx(upir):
    c = U.upir_init(0)
    yield c
    U.upir_finalize(c)


def test_to_from_round_trip_and_counters(ctx):
    x = synth.f32_sym(1, 0, 10_000)
    y = x.copy()
    m = U.upir_data_map(ctx, y, U.MAP_TOFROM)
    st = U.upir_ctx_stats(ctx)
    assert st["h2d_bytes"] == x.nbytes and st["live_maps"] == 1
    y[:] = 0                                 # host copy changes; device keeps the data
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    assert (y == x).all()                    # tofrom: copied back at exit
    st = U.upir_ctx_stats(ctx)
    assert st["d2h_bytes"] == x.nbytes and st["live_maps"] == 0


def test_present_table_refcount_copies_once(ctx):
    # reading c18 vs the oracle's MapSpace on the same sequence
    orc = MapSpace()
    x = np.arange(1000, dtype=np.float64)
    orc.host_buffer("x", x)
    m1 = U.upir_data_map(ctx, x, U.MAP_TOFROM)
    orc.enter("x", oracle.mapspace.TOFROM)
    m2 = U.upir_data_map(ctx, x, U.MAP_TOFROM)   # present: refcount only
    orc.enter("x", oracle.mapspace.TOFROM)
    assert m1.value == m2.value
    U.upir_data_unmap(ctx, m2)
    orc.exit("x")
    st = U.upir_ctx_stats(ctx)
    assert st["live_maps"] == 1 and st["d2h_bytes"] == 0
    U.upir_data_unmap(ctx, m1)
    orc.exit("x")
    U.upir_sync(ctx)
    st = U.upir_ctx_stats(ctx)
    assert st["h2d_bytes"] == orc.h2d and st["d2h_bytes"] == orc.d2h


def test_alloc_and_from_do_not_copy_in(ctx):
    a = np.full(4096, 7, np.int64)
    m = U.upir_data_map(ctx, a, U.MAP_ALLOC)
    b = np.full(4096, 9, np.int64)
    mf = U.upir_data_map(ctx, b, U.MAP_FROM)
    assert U.upir_ctx_stats(ctx)["h2d_bytes"] == 0
    # the loop writes the FROM buffer: fill it on the device, then exit copies back
    U.upir_synth_fill(ctx, mf, 2, 6)
    U.upir_data_unmap(ctx, mf)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    assert (b == synth.i64_sym(6, 0, 4096)).all()
    assert (a == 7).all()                    # alloc: never copied back


def test_update_directions(ctx):
    x = np.arange(256, dtype=np.int64)
    m = U.upir_data_map(ctx, x, U.MAP_TO)
    x[:] = -5
    U.upir_data_update(ctx, m, 0)            # forward: host -> device
    r = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    s = U.upir_spmd_launch(ctx, U.spmd_desc(2, 64))
    U.upir_loop_exec(s, U.loop_desc(0, 256), U.body(U.BODY_REDUCE, U.I64, in0=m), [U.reduction(U.OP_SUM, U.I64, r)])
    U.upir_spmd_end(s)
    U.upir_sync(ctx)
    assert r.item() == -5 * 256
    U.upir_synth_fill(ctx, m, 2, 6)
    U.upir_data_update(ctx, m, 1)            # backward: device -> host
    U.upir_sync(ctx)
    assert (x == synth.i64_sym(6, 0, 256)).all()
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)


def test_errors_not_mapped_leak_and_sync(upir):
    c = U.upir_init(0)
    x = np.zeros(16, np.int64)
    m = U.upir_data_map(c, x, U.MAP_TO)
    U.upir_data_unmap(c, m)
    s = U.upir_spmd_launch(c, U.spmd_desc(1, 32))
    with pytest.raises(U.UpirError) as ei:         # body names an unmapped buffer
        U.upir_loop_exec(s, U.loop_desc(0, 16), U.body(U.BODY_REDUCE, U.I64, in0=m),
                         [U.reduction(U.OP_SUM, U.I64, 0)])
    assert ei.value.status == U.E_NOT_MAPPED
    U.upir_spmd_end(s)
    with pytest.raises(U.UpirError) as ei:         # wait without arrive
        U.upir_sync(c, U.SYNC_WAIT)
    assert ei.value.status == U.E_SYNC
    tok = U.upir_sync(c, U.SYNC_ARRIVE)
    U.upir_sync(c, U.SYNC_WAIT, token=tok)
    m2 = U.upir_data_map(c, x, U.MAP_TO)
    with pytest.raises(U.UpirError) as ei:         # finalize with a live map
        U.upir_finalize(c)
    assert ei.value.status == U.E_LEAK
    U.upir_data_unmap(c, m2)
    U.upir_finalize(c)


def test_cluster_target_world1_reduce_and_world_combine(ctx):
    n = 50_000
    x = synth.i64_sym(6, 0, n)
    d = U.dist(n, 1, 8)
    m = U.upir_data_map(ctx, x, U.MAP_TO, d)
    _, local, off = U.upir_data_device_ptr(m)
    assert local == n and off == 0
    r = torch.zeros(4, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    s = U.upir_spmd_launch(ctx, U.spmd_desc(16, 128, U.TARGET_CLUSTER))
    U.upir_loop_exec(s, U.loop_desc(0, n), U.body(U.BODY_REDUCE, U.I64, in0=m),
                     [U.reduction(U.OP_SUM, U.I64, r.data_ptr()), U.reduction(U.OP_MAX, U.I64, r.data_ptr() + 8)])
    U.upir_spmd_end(s)
    U.upir_reduce(ctx, U.OP_SUM, U.I64, r.data_ptr(), 1, r.data_ptr() + 16, U.SCOPE_WORLD)
    U.upir_reduce(ctx, U.OP_MAX, U.I64, r.data_ptr() + 8, 1, r.data_ptr() + 24, U.SCOPE_WORLD)
    U.upir_sync(ctx, U.SYNC_WORLD_BARRIER)
    got = r.cpu().tolist()
    assert got[2] == oracle.world_reduce(oracle.SUM, [oracle.reduce_i64(oracle.SUM, x)]) == got[0]
    assert got[3] == int(x.max())
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)


def test_device_scope_reduce(ctx):
    x = torch.from_numpy(synth.f32_sym(7, 0, 1_000_003)).cuda()
    xi = torch.from_numpy(synth.i64_sym(6, 0, 777_777)).cuda()
    out = torch.zeros(2, dtype=torch.float32, device="cuda")
    outi = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    U.upir_reduce(ctx, U.OP_SUM, U.F32, x, x.numel(), out, U.SCOPE_DEVICE)
    U.upir_sync(ctx)
    U.upir_reduce(ctx, U.OP_MAX, U.F32, x, x.numel(), out.data_ptr() + 4, U.SCOPE_DEVICE)
    U.upir_sync(ctx)
    U.upir_reduce(ctx, U.OP_MIN, U.I64, xi, xi.numel(), outi, U.SCOPE_DEVICE)
    U.upir_sync(ctx)
    xs = x.cpu().numpy()
    assert abs(out[0].item() - oracle.reduce_f32(oracle.SUM, xs)) <= 1e-5 * np.abs(xs).sum()
    assert out[1].item() == float(xs.max())
    assert outi.item() == int(xi.cpu().numpy().min())


def test_cluster_jacobi_world1_with_halo_sync(ctx):
    ny, nx, S = 66, 132, 4
    g = synth.jacobi_init(ny, nx)
    a, b = g.copy(), g.copy()
    d = U.dist(ny, nx, 4, halo_rows=1)
    ma = U.upir_data_map(ctx, a, U.MAP_TOFROM, d)
    mb = U.upir_data_map(ctx, b, U.MAP_TOFROM, d)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(8, 256, U.TARGET_CLUSTER))
    loop = U.loop_desc([1, 1], [ny - 1, nx - 1], tile=[32, 128], distribute=U.DIST_TEAMS, inner_chunk=4)
    src, dst = ma, mb
    for _ in range(S):
        U.upir_sync(ctx, U.SYNC_HALO, halo_map=src)     # no-op at world size 1
        U.upir_loop_exec(s, loop, U.body(U.BODY_JACOBI5, U.F32, in0=src, out=dst, ld=(nx, 0, 0), dims=(ny, 0, 0)))
        src, dst = dst, src
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, mb)
    U.upir_data_unmap(ctx, ma)
    U.upir_sync(ctx)
    ref = oracle.jacobi5(g, S)
    assert np.abs(a - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.parametrize("teams,units", [(1, 1), (148 * 4, 256)])
def test_c1_axpy_sum_1e6(ctx, teams, units):
    """BASELINE configs[0]: axpy + fp32 sum, n = 1,000,000, static schedule;
    literal 1 unit and the default geometry (reading c21)."""
    from gpu_helpers import run_axpy
    n = 1_000_000
    x = synth.f32_unit(1, 0, n)
    y = synth.f32_unit(2, 0, n)
    yy, s, (team, unit, hits) = run_axpy(ctx, 2.0, x, y, teams, units, sum_=True, trace=True)
    ref = oracle.axpy(2.0, x, y)
    assert (yy == ref.astype(np.float32)).all()          # exact on the 2^-24 grid
    assert abs(s - oracle.reduce_f32(oracle.SUM, yy, p=teams * units)) <= 1e-5 * abs(s)
    assert (hits == 1).all()
    g = team.astype(np.int64) * units + unit
    assert (g == oracle.owner_map(oracle.STATIC, 0, n, teams * units)).all()


# ---- NEXT #1: async two-step sync and chunk-pipelined map -----------------------
@pytest.mark.parametrize("direction", [U.UPDATE_FORWARD, U.UPDATE_FORWARD_ASYNC])
def test_pipelined_map_sections_reduce(ctx, direction):
    """map(alloc) + per-section forward update + a loop over that section:
    the loop of section k waits only for copy k (overlap), results combine
    with a device-scope upir_reduce.  FORWARD_ASYNC copies are not ordered
    after the earlier section loops (they run back to back on the copy
    stream); the result is the same."""
    n, K = 1_000_000, 8
    x = synth.i64_sym(6, 0, n)
    m = U.upir_data_map(ctx, x, U.MAP_ALLOC)
    parts = torch.zeros(K, dtype=torch.int64, device="cuda")
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    s = U.upir_spmd_launch(ctx, U.spmd_desc(148, 256))
    bounds = np.linspace(0, n, K + 1).astype(np.int64)
    for k in range(K):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        U.upir_data_update_section(ctx, m, lo * 8, (hi - lo) * 8, direction)
        U.upir_loop_exec(s, U.loop_desc(lo, hi), U.body(U.BODY_REDUCE, U.I64, in0=m),
                         [U.reduction(U.OP_SUM, U.I64, parts.data_ptr() + 8 * k)])
    U.upir_spmd_end(s)
    U.upir_reduce(ctx, U.OP_SUM, U.I64, parts, K, total, U.SCOPE_DEVICE)
    U.upir_sync(ctx)
    assert total.item() == oracle.reduce_i64(oracle.SUM, x)
    assert U.upir_ctx_stats(ctx)["h2d_bytes"] == x.nbytes
    # backward section update
    y = np.zeros(1000, np.int64)
    my = U.upir_data_map(ctx, y, U.MAP_ALLOC)
    U.upir_synth_fill(ctx, my, 2, 6)
    U.upir_data_update_section(ctx, my, 800, 1600, 1)     # elements [100, 300)
    U.upir_sync(ctx)
    ref = synth.i64_sym(6, 0, 1000)
    assert (y[100:300] == ref[100:300]).all() and (y[:100] == 0).all() and (y[300:] == 0).all()
    with pytest.raises(U.UpirError):
        U.upir_data_update_section(ctx, my, 7000, 2000, 0)
    U.upir_data_unmap(ctx, my)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)


def test_async_halo_join_overlapped_sweeps(ctx):
    """Per sweep: HALO arrive-compute (async) -> interior rows -> JOIN
    (wait-release on the device) -> boundary rows; equals plain sweeps bit for
    bit (world size 1: the exchange is empty, the ordering is exercised)."""
    ny, nx, S = 70, 264, 6
    g = synth.jacobi_init(ny, nx)
    d = U.dist(ny, nx, 4, halo_rows=1)

    def run(split):
        a, b = g.copy(), g.copy()
        ma = U.upir_data_map(ctx, a, U.MAP_TOFROM, d)
        mb = U.upir_data_map(ctx, b, U.MAP_TOFROM, d)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(6, 256, U.TARGET_CLUSTER))
        src, dst = ma, mb
        for _ in range(S):
            body = U.body(U.BODY_JACOBI5, U.F32, in0=src, out=dst, ld=(nx, 0, 0), dims=(ny, 0, 0))
            if split:
                tok = U.upir_sync(ctx, U.SYNC_HALO, halo_map=src, async_=True)
                U.upir_loop_exec(s, U.loop_desc([2, 1], [ny - 2, nx - 1], tile=[16, 256], distribute=U.DIST_TEAMS,
                                                inner_chunk=4), body)
                U.upir_sync(ctx, U.SYNC_JOIN, token=tok)
                for r0 in (1, ny - 2):
                    U.upir_loop_exec(s, U.loop_desc([r0, 1], [r0 + 1, nx - 1], tile=[16, 256],
                                                    distribute=U.DIST_TEAMS, inner_chunk=4), body)
            else:
                U.upir_sync(ctx, U.SYNC_HALO, halo_map=src)
                U.upir_loop_exec(s, U.loop_desc([1, 1], [ny - 1, nx - 1], tile=[16, 256], distribute=U.DIST_TEAMS,
                                                inner_chunk=4), body)
            src, dst = dst, src
        U.upir_spmd_end(s)
        U.upir_data_unmap(ctx, mb)
        U.upir_data_unmap(ctx, ma)
        U.upir_sync(ctx)
        return a if S % 2 == 0 else b

    plain, split = run(False), run(True)
    assert (plain == split).all()
    assert np.abs(plain - oracle.jacobi5(g, S)).max() <= 1e-5
    with pytest.raises(U.UpirError) as ei:
        U.upir_sync(ctx, U.SYNC_JOIN)
    assert ei.value.status == U.E_SYNC


def test_async_halo_join_graph_capture(ctx):
    """The split sweep (async HALO on the copy stream, interior rows, JOIN,
    boundary rows) captured as one CUDA graph -- the form bench.py times for
    C5b -- replays to the same bits as eager synchronous sweeps."""
    ny, nx, S = 66, 520, 8
    g = synth.jacobi_init(ny, nx)
    d = U.dist(ny, nx, 4, halo_rows=1)
    res = []
    for graph in (False, True):
        a, b = g.copy(), g.copy()
        ma = U.upir_data_map(ctx, a, U.MAP_TOFROM, d)
        mb = U.upir_data_map(ctx, b, U.MAP_TOFROM, d)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(7, 256, U.TARGET_CLUSTER))
        bodies = [(ma, U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(nx, 0, 0), dims=(ny, 0, 0))),
                  (mb, U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(nx, 0, 0), dims=(ny, 0, 0)))]
        full = U.loop_desc([1, 1], [ny - 1, nx - 1], tile=[16, 256], distribute=U.DIST_TEAMS, inner_chunk=4)
        inner = U.loop_desc([2, 1], [ny - 2, nx - 1], tile=[16, 256], distribute=U.DIST_TEAMS, inner_chunk=4)
        edges = [U.loop_desc([r, 1], [r + 1, nx - 1], tile=[16, 256], distribute=U.DIST_TEAMS, inner_chunk=4)
                 for r in (1, ny - 2)]
        if graph:
            U.upir_graph_begin(ctx)
            for k in range(S):
                src, body = bodies[k % 2]
                tok = U.upir_sync(ctx, U.SYNC_HALO, halo_map=src, async_=True)
                U.upir_loop_exec(s, inner, body)
                U.upir_sync(ctx, U.SYNC_JOIN, token=tok)
                for e in edges:
                    U.upir_loop_exec(s, e, body)
            gr = U.upir_graph_end(ctx)
            U.upir_graph_launch(ctx, gr)
            U.upir_sync(ctx)
            U.upir_graph_destroy(gr)
        else:
            for k in range(S):
                src, body = bodies[k % 2]
                U.upir_sync(ctx, U.SYNC_HALO, halo_map=src)
                U.upir_loop_exec(s, full, body)
        U.upir_spmd_end(s)
        U.upir_data_unmap(ctx, mb)
        U.upir_data_unmap(ctx, ma)
        U.upir_sync(ctx)
        res.append(a if S % 2 == 0 else b)
    assert (res[0] == res[1]).all()
    assert np.abs(res[0] - oracle.jacobi5(g, S)).max() <= 1e-5


@pytest.mark.parametrize("dt", ["i64", "f32"])
def test_world_combine_path_world1_matches_plain(ctx, dt):
    """The communicator world-reduction path (last team writes the int64 /
    fp64 partial, gather, one combine kernel applies init and rounds once) run
    at world size 1 via UPIR_WORLD_VIA_COMM: bit-identical to the plain loop
    for sum / max / min with an original value (reading c9, c10)."""
    n = 300_007
    if dt == "i64":
        x, dtype, tdt, inits = synth.i64_sym(6, 0, n), U.I64, torch.int64, [7, -3]
    else:
        x, dtype, tdt, inits = synth.f32_unit(7, 0, n), U.F32, torch.float32, [0.5, 0.25]
    m = U.upir_data_map(ctx, x, U.MAP_TO)
    outs = {}
    for flags in (0, U.WORLD_REDUCE | U.WORLD_VIA_COMM):
        for ops in ((U.OP_SUM, U.OP_MAX), (U.OP_MIN, U.OP_SUM)):
            r = torch.zeros(2, dtype=tdt, device="cuda")
            torch.cuda.synchronize()
            s = U.upir_spmd_launch(ctx, U.spmd_desc(37, 128))
            U.upir_loop_exec(s, U.loop_desc(0, n, chunk=4, flags=flags), U.body(U.BODY_REDUCE, dtype, in0=m),
                             [U.reduction(ops[0], dtype, r.data_ptr(), init=inits[0]),
                              U.reduction(ops[1], dtype, r.data_ptr() + r.element_size(), init=inits[1])])
            U.upir_spmd_end(s)
            U.upir_sync(ctx)
            outs[(flags, ops)] = r.cpu().numpy().tobytes()
    for ops in ((U.OP_SUM, U.OP_MAX), (U.OP_MIN, U.OP_SUM)):
        assert outs[(0, ops)] == outs[(U.WORLD_REDUCE | U.WORLD_VIA_COMM, ops)]
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)


@pytest.mark.parametrize("graph", [False, True])
def test_async_allreduce_join_and_wait(ctx, graph):
    """upir_reduce_async (NEXT #1 async allreduce): ordered after the compute
    work issued before it (it sees the fill), JOIN orders later compute work
    after it (the device reduction of its result sees it), WAIT releases on the
    host; world size 1 (the gather is a device copy); eager and captured."""
    n = 1000
    x = torch.zeros(n, dtype=torch.int64, device="cuda")
    out = torch.zeros(n, dtype=torch.int64, device="cuda")
    tot = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    mx = U.upir_data_adopt(ctx, x)

    def seq():
        U.upir_synth_fill(ctx, mx, 2, 6)
        tok = U.upir_reduce_async(ctx, U.OP_SUM, U.I64, x, n, out)
        U.upir_sync(ctx, U.SYNC_JOIN, token=tok)
        U.upir_reduce(ctx, U.OP_SUM, U.I64, out, n, tot, U.SCOPE_DEVICE)

    if graph:
        U.upir_graph_begin(ctx)
        seq()
        g = U.upir_graph_end(ctx)
        U.upir_graph_launch(ctx, g)
        U.upir_sync(ctx)
        U.upir_graph_destroy(g)
    else:
        seq()
        U.upir_sync(ctx)
    ref = synth.i64_sym(6, 0, n)
    assert (out.cpu().numpy() == ref).all()
    assert tot.item() == oracle.reduce_i64(oracle.SUM, ref)
    # host-side release
    out.zero_()
    torch.cuda.synchronize()
    tok = U.upir_reduce_async(ctx, U.OP_MAX, U.I64, x, n, out)
    U.upir_sync(ctx, U.SYNC_WAIT, token=tok)
    assert (out.cpu().numpy() == ref).all()
    U.upir_data_unmap(ctx, mx)
    U.upir_sync(ctx)


def test_async_edges(ctx):
    """Edge cases of the NEXT #1 calls: an empty FORWARD_ASYNC section is a
    no-op, an out-of-range one is rejected; upir_reduce_async rejects bad
    arguments before enqueueing anything; a count of 1 works."""
    x = np.arange(1000, dtype=np.int64)
    m = U.upir_data_map(ctx, x, U.MAP_ALLOC)
    U.upir_data_update_section(ctx, m, 0, 0, U.UPDATE_FORWARD_ASYNC)
    with pytest.raises(U.UpirError):
        U.upir_data_update_section(ctx, m, 7992, 16, U.UPDATE_FORWARD_ASYNC)
    with pytest.raises(U.UpirError):
        U.upir_data_update_section(ctx, m, 0, 8, 3)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    a = torch.tensor([5], dtype=torch.int64, device="cuda")
    b = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    for bad in (dict(count=0), dict(dtype=U.BF16), dict(op=7)):
        kw = dict(op=U.OP_SUM, dtype=U.I64, count=1)
        kw.update(bad)
        with pytest.raises(U.UpirError):
            U.upir_reduce_async(ctx, kw["op"], kw["dtype"], a, kw["count"], b)
    tok = U.upir_reduce_async(ctx, U.OP_SUM, U.I64, a, 1, b)
    U.upir_sync(ctx, U.SYNC_WAIT, token=tok)
    assert b.item() == 5

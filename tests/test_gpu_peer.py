"""Peer-window paths (NVLink peer memory between ranks) at world sizes 2 and
3, with the ranks as separate processes sharing the one GPU of this
environment (see tests/peer_worker.py):

* UPIR_WORLD_REDUCE -- upir.sync allreduce fused into the loop kernel:
  every rank gets init (+) the global reduction; int64 and fp32 max
  bit-exact against the oracle, fp32 sum within 1e-5 * sum|x| (north_star);
  repeated and graph-replayed reductions (generation / parity logic).
* Fused halo -- peer-mode JACOBI5 sweeps store boundary rows into the
  neighbours' halo rows and wait in-kernel for the neighbours' previous
  sweep; the assembled grid after S sweeps matches the fp64 oracle within
  1e-5 * max|ref| and is bit-identical to the one-rank sweep of the same
  kernel (decomposition invariance, reading c16).
"""
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import paper_2209_10643_b200 as U
import peer_worker
import synth

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args):
    mp.spawn(fn, args=(world, _port()) + args, nprocs=world, join=True)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,use_graph", [(2, False), (3, False), (2, True)])
def test_fused_world_reduce(upir, tmp_path, world, use_graph):
    n, reps = 300_007, 3
    _spawn(peer_worker.world_reduce_worker, world, str(tmp_path), n, reps, use_graph)
    xi = synth.i64_sym(6, 0, n)
    xf = synth.f32_unit(7, 0, n)
    want_si = oracle.world_reduce(oracle.SUM, [7, oracle.reduce_i64(oracle.SUM, xi)])
    want_mi = int(xi.max())
    want_sf = 0.5 + oracle.reduce_f32(oracle.SUM, xf)
    want_mf = float(xf.max())
    for r in range(world):
        raw = np.load(tmp_path / f"wri_{r}.npy")
        got = np.load(tmp_path / f"wr_{r}.npy")
        for k in range(reps):
            assert int(raw[k, 0]) == want_si, (r, k)
            assert int(raw[k, 1]) == want_mi, (r, k)
            assert abs(got[k, 2] - want_sf) <= 1e-5 * want_sf, (r, k)
            assert got[k, 3] == want_mf, (r, k)
    # every rank holds the identical combination (ascending rank order)
    ref = np.load(tmp_path / "wr_0.npy")
    for r in range(1, world):
        assert (np.load(tmp_path / f"wr_{r}.npy") == ref).all()


def _jacobi_one_rank(g, S, tile):
    ny, nx = g.shape
    ctx = U.upir_init(0)
    a, b = g.copy(), g.copy()
    ma = U.upir_data_map(ctx, a, U.MAP_TOFROM)
    mb = U.upir_data_map(ctx, b, U.MAP_TOFROM)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(5, 128))
    loop = U.loop_desc([1, 1], [ny - 1, nx - 1], tile=list(tile), distribute=U.DIST_TEAMS, inner_chunk=4)
    for k in range(S):
        src, dst = (ma, mb) if k % 2 == 0 else (mb, ma)
        U.upir_loop_exec(s, loop, U.body(U.BODY_JACOBI5, U.F32, in0=src, out=dst, ld=(nx, 0, 0), dims=(ny, 0, 0)))
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, mb)
    U.upir_data_unmap(ctx, ma)
    U.upir_sync(ctx)
    U.upir_finalize(ctx)
    return a if S % 2 == 0 else b


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,ny,nx,S,tile,use_graph,adopt", [
    (2, 70, 132, 6, (8, 64), False, False),
    (3, 61, 200, 5, (8, 64), False, False),
    (2, 67, 264, 8, (16, 256), True, False),
    (2, 70, 132, 4, (8, 64), False, True),
])
def test_fused_halo_jacobi(upir, tmp_path, world, ny, nx, S, tile, use_graph, adopt):
    _jacobi_multirank_check(tmp_path, world, ny, nx, S, tile, use_graph, adopt, "fused")


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,ny,nx,S,tile,use_graph,mode", [
    (2, 70, 132, 6, (8, 64), False, "explicit"),
    (3, 61, 200, 5, (8, 64), False, "explicit"),
    (2, 67, 264, 8, (16, 256), True, "explicit"),
    (2, 70, 132, 6, (8, 64), False, "async"),
    (3, 61, 200, 5, (8, 64), False, "async"),
    (3, 67, 264, 8, (16, 256), True, "async"),
    (3, 61, 200, 7, (8, 64), False, "mixed"),
    (2, 67, 264, 12, (16, 256), True, "mixed"),
])
def test_peer_halo_exchange_jacobi(upir, tmp_path, world, ny, nx, S, tile, use_graph, mode):
    """upir_sync(HALO) over the peer mappings (Fig. 7 send/recv, PAPER.md:889;
    SURVEY 8(e) 1-row halos) with a NON-empty exchange at world sizes 2 / 3:
    UPIR_HALO_EXPLICIT sweeps with the exchange before each sweep, and the
    async two-step form (arrive-compute on the copy stream
    overlapping the interior rows, JOIN, then the boundary rows).  The
    assembled grid equals one rank's bit for bit."""
    _jacobi_multirank_check(tmp_path, world, ny, nx, S, tile, use_graph, False, mode)


def _jacobi_multirank_check(tmp_path, world, ny, nx, S, tile, use_graph, adopt, mode):
    _spawn(peer_worker.jacobi_worker, world, str(tmp_path), ny, nx, S, tile, use_graph, adopt, mode)
    g = synth.jacobi_init(ny, nx)
    got = np.concatenate([np.load(tmp_path / f"jac_{r}.npy") for r in range(world)])
    assert got.shape == (ny, nx)
    ref = oracle.jacobi5(g, S)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()
    one = _jacobi_one_rank(g, S, tile)
    assert (got == one).all()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,n,sched,chunk", [(3, 1_000_003, U.SCHED_STATIC, 0), (3, 1_000_003, U.SCHED_STATIC, 2),
                                                 (2, 777_777, U.SCHED_STATIC, 4), (3, 1_000_003, U.SCHED_DYNAMIC, 4)])
def test_block_slices_odd_offsets_world_reduce(upir, tmp_path, world, n, sched, chunk):
    """C5a pattern with rank offsets that are not multiples of the vector
    width: the global result on every rank equals the oracle
    on the whole stream; int64 bit-exact, fp32 within 1e-5 (sum) / exact (max)."""
    _spawn(peer_worker.block_reduce_worker, world, str(tmp_path), n, sched, chunk)
    offs = [int(np.load(tmp_path / f"blkoff_{r}.npy")[0]) for r in range(world)]
    assert any(o % 4 for o in offs)   # at least one rank starts mid-vector
    xi = synth.i64_sym(6, 0, n)
    xf = synth.f32_unit(7, 0, n)
    for r in range(world):
        got = np.load(tmp_path / f"blk_{r}.npy")
        assert int(got[0]) == oracle.reduce_i64(oracle.SUM, xi)
        assert int(got[1]) == oracle.reduce_i64(oracle.MAX, xi)
        fs, fm = np.frombuffer(got[2:].tobytes(), np.float32)[[0, 2]]
        rs = oracle.reduce_f32(oracle.SUM, xf)
        assert abs(float(fs) - rs) <= 1e-5 * rs
        assert float(fm) == oracle.reduce_f32(oracle.MAX, xf)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,M,N,K,dt", [(2, 600, 512, 256, "bf16"), (3, 1000, 768, 128, "bf16"),
                                            (2, 768, 512, 320, "int"), (2, 500, 512, 96, "f32")])
def test_multirank_matmul_block_rows(upir, tmp_path, world, M, N, K, dt):
    """NEXT #4: rows of A / C BLOCK-sharded, B replicated; the
    assembled C matches the oracle (small integers: bit-exact, else
    componentwise-scaled 1e-5) and, for bf16, is bit-identical to one rank."""
    _spawn(peer_worker.matmul_rows_worker, world, str(tmp_path), M, N, K, dt)
    got = np.concatenate([np.load(tmp_path / f"mm_{r}.npy") for r in range(world)])
    assert got.shape == (M, N)
    if dt == "int":
        rng = np.random.default_rng(5)
        A = rng.integers(-2, 3, (M, K)).astype(np.float32)
        B = rng.integers(-2, 3, (K, N)).astype(np.float32)
        assert (got == oracle.matmul(A, B)).all()
        return
    gen = synth.bf16_sym_as_f32 if dt == "bf16" else synth.f32_sym
    A = gen(3, 0, M * K).reshape(M, K)
    B = gen(4, 0, K * N).reshape(K, N)
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
    assert (np.abs(got - oracle.matmul(A, B)) / scale).max() <= 1e-5
    _spawn(peer_worker.matmul_rows_worker, 1, str(tmp_path), M, N, K, dt)
    one = np.load(tmp_path / "mm_0.npy")
    if dt == "bf16":
        assert (got == one).all()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,n_rows,row_elems,dt,halo_rows,use_async", [
    (2, 20, 36, "i64", 1, False),    # 288-B rows: 16-B vector copies
    (3, 23, 37, "i32", 2, False),    # 148-B rows: byte copies, 2 halo rows
    (3, 17, 50, "u8", 3, True),      # async (copy stream) + JOIN, 3 halo rows
    (2, 9, 64, "i32", 2, True),
])
def test_peer_halo_exchange_rows(upir, tmp_path, world, n_rows, row_elems, dt, halo_rows, use_async):
    """upir_sync(HALO) over the peer mappings on its own (Fig. 7 send/recv,
    PAPER.md:889): after each of 3 exchanges every rank's halo rows hold its
    neighbours' owned rows of that round (plan of upir_halo_plan, checked here
    from the block rule), its own rows untouched, for several element sizes,
    halo depths and row sizes that do / do not allow 16-B copies."""
    reps = 3
    _spawn(peer_worker.halo_unit_worker, world, str(tmp_path), n_rows, row_elems, dt, halo_rows, use_async, reps)
    owner = {}
    for r in range(world):
        lo, hi = U.upir_dist_owned_rows(n_rows, r, world)
        for i in range(lo, hi):
            owner[i] = r

    def val(r, rep, i, j):
        return (r * 100000 + rep * 1000 + i * 7 + j) if dt != "u8" else (r * 37 + rep * 11 + i * 3 + j) % 251

    j = np.arange(row_elems)
    for r in range(world):
        got = np.load(tmp_path / f"halo_{r}.npy")
        lo, hi, r0, r1 = np.load(tmp_path / f"halo_rng_{r}.npy")
        for rep in range(reps):
            for i in range(r0, r1):
                want = val(owner[i], rep, i, j)   # own rows: mine; halo rows: the neighbour's
                assert (got[rep, i - r0] == want).all(), (r, rep, i)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,count,dt,use_async", [
    (2, 1, "i64", False), (3, 1000, "i64", True), (3, 50_000, "f32", False), (2, 65_536, "f32", True),
    (3, 777, "f32", True),
])
def test_peer_allreduce(upir, tmp_path, world, count, dt, use_async):
    """upir_reduce(WORLD) and its async two-step form (PAPER.md:889
    'allreduce', 880-882 arrive-compute / wait-release) over the peer
    windows at world sizes 2 / 3: element-wise, every rank gets the combine
    of all ranks in ascending rank order (oracle o8; int64 wrapping sum,
    fp32 combined in fp64 and rounded once -- reading c10), bit-exact, for
    sum / max / min over three rounds (both staging halves reused)."""
    reps, ops = 3, [U.OP_SUM, U.OP_MAX, U.OP_MIN]
    _spawn(peer_worker.allreduce_worker, world, str(tmp_path), count, dt, ops, use_async, reps)
    oop = {U.OP_SUM: oracle.SUM, U.OP_MAX: oracle.MAX, U.OP_MIN: oracle.MIN}
    k = 0
    got = [np.load(tmp_path / f"ar_{r}.npy") for r in range(world)]
    for rep in range(reps):
        for op in ops:
            vals = [(synth.i64_sym if dt == "i64" else synth.f32_sym)(100 + 10 * rep + r, 0, count)
                    for r in range(world)]
            if dt == "i64":
                want = np.array([oracle.world_reduce(oop[op], [int(v[i]) for v in vals]) for i in range(count)],
                                np.int64)
            else:
                want = np.array([oracle.world_reduce(oop[op], [float(v[i]) for v in vals]) for i in range(count)],
                                np.float64).astype(np.float32).view(np.int32).astype(np.int64)
            for r in range(world):
                assert (got[r][k] == want).all(), (r, rep, op)
            k += 1

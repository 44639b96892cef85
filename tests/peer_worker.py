"""Worker processes of the peer-window tests (test harness only).

Each worker is one rank of a communicator-less world (nccl_id NULL): the
ranks share ONE GPU here (the only one this environment has), so the CUDA-IPC
peer mappings, the .sys-scope signals and the in-kernel waits run exactly as
between GPUs, with the ranks' kernels time-sliced instead of concurrent.
Records move over a gloo process group; results go to .npy files.
"""
import os

import numpy as np


def _setup(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_10643_b200 as U
    ctx = U.upir_init(0, rank, world, None)
    return dist, U, ctx


def world_reduce_worker(rank, world, port, out_dir, n, reps, use_graph):
    dist, U, ctx = _setup(rank, world, port)
    import torch

    import synth
    xi = synth.i64_sym(6, 0, n)
    xf = synth.f32_unit(7, 0, n)
    U.upir_peer_share(ctx)
    mi = U.upir_data_map(ctx, xi, U.MAP_TO)
    mf = U.upir_data_map(ctx, xf, U.MAP_TO)
    res = torch.zeros(4 * reps, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    base = res.data_ptr()
    s = U.upir_spmd_launch(ctx, U.spmd_desc(37, 96, U.TARGET_CLUSTER))
    loop_i = U.loop_desc(0, n, policy=U.SCHED_STATIC, chunk=2, flags=U.WORLD_REDUCE)
    loop_f = U.loop_desc(0, n, policy=U.SCHED_DYNAMIC, chunk=64, flags=U.WORLD_REDUCE)
    init_i = np.array([7], np.int64)
    init_f = np.array([0.5], np.float32)

    def rep(k):
        o = base + 32 * k
        U.upir_loop_exec(s, loop_i, U.body(U.BODY_REDUCE, U.I64, in0=mi),
                         [U.reduction(U.OP_SUM, U.I64, o, init=init_i), U.reduction(U.OP_MAX, U.I64, o + 8)])
        U.upir_loop_exec(s, loop_f, U.body(U.BODY_REDUCE, U.F32, in0=mf),
                         [U.reduction(U.OP_SUM, U.F32, o + 16, init=init_f), U.reduction(U.OP_MAX, U.F32, o + 24)])

    if use_graph:
        U.upir_graph_begin(ctx)
        for k in range(reps):
            rep(k)
        g = U.upir_graph_end(ctx)
        U.upir_graph_launch(ctx, g)
        U.upir_sync(ctx)
        U.upir_graph_launch(ctx, g)   # replay: the generation counters advance on the device
        U.upir_sync(ctx)
        U.upir_graph_destroy(g)
    else:
        for k in range(reps):
            rep(k)
    U.upir_spmd_end(s)
    U.upir_sync(ctx, U.SYNC_WORLD_BARRIER)
    raw = res.cpu().numpy().view(np.int64).reshape(reps, 4)
    out = np.zeros((reps, 4), np.float64)
    for k in range(reps):
        out[k, 0] = float(raw[k, 0])
        out[k, 1] = float(raw[k, 1])
        out[k, 2] = float(np.frombuffer(raw[k, 2].tobytes()[:4], np.float32)[0])
        out[k, 3] = float(np.frombuffer(raw[k, 3].tobytes()[:4], np.float32)[0])
    np.save(os.path.join(out_dir, f"wr_{rank}.npy"), out)
    np.save(os.path.join(out_dir, f"wri_{rank}.npy"), raw[:, :2].copy())
    U.upir_data_unmap(ctx, mf)
    U.upir_data_unmap(ctx, mi)
    U.upir_sync(ctx)
    U.upir_finalize(ctx)
    dist.destroy_process_group()


def jacobi_worker(rank, world, port, out_dir, ny, nx, S, tile, use_graph, adopt, mode="fused"):
    """mode: 'fused' = peer-mode sweeps (halo stores inside the sweep);
    'explicit' = UPIR_HALO_EXPLICIT sweeps + upir_sync(HALO) over the peer
    mappings before each sweep; 'mixed' = every third sweep fused, the others
    explicit; 'async' = async HALO on the copy stream overlapping the interior
    rows, JOIN, then the boundary rows."""
    dist, U, ctx = _setup(rank, world, port)
    import torch

    import synth
    g = synth.jacobi_init(ny, nx)
    d = U.dist(ny, nx, 4, halo_rows=1)
    a, b = g.copy(), g.copy()
    keep = []
    if adopt:
        # torch-owned device grids (cudaMalloc-backed): local rows incl. halos
        lo, hi = U.upir_dist_owned_rows(ny, rank, world)
        r0, r1 = max(0, lo - 1), min(ny, hi + 1)
        ta = torch.from_numpy(g[r0:r1].copy()).cuda()
        tb = torch.from_numpy(g[r0:r1].copy()).cuda()
        torch.cuda.synchronize()
        keep = [ta, tb]
        ma = U.upir_data_adopt(ctx, ta, d, nbytes=g.nbytes)
        mb = U.upir_data_adopt(ctx, tb, d, nbytes=g.nbytes)
    else:
        ma = U.upir_data_map(ctx, a, U.MAP_TOFROM, d)
        mb = U.upir_data_map(ctx, b, U.MAP_TOFROM, d)
    U.upir_peer_share(ctx, [ma, mb])
    s = U.upir_spmd_launch(ctx, U.spmd_desc(5, 128, U.TARGET_CLUSTER))
    loop = U.loop_desc([1, 1], [ny - 1, nx - 1], tile=list(tile), distribute=U.DIST_TEAMS, inner_chunk=4)
    bodies = [U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(nx, 0, 0), dims=(ny, 0, 0)),
              U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(nx, 0, 0), dims=(ny, 0, 0))]

    lo, hi = U.upir_dist_owned_rows(ny, rank, world)
    r_lo, r_hi = max(lo, 1), min(hi, ny - 1)
    xl = U.loop_desc([1, 1], [ny - 1, nx - 1], tile=list(tile), distribute=U.DIST_TEAMS, inner_chunk=4,
                     flags=U.HALO_EXPLICIT)
    inner = U.loop_desc([r_lo + 1, 1], [r_hi - 1, nx - 1], tile=list(tile), distribute=U.DIST_TEAMS, inner_chunk=4,
                        flags=U.HALO_EXPLICIT)
    edges = [U.loop_desc([r, 1], [r + 1, nx - 1], tile=list(tile), distribute=U.DIST_TEAMS, inner_chunk=4,
                         flags=U.HALO_EXPLICIT) for r in sorted({r_lo, r_hi - 1}) if r_lo < r_hi]

    def sweeps(k0, count):
        for k in range(k0, k0 + count):
            if mode == "fused":
                U.upir_loop_exec(s, loop, bodies[k % 2])
                U.upir_sync(ctx, U.SYNC_HALO, halo_map=bodies[k % 2].out)   # fused: drains the deliveries
            elif mode == "explicit":
                U.upir_sync(ctx, U.SYNC_HALO, halo_map=bodies[k % 2].in0)   # peer-mapping exchange kernel
                U.upir_loop_exec(s, xl, bodies[k % 2])
            elif mode == "mixed":
                # fused and explicit sweeps interleaved on one generation
                # counter: HALO(in) is a no-op after a fused sweep
                U.upir_sync(ctx, U.SYNC_HALO, halo_map=bodies[k % 2].in0)
                U.upir_loop_exec(s, loop if k % 3 == 0 else xl, bodies[k % 2])
            else:
                tok = U.upir_sync(ctx, U.SYNC_HALO, halo_map=bodies[k % 2].in0, async_=True)
                if r_hi - r_lo > 2:
                    U.upir_loop_exec(s, inner, bodies[k % 2])
                U.upir_sync(ctx, U.SYNC_JOIN, token=tok)
                for e in edges:
                    U.upir_loop_exec(s, e, bodies[k % 2])

    if use_graph:
        assert S % 4 == 0
        U.upir_graph_begin(ctx)
        sweeps(0, S // 2)
        gr = U.upir_graph_end(ctx)
        U.upir_graph_launch(ctx, gr)
        U.upir_graph_launch(ctx, gr)
        U.upir_graph_destroy(gr)
    else:
        sweeps(0, S)
    U.upir_spmd_end(s)
    if adopt:
        U.upir_sync(ctx)
        fin = (keep[0] if S % 2 == 0 else keep[1]).cpu().numpy()
        r0 = max(0, lo - 1)
        own = fin[lo - r0:hi - r0].copy()
        U.upir_data_unmap(ctx, mb)
        U.upir_data_unmap(ctx, ma)
    else:
        U.upir_data_unmap(ctx, mb)
        U.upir_data_unmap(ctx, ma)
        U.upir_sync(ctx)
        own = (a if S % 2 == 0 else b)[lo:hi].copy()
    np.save(os.path.join(out_dir, f"jac_{rank}.npy"), own)
    U.upir_sync(ctx, U.SYNC_WORLD_BARRIER)
    U.upir_finalize(ctx)
    dist.destroy_process_group()


def block_reduce_worker(rank, world, port, out_dir, n, sched, chunk):
    """C5a pattern: each rank adopts ONLY its BLOCK slice (rank r's first
    element is global index lo_r, generally not a multiple of the 32-B vector:
    the vector paths must align by address), fills it on the device from the
    global stream, and runs a CLUSTER-target loop with the world reduction
    fused over the peer windows."""
    dist, U, ctx = _setup(rank, world, port)
    import torch
    lo, hi = U.upir_dist_owned_rows(n, rank, world)
    xi = torch.empty(hi - lo, dtype=torch.int64, device="cuda")
    xf = torch.empty(hi - lo, dtype=torch.float32, device="cuda")
    res = torch.zeros(4, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    mi = U.upir_data_adopt(ctx, xi, U.dist(n, 1, 8))
    mf = U.upir_data_adopt(ctx, xf, U.dist(n, 1, 4))
    U.upir_synth_fill(ctx, mi, 2, 6)
    U.upir_synth_fill(ctx, mf, 0, 7)
    U.upir_peer_share(ctx)
    b = res.data_ptr()
    s = U.upir_spmd_launch(ctx, U.spmd_desc(37, 128, U.TARGET_CLUSTER))
    U.upir_loop_exec(s, U.loop_desc(0, n, policy=sched, chunk=chunk, flags=U.WORLD_REDUCE),
                     U.body(U.BODY_REDUCE, U.I64, in0=mi),
                     [U.reduction(U.OP_SUM, U.I64, b), U.reduction(U.OP_MAX, U.I64, b + 8)])
    U.upir_loop_exec(s, U.loop_desc(0, n, policy=sched, chunk=chunk, flags=U.WORLD_REDUCE),
                     U.body(U.BODY_REDUCE, U.F32, in0=mf),
                     [U.reduction(U.OP_SUM, U.F32, b + 16), U.reduction(U.OP_MAX, U.F32, b + 24)])
    U.upir_spmd_end(s)
    U.upir_sync(ctx)
    np.save(os.path.join(out_dir, f"blk_{rank}.npy"), res.cpu().numpy())
    np.save(os.path.join(out_dir, f"blkoff_{rank}.npy"), np.array([lo, hi], np.int64))
    U.upir_sync(ctx, U.SYNC_WORLD_BARRIER)
    U.upir_data_unmap(ctx, mf)
    U.upir_data_unmap(ctx, mi)
    U.upir_sync(ctx)
    U.upir_finalize(ctx)
    dist.destroy_process_group()


def matmul_rows_worker(rank, world, port, out_dir, M, N, K, dtype_name):
    """NEXT #4 multi-GPU matmul: A and C BLOCK-distributed by rows, B
    replicated, CLUSTER-target collapse(2) loop; every rank computes its own
    rows (no collective)."""
    dist, U, ctx = _setup(rank, world, port)
    import synth
    if dtype_name == "bf16":
        A = synth.bf16_sym_as_f32(3, 0, M * K).reshape(M, K)
        B = synth.bf16_sym_as_f32(4, 0, K * N).reshape(K, N)
        a = (A.view(np.uint32) >> 16).astype(np.uint16)
        b = (B.view(np.uint32) >> 16).astype(np.uint16)
        dt, esz, units = U.BF16, 2, 256
    elif dtype_name == "int":
        rng = np.random.default_rng(5)
        A = rng.integers(-2, 3, (M, K)).astype(np.float32)
        B = rng.integers(-2, 3, (K, N)).astype(np.float32)
        a = (A.view(np.uint32) >> 16).astype(np.uint16)
        b = (B.view(np.uint32) >> 16).astype(np.uint16)
        dt, esz, units = U.BF16, 2, 512
    else:
        a = synth.f32_sym(3, 0, M * K).reshape(M, K)
        b = synth.f32_sym(4, 0, K * N).reshape(K, N)
        dt, esz, units = U.F32, 4, 384
    C = np.zeros((M, N), np.float32)
    ma = U.upir_data_map(ctx, a, U.MAP_TO, U.dist(M, K, esz))
    mb = U.upir_data_map(ctx, b, U.MAP_TO)
    mc = U.upir_data_map(ctx, C, U.MAP_FROM, U.dist(M, N, 4))
    s = U.upir_spmd_launch(ctx, U.spmd_desc(7, units, U.TARGET_CLUSTER))
    U.upir_loop_exec(s, U.loop_desc([0, 0], [M, N], chunk=1, distribute=U.DIST_TEAMS),
                     U.body(U.BODY_MATMUL, dt, in0=ma, in1=mb, out=mc, ld=(K, N, N), dims=(K, M, N)))
    U.upir_spmd_end(s)
    for m in (mc, mb, ma):
        U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    lo, hi = U.upir_dist_owned_rows(M, rank, world)
    np.save(os.path.join(out_dir, f"mm_{rank}.npy"), C[lo:hi].copy())
    dist.barrier()   # no collective on the data path: host barrier only
    U.upir_finalize(ctx)
    dist.destroy_process_group()


def halo_unit_worker(rank, world, port, out_dir, n_rows, row_elems, dtype_name, halo_rows, use_async, reps):
    """upir_sync(HALO) alone over the peer mappings: every rep each rank
    writes a rank / rep / row pattern into its owned rows (torch, then a
    device sync), exchanges, and records its halo rows."""
    dist, U, ctx = _setup(rank, world, port)
    import torch
    tdt = {"i32": torch.int32, "i64": torch.int64, "u8": torch.uint8}[dtype_name]
    esz = torch.tensor([], dtype=tdt).element_size()
    d = U.dist(n_rows, row_elems, esz, halo_rows=halo_rows)
    lo, hi = U.upir_dist_owned_rows(n_rows, rank, world)
    r0, r1 = max(0, lo - halo_rows), min(n_rows, hi + halo_rows)
    t = torch.full((r1 - r0, row_elems), -1 if dtype_name != "u8" else 255, dtype=tdt, device="cuda")
    torch.cuda.synchronize()
    m = U.upir_data_adopt(ctx, t, d, nbytes=n_rows * row_elems * esz)
    U.upir_peer_share(ctx, [m])
    rows = torch.arange(r0, r1, device="cuda", dtype=torch.int64)[:, None].expand(-1, row_elems)
    cols = torch.arange(row_elems, device="cuda", dtype=torch.int64)[None, :]
    got = []
    for rep in range(reps):
        val = (rank * 100000 + rep * 1000 + rows * 7 + cols) if dtype_name != "u8" else \
            (rank * 37 + rep * 11 + rows * 3 + cols) % 251
        t[lo - r0:hi - r0] = val[lo - r0:hi - r0].to(tdt)
        torch.cuda.synchronize()
        if use_async:
            tok = U.upir_sync(ctx, U.SYNC_HALO, halo_map=m, async_=True)
            U.upir_sync(ctx, U.SYNC_JOIN, token=tok)
        else:
            U.upir_sync(ctx, U.SYNC_HALO, halo_map=m)
        U.upir_sync(ctx)
        got.append(t.cpu().numpy().astype(np.int64))
        U.upir_sync(ctx, U.SYNC_WORLD_BARRIER)   # every rank read its halos before the next rep's writes
    np.save(os.path.join(out_dir, f"halo_{rank}.npy"), np.stack(got))
    np.save(os.path.join(out_dir, f"halo_rng_{rank}.npy"), np.array([lo, hi, r0, r1]))
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx, U.SYNC_WORLD_BARRIER)
    U.upir_finalize(ctx)
    dist.destroy_process_group()


def allreduce_worker(rank, world, port, out_dir, count, dtype_name, ops, use_async, reps):
    """upir_reduce(WORLD) / upir_reduce_async over the peer windows: each rep
    every rank reduces its own seeded vector element-wise with every other
    rank's (ascending rank order); interleaved with a device-scope loop to
    show the async form overlaps nothing it should not."""
    dist, U, ctx = _setup(rank, world, port)
    import torch

    import synth
    U.upir_peer_share(ctx, [])
    dt = U.I64 if dtype_name == "i64" else U.F32
    out = []
    for rep in range(reps):
        for op in ops:
            stream = 100 + 10 * rep + rank
            host = synth.i64_sym(stream, 0, count) if dt == U.I64 else synth.f32_sym(stream, 0, count)
            x = torch.from_numpy(host).cuda()
            y = torch.zeros_like(x)
            torch.cuda.synchronize()
            if use_async:
                tok = U.upir_reduce_async(ctx, op, dt, x, count, y)
                U.upir_sync(ctx, U.SYNC_JOIN, token=tok)
            else:
                U.upir_reduce(ctx, op, dt, x, count, y, U.SCOPE_WORLD)
            U.upir_sync(ctx)
            out.append(y.cpu().numpy().view(np.int64 if dt == U.I64 else np.int32).astype(np.int64))
    np.save(os.path.join(out_dir, f"ar_{rank}.npy"), np.stack(out))
    U.upir_sync(ctx, U.SYNC_WORLD_BARRIER)
    U.upir_finalize(ctx)
    dist.destroy_process_group()

"""World-size-2 checks of the multi-GPU host logic on CPU (gloo).

The product's decomposition rules -- the BLOCK split of the iteration space /
rows over ranks (upir_dist_owned_rows, reading c20) and the halo plan that
upir_sync(HALO) executes (upir_halo_plan) -- are exercised across two real
processes, with gloo standing in for NCCL as the byte mover:
  * reductions: per-rank partials over the product's block split, combined in
    ascending rank order (upir_reduce WORLD semantics, o8) == the global oracle;
  * Jacobi: row slabs with 1-row halos exchanged per the halo plan every sweep
    == the single-rank result bit for bit (same per-point arithmetic), and
    within 1e-5 of the fp64 oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sweep_f32(g):
    """One Jacobi sweep in fp32 with the kernel's association (reading c16)."""
    out = g.copy()
    n, s, w, e = g[:-2, 1:-1], g[2:, 1:-1], g[1:-1, :-2], g[1:-1, 2:]
    out[1:-1, 1:-1] = np.float32(0.25) * ((n + s) + (w + e))
    return out


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2209_10643_b200 as U
    import synth
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = {}
    # ---- reductions over the block split of the normalised space ----------
    n = 100_003
    x = synth.i64_sym(6, 0, n)
    xf = synth.f32_sym(7, 0, n)
    lo, hi = U.upir_dist_owned_rows(n, rank, world)
    p = 148 * 256
    mine = [oracle.reduce_i64(oracle.SUM, x[lo:hi], p=p), oracle.reduce_i64(oracle.MAX, x[lo:hi], p=p),
            oracle.reduce_f32(oracle.SUM, xf[lo:hi], p=p)]
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, mine))
    spans = [(g[0], g[1]) for g in gathered]
    res["spans"] = spans
    res["sum"] = oracle.world_reduce(oracle.SUM, [g[2][0] for g in gathered])
    res["max"] = oracle.world_reduce(oracle.MAX, [g[2][1] for g in gathered])
    res["fsum"] = oracle.world_reduce(oracle.SUM, [g[2][2] for g in gathered])
    # ---- Jacobi slabs with halo exchange per upir_halo_plan ---------------
    ny, nx, S = 53, 40, 7
    g = synth.jacobi_init(ny, nx)
    rlo, rhi = U.upir_dist_owned_rows(ny, rank, world)
    llo, lhi = max(0, rlo - 1), min(ny, rhi + 1)
    slab = g[llo:lhi].copy()
    plan = U.upir_halo_plan(ny, 1, rank, world)
    for _ in range(S):
        reqs = []
        for key, peer in (("send_up", rank - 1), ("send_dn", rank + 1)):
            a, b = plan[key]
            if b > a:
                reqs.append(dist.isend(torch.from_numpy(slab[a - llo:b - llo].copy()), peer))
        for key, peer in (("recv_up", rank - 1), ("recv_dn", rank + 1)):
            a, b = plan[key]
            if b > a:
                buf = torch.empty((b - a, nx), dtype=torch.float32)
                dist.recv(buf, peer)
                slab[a - llo:b - llo] = buf.numpy()
        for r in reqs:
            r.wait()
        new = _sweep_f32(slab)
        # only owned interior rows are iterations of this rank
        for i in range(rlo, rhi):
            if 1 <= i < ny - 1:
                slab[i - llo] = new[i - llo]
    owned = [None] * world
    dist.all_gather_object(owned, (rlo, rhi, slab[rlo - llo:rhi - llo]))
    res["jacobi"] = np.concatenate([o[2] for o in sorted(owned, key=lambda t: t[0])])
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(res)


@pytest.mark.parametrize("world", [2])
def test_two_rank_decomposition(world):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 100_003
    x = synth.i64_sym(6, 0, n)
    xf = synth.f32_sym(7, 0, n)
    # the block split partitions [0, n) in rank order
    spans = res["spans"]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
    assert res["sum"] == oracle.reduce_i64(oracle.SUM, x)
    assert res["max"] == oracle.reduce_i64(oracle.MAX, x)
    assert abs(res["fsum"] - oracle.reduce_f32(oracle.SUM, xf)) <= 1e-12 * np.abs(xf).sum()
    # Jacobi: decomposition invariance (bit-exact) and fp64 oracle tolerance
    ny, nx, S = 53, 40, 7
    g = synth.jacobi_init(ny, nx)
    single = g.copy()
    for _ in range(S):
        single = _sweep_f32(single)
    assert (res["jacobi"] == single).all()
    ref = oracle.jacobi5(g, S)
    assert np.abs(res["jacobi"] - ref).max() <= 1e-5 * np.abs(ref).max()


def test_halo_plan_shapes():
    import paper_2209_10643_b200 as U
    # 4 ranks over 10 rows, halo 1: block rule 3,3,2,2
    plans = [U.upir_halo_plan(10, 1, r, 4) for r in range(4)]
    assert plans[0]["send_up"] == (0, 0) and plans[0]["send_dn"] == (2, 3) and plans[0]["recv_dn"] == (3, 4)
    assert plans[1]["send_up"] == (3, 4) and plans[1]["recv_up"] == (2, 3)
    assert plans[3]["send_dn"] == (0, 0) and plans[3]["recv_up"] == (7, 8)
    # what rank r sends down is exactly what rank r+1 receives from above
    for r in range(3):
        assert plans[r]["send_dn"] == plans[r + 1]["recv_up"]
        assert plans[r + 1]["send_up"] == plans[r]["recv_dn"]

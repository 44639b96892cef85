"""GPU parity of the MATMUL loop body (tcgen05 tensor cores, bf16 inputs,
fp32 accumulation) against the fp64 oracle, through the C-ABI.

Tolerance (north_star 1e-5; reading c22): max_ij |dC_ij| / (|A| |B|)_ij <=
1e-5 (componentwise-scaled).  Small-integer inputs and the identity are
bit-exact under any accumulation order; the tile -> team map of static
schedules is bit-exact.
"""
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


def to_bf16_bits(x):
    x = np.ascontiguousarray(x, np.float32)
    assert ((x.view(np.uint32) & 0xFFFF) == 0).all(), "value not exact in bf16"
    return (x.view(np.uint32) >> 16).astype(np.uint16)


def matmul_gpu(ctx, A, B, teams=148, policy=U.SCHED_STATIC, chunk=1, space=None, trace=False, C0=None,
               dtype=U.BF16, units=None):
    M, K = A.shape
    _, N = B.shape
    if dtype == U.BF16:
        a, b = to_bf16_bits(A), to_bf16_bits(B)
    else:
        a, b = np.ascontiguousarray(A, np.float32), np.ascontiguousarray(B, np.float32)
    units = units or (256 if dtype == U.BF16 else 384)
    tm_rows = 256 if units in (512, 768) else 128
    C = np.zeros((M, N), np.float32) if C0 is None else C0.copy()
    ma = U.upir_data_map(ctx, a, U.MAP_TO)
    mb = U.upir_data_map(ctx, b, U.MAP_TO)
    mc = U.upir_data_map(ctx, C, U.MAP_TOFROM)
    lb0, ub0, lb1, ub1 = space or (0, M, 0, N)
    tr = tm = None
    if trace:
        nt = ((ub0 + tm_rows - 1) // tm_rows - lb0 // tm_rows) * ((ub1 + 255) // 256 - lb1 // 256)
        tr = np.zeros(3 * nt, np.int32)
        tm = U.upir_data_map(ctx, tr, U.MAP_TOFROM)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
    try:
        U.upir_loop_exec(s, U.loop_desc([lb0, lb1], [ub0, ub1], policy=policy, chunk=chunk, distribute=U.DIST_TEAMS),
                         U.body(U.BODY_MATMUL, dtype, in0=ma, in1=mb, out=mc, ld=(K, N, N), dims=(K, M, N)),
                         trace=tm)
    finally:
        U.upir_spmd_end(s)
        if tm is not None:
            U.upir_data_unmap(ctx, tm)
        for m in (mc, mb, ma):
            U.upir_data_unmap(ctx, m)
        U.upir_sync(ctx)
    return C, tr


def scaled_err(C, A, B, ref):
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
    scale[scale == 0] = 1.0
    return (np.abs(C.astype(np.float64) - ref) / scale).max()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 256), (384, 256, 1024), (200, 312, 72),
                                   (1, 8, 8), (130, 264, 136)])
def test_matmul_parity(ctx, M, N, K):
    A = synth.bf16_sym_as_f32(3, 0, M * K).reshape(M, K)
    B = synth.bf16_sym_as_f32(4, 0, K * N).reshape(K, N)
    C, _ = matmul_gpu(ctx, A, B)
    ref = oracle.matmul(A, B)
    assert scaled_err(C, A, B, ref) <= 1e-5


def test_matmul_small_integers_bit_exact(ctx):
    rng = np.random.default_rng(7)
    M, N, K = 256, 512, 512
    A = rng.integers(-2, 3, (M, K)).astype(np.float32)
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    C, _ = matmul_gpu(ctx, A, B)
    assert (C == oracle.matmul(A, B)).all()


def test_matmul_identity_spec(ctx):
    # SPEC.md:404 generalised: A = I -> C = B exactly
    n = 256
    A = np.eye(n, dtype=np.float32)
    B = synth.bf16_sym_as_f32(4, 0, n * 512).reshape(n, 512)
    C, _ = matmul_gpu(ctx, A, B)
    assert (C == B).all()


def test_matmul_rank1_closed_form(ctx):
    M, N, K = 128, 256, 192
    u = synth.bf16_sym_as_f32(1, 0, M)
    v = synth.bf16_sym_as_f32(2, 0, N)
    A = np.repeat(u[:, None], K, axis=1)
    B = np.repeat(v[None, :], K, axis=0)
    C, _ = matmul_gpu(ctx, A, B)
    # K * u_i * v_j: products of 2^-6-grid values times 192 are exact in fp32
    assert (C == (K * np.outer(u.astype(np.float64), v.astype(np.float64))).astype(np.float32)).all()


@pytest.mark.parametrize("teams", [1, 3, 148, 400])
@pytest.mark.parametrize("policy,chunk", [(U.SCHED_STATIC, 0), (U.SCHED_STATIC, 1), (U.SCHED_STATIC, 2)])
def test_matmul_schedules_and_trace(ctx, teams, policy, chunk):
    M, N, K = 512, 768, 128
    A = synth.bf16_sym_as_f32(3, 0, M * K).reshape(M, K)
    B = synth.bf16_sym_as_f32(4, 0, K * N).reshape(K, N)
    C, tr = matmul_gpu(ctx, A, B, teams=teams, policy=policy, chunk=chunk, trace=True)
    assert scaled_err(C, A, B, oracle.matmul(A, B)) <= 1e-5
    nt = len(tr) // 3
    opol = oracle.STATIC
    assert (tr[2 * nt:] == 1).all()
    assert (tr[:nt] == oracle.tile_owner(M, N, 128, 256, opol, chunk, teams)).all()


def test_matmul_subspace_only_writes_its_iterations(ctx):
    M, N, K = 300, 520, 64
    A = synth.bf16_sym_as_f32(3, 0, M * K).reshape(M, K)
    B = synth.bf16_sym_as_f32(4, 0, K * N).reshape(K, N)
    C0 = np.full((M, N), -7.0, np.float32)
    space = (37, 290, 100, 500)
    C, _ = matmul_gpu(ctx, A, B, space=space, C0=C0)
    ref = oracle.matmul(A, B)
    sub = np.s_[37:290, 100:500]
    assert scaled_err(C[sub], A[37:290], B[:, 100:500], ref[sub]) <= 1e-5
    mask = np.ones((M, N), bool)
    mask[sub] = False
    assert (C[mask] == -7.0).all()


def test_matmul_rejects_bad_geometry(ctx):
    A = np.zeros((128, 64), np.float32)
    B = np.zeros((64, 256), np.float32)
    ma = U.upir_data_map(ctx, to_bf16_bits(A), U.MAP_TO)
    try:
        s = U.upir_spmd_launch(ctx, U.spmd_desc(4, 128))
        with pytest.raises(U.UpirError):
            U.upir_loop_exec(s, U.loop_desc([0, 0], [128, 256], distribute=U.DIST_TEAMS),
                             U.body(U.BODY_MATMUL, U.BF16, in0=ma, in1=ma, out=ma, ld=(64, 256, 256),
                                    dims=(64, 128, 256)))
        U.upir_spmd_end(s)
    finally:
        U.upir_data_unmap(ctx, ma)


# ---- fp32 inputs: 3xTF32 on kind::tf32 ------------------------------------------
@pytest.mark.parametrize("M,N,K", [(128, 256, 32), (256, 512, 512), (200, 312, 72), (130, 264, 4096)])
def test_matmul_f32_parity(ctx, M, N, K):
    A = synth.f32_sym(3, 0, M * K).reshape(M, K)
    B = synth.f32_sym(4, 0, K * N).reshape(K, N)
    C, _ = matmul_gpu(ctx, A, B, dtype=U.F32)
    assert scaled_err(C, A, B, oracle.matmul(A, B)) <= 1e-5


def test_matmul_f32_small_integers_bit_exact(ctx):
    rng = np.random.default_rng(11)
    M, N, K = 256, 256, 256
    A = rng.integers(-2, 3, (M, K)).astype(np.float32)
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    C, _ = matmul_gpu(ctx, A, B, dtype=U.F32)
    assert (C == oracle.matmul(A, B)).all()


@pytest.mark.parametrize("teams,chunk", [(1, 1), (148, 0), (5, 2)])
def test_matmul_f32_schedules_and_trace(ctx, teams, chunk):
    M, N, K = 384, 512, 96
    A = synth.f32_sym(3, 0, M * K).reshape(M, K)
    B = synth.f32_sym(4, 0, K * N).reshape(K, N)
    C, tr = matmul_gpu(ctx, A, B, teams=teams, chunk=chunk, trace=True, dtype=U.F32)
    assert scaled_err(C, A, B, oracle.matmul(A, B)) <= 1e-5
    nt = len(tr) // 3
    assert (tr[2 * nt:] == 1).all()
    assert (tr[:nt] == oracle.tile_owner(M, N, 128, 256, oracle.STATIC, chunk, teams)).all()


def test_matmul_f32_needs_384_units(ctx):
    a = np.zeros((128, 32), np.float32)
    ma = U.upir_data_map(ctx, a, U.MAP_TO)
    try:
        s = U.upir_spmd_launch(ctx, U.spmd_desc(4, 256))
        with pytest.raises(U.UpirError):
            U.upir_loop_exec(s, U.loop_desc([0, 0], [128, 32], distribute=U.DIST_TEAMS),
                             U.body(U.BODY_MATMUL, U.F32, in0=ma, in1=ma, out=ma, ld=(32, 32, 32),
                                    dims=(32, 128, 32)))
        U.upir_spmd_end(s)
    finally:
        U.upir_data_unmap(ctx, ma)


@pytest.mark.slow
def test_matmul_full_size_sampled_rows(ctx):
    """C4 at full size: 8192^3 bf16 -> fp32, 148 persistent teams; sampled
    rows against the oracle."""
    import torch
    n = 8192
    A = torch.empty(n * n, dtype=torch.bfloat16, device="cuda")
    B = torch.empty(n * n, dtype=torch.bfloat16, device="cuda")
    C = torch.empty(n * n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma, mb, mc = U.upir_data_adopt(ctx, A), U.upir_data_adopt(ctx, B), U.upir_data_adopt(ctx, C)
    U.upir_synth_fill(ctx, ma, 3, 3)
    U.upir_synth_fill(ctx, mb, 3, 4)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(148, 256))
    U.upir_loop_exec(s, U.loop_desc([0, 0], [n, n], policy=U.SCHED_STATIC, chunk=1, distribute=U.DIST_TEAMS),
                     U.body(U.BODY_MATMUL, U.BF16, in0=ma, in1=mb, out=mc, ld=(n, n, n), dims=(n, n, n)))
    U.upir_spmd_end(s)
    U.upir_sync(ctx)
    rows = np.array([0, 1, 127, 128, 4095, 5000, 8191])
    Ah = synth.bf16_sym_as_f32(3, 0, n * n).reshape(n, n)
    Bh = synth.bf16_sym_as_f32(4, 0, n * n).reshape(n, n)
    ref = oracle.matmul_rows(Ah, Bh, rows)
    got = C.view(n, n)[torch.from_numpy(rows).cuda()].cpu().numpy()
    scale = np.abs(Ah[rows].astype(np.float64)) @ np.abs(Bh.astype(np.float64))
    assert (np.abs(got - ref) / scale).max() <= 1e-5
    for m in (mc, mb, ma):
        U.upir_data_unmap(ctx, m)


def test_matmul_cluster_block_rows_world1(ctx):
    """NEXT #4 multi-GPU matmul: A and C BLOCK-distributed by rows, B
    replicated, CLUSTER-target loop (world size 1 here: rank 0 holds all rows)."""
    M, N, K = 384, 512, 128
    A = synth.bf16_sym_as_f32(3, 0, M * K).reshape(M, K)
    B = synth.bf16_sym_as_f32(4, 0, K * N).reshape(K, N)
    a, b = to_bf16_bits(A), to_bf16_bits(B)
    C = np.zeros((M, N), np.float32)
    ma = U.upir_data_map(ctx, a, U.MAP_TO, U.dist(M, K, 2))
    mb = U.upir_data_map(ctx, b, U.MAP_TO)
    mc = U.upir_data_map(ctx, C, U.MAP_FROM, U.dist(M, N, 4))
    s = U.upir_spmd_launch(ctx, U.spmd_desc(8, 256, U.TARGET_CLUSTER))
    U.upir_loop_exec(s, U.loop_desc([0, 0], [M, N], chunk=1, distribute=U.DIST_TEAMS),
                     U.body(U.BODY_MATMUL, U.BF16, in0=ma, in1=mb, out=mc, ld=(K, N, N), dims=(K, M, N)))
    U.upir_spmd_end(s)
    for m in (mc, mb, ma):
        U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    assert scaled_err(C, A, B, oracle.matmul(A, B)) <= 1e-5



# ---- CTA pairs (cta_group::2): a team = 2 CTAs = 512 units, 256 x 256 tiles ----------
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (512, 768, 256), (300, 520, 136), (1024, 1024, 1024)])
def test_matmul_pair_parity(ctx, M, N, K):
    A = synth.bf16_sym_as_f32(3, 0, M * K).reshape(M, K)
    B = synth.bf16_sym_as_f32(4, 0, K * N).reshape(K, N)
    C, _ = matmul_gpu(ctx, A, B, teams=74, units=512)
    assert scaled_err(C, A, B, oracle.matmul(A, B)) <= 1e-5


def test_matmul_pair_exact_and_trace(ctx):
    rng = np.random.default_rng(8)
    M, N, K = 768, 1024, 320
    A = rng.integers(-2, 3, (M, K)).astype(np.float32)
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    C, tr = matmul_gpu(ctx, A, B, teams=5, units=512, chunk=1, trace=True)
    assert (C == oracle.matmul(A, B)).all()
    nt = len(tr) // 3
    assert (tr[2 * nt:] == 1).all()
    assert (tr[:nt] == oracle.tile_owner(M, N, 256, 256, oracle.STATIC, 1, 5)).all()


def test_matmul_pair_subspace(ctx):
    M, N, K = 600, 704, 64
    A = synth.bf16_sym_as_f32(3, 0, M * K).reshape(M, K)
    B = synth.bf16_sym_as_f32(4, 0, K * N).reshape(K, N)
    C0 = np.full((M, N), -7.0, np.float32)
    C, _ = matmul_gpu(ctx, A, B, teams=3, units=512, space=(37, 590, 100, 600), C0=C0)
    ref = oracle.matmul(A, B)
    sub = np.s_[37:590, 100:600]
    assert scaled_err(C[sub], A[37:590], B[:, 100:600], ref[sub]) <= 1e-5
    mask = np.ones((M, N), bool)
    mask[sub] = False
    assert (C[mask] == -7.0).all()


@pytest.mark.parametrize("M,N,K", [(256, 256, 32), (512, 768, 256), (300, 520, 72)])
def test_matmul_pair_f32_parity(ctx, M, N, K):
    A = synth.f32_sym(3, 0, M * K).reshape(M, K)
    B = synth.f32_sym(4, 0, K * N).reshape(K, N)
    C, _ = matmul_gpu(ctx, A, B, teams=74, units=768, dtype=U.F32)
    assert scaled_err(C, A, B, oracle.matmul(A, B)) <= 1e-5


def test_matmul_pair_f32_exact_and_trace(ctx):
    rng = np.random.default_rng(12)
    M, N, K = 512, 512, 96
    A = rng.integers(-2, 3, (M, K)).astype(np.float32)
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    C, tr = matmul_gpu(ctx, A, B, teams=3, units=768, chunk=1, trace=True, dtype=U.F32)
    assert (C == oracle.matmul(A, B)).all()
    nt = len(tr) // 3
    assert (tr[2 * nt:] == 1).all()
    assert (tr[:nt] == oracle.tile_owner(M, N, 256, 256, oracle.STATIC, 1, 3)).all()

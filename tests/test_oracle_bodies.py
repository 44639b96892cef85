"""Pins of the oracle's loop bodies (o4 axpy, o5 reductions, o6 Jacobi,
o7 matmul, o8 world reduce): SPEC worked examples, closed forms, exact
integer references, invariants, numpy/BLAS as a library routine."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from conftest import GOLDEN

SPEC = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


# ---- o4 axpy ------------------------------------------------------------------
def test_axpy_spec_example():
    ex = SPEC["axpy"]
    got = oracle.axpy(ex["a"], np.array(ex["x"], np.float32), np.array(ex["y"], np.float32))
    assert got.tolist() == ex["expect_y"], ex["cite"]


def test_axpy_constants_closed_form():
    n = 1000
    got = oracle.axpy(3.0, np.ones(n, np.float32), np.full(n, 2.0, np.float32))
    assert (got == 5.0).all()
    y = synth.f32_unit(2, 0, n)
    assert (oracle.axpy(0.0, synth.f32_unit(1, 0, n), y) == y.astype(np.float64)).all()


def test_axpy_partial_range_and_step():
    # only iterations i = lb + k*step are written; others keep y (Fig. 9 guard i<n)
    x = np.arange(10, dtype=np.float32)
    y = np.full(10, 1.0, np.float32)
    got = oracle.axpy(2.0, x, y, lb=1, ub=9, step=3)   # i = 1, 4, 7
    exp = [1, 1 + 2 * 1, 1, 1, 1 + 2 * 4, 1, 1, 1 + 2 * 7, 1, 1]
    assert got.tolist() == exp


def test_axpy_exact_on_grid():
    # x, y on the 2^-24 grid, a = 2: a*x + y is exact in fp64; compare to an
    # integer computation of the same quantity
    n = 4096
    x = synth.f32_unit(1, 0, n)
    y = synth.f32_unit(2, 0, n)
    mx = (x.astype(np.float64) * 2 ** 24).astype(np.int64)
    my = (y.astype(np.float64) * 2 ** 24).astype(np.int64)
    exact = (2 * mx + my).astype(np.float64) * 2.0 ** -24
    assert (oracle.axpy(2.0, x, y) == exact).all()


# ---- o5 reductions -----------------------------------------------------------
def test_reduce_spec_sum_1_10_p3():
    ex = SPEC["reduction_sum_1_10"]
    v = np.array(ex["values"], np.int64)
    assert oracle.reduce_i64(oracle.SUM, v, p=ex["p"]) == ex["expect"]
    assert oracle.reduce_f32(oracle.SUM, v.astype(np.float32), p=ex["p"]) == ex["expect"]


def test_reduce_i64_closed_form_arith_series():
    n = 1 << 20
    x = np.arange(1, n + 1, dtype=np.int64)
    for pol, c, p in ((oracle.STATIC, 0, 7), (oracle.STATIC, 3, 148), (oracle.DYNAMIC, 5, 9)):
        assert oracle.reduce_i64(oracle.SUM, x, policy=pol, chunk=c, p=p) == n * (n + 1) // 2


def test_reduce_i64_init_and_partials():
    x = np.arange(1, 11, dtype=np.int64)
    r, parts = oracle.reduce_i64(oracle.SUM, x, init=100, p=3, want_partials=True)
    assert r == 155
    assert parts.tolist() == [1 + 2 + 3 + 4, 5 + 6 + 7, 8 + 9 + 10]   # static T=10,p=3 blocks
    r, parts = oracle.reduce_i64(oracle.MAX, x, init=-5, p=4, want_partials=True)
    assert r == 10 and parts.tolist() == [3, 6, 8, 10]


def test_reduce_i64_planted_extremum():
    n = 100_003
    rng = np.random.default_rng(1)
    x = rng.permutation(n).astype(np.int64) - 50_000
    assert oracle.reduce_i64(oracle.MAX, x, p=13) == n - 1 - 50_000
    assert oracle.reduce_i64(oracle.MIN, x, p=13) == -50_000


def test_reduce_i64_identities():
    e = np.zeros(0, np.int64)
    assert oracle.reduce_i64(oracle.SUM, e, p=4) == 0
    assert oracle.reduce_i64(oracle.MAX, e, p=4) == -(1 << 63)
    assert oracle.reduce_i64(oracle.MAX, e, init=7, p=4) == 7


def test_reduce_i64_wraps():
    # reading c12: two's-complement wrap
    x = np.array([(1 << 62), (1 << 62)], np.int64)
    assert oracle.reduce_i64(oracle.SUM, x, p=2) == -(1 << 63)


def test_reduce_f32_exact_grid_sum():
    # inputs m*2^-24: the exact sum is (sum m)*2^-24 computed in int64
    n = 1 << 20
    x = synth.f32_unit(7, 0, n)
    m = (x.astype(np.float64) * 2 ** 24).astype(np.int64)
    exact = float(m.sum()) * 2.0 ** -24     # sum m < 2^44: exact in fp64
    got = oracle.reduce_f32(oracle.SUM, x, p=148 * 4)
    assert abs(got - exact) <= 1e-12 * exact
    assert math.fsum(x.astype(np.float64)) == exact


def test_reduce_f32_closed_form_and_max():
    n = 10 ** 6
    x = np.arange(1, n + 1, dtype=np.float32)
    assert oracle.reduce_f32(oracle.SUM, x, p=64) == n * (n + 1) / 2
    y = synth.f32_unit(7, 0, n)
    y[123_457] = 2.0
    assert oracle.reduce_f32(oracle.MAX, y, p=37) == 2.0
    assert oracle.reduce_f32(oracle.MIN, np.array([3.0, -0.0, 0.0, 5.0], np.float32), p=2) == 0.0


def test_reduce_f32_geometry_invariance():
    x = synth.f32_sym(7, 0, 50_000)
    base = oracle.reduce_f32(oracle.SUM, x, p=1)
    for p in (2, 3, 64, 1000):
        assert abs(oracle.reduce_f32(oracle.SUM, x, p=p) - base) <= 1e-12 * np.abs(x).sum()


def test_world_reduce_equals_global():
    x = synth.i64_sym(6, 0, 10_000)
    parts = [oracle.reduce_i64(oracle.SUM, x[r * 2500:(r + 1) * 2500], p=5) for r in range(4)]
    assert oracle.world_reduce(oracle.SUM, parts) == int(x.sum())
    mparts = [oracle.reduce_i64(oracle.MAX, x[r * 2500:(r + 1) * 2500]) for r in range(4)]
    assert oracle.world_reduce(oracle.MAX, mparts) == int(x.max())


# ---- o6 Jacobi ----------------------------------------------------------------
def _fields(n):
    i = np.arange(n)[:, None].astype(np.float64)
    j = np.arange(n)[None, :].astype(np.float64)
    c = n // 2
    return {
        "constant": np.full((n, n), 0.75),
        "linear": 3 * i + 5 * j + 7,
        "bilinear": (i - c) * (j - c),
    }


@pytest.mark.parametrize("name", ["constant", "linear", "bilinear"])
def test_jacobi_harmonic_fixed_points(name):
    # discrete-harmonic fields are fixed points of the 5-point average
    g = _fields(33)[name].astype(np.float32)
    out = oracle.jacobi5(g, 7)
    assert (out == g.astype(np.float64)).all()


def test_jacobi_S0_identity_and_boundary_fixed():
    g = synth.jacobi_init(17, 23)
    assert (oracle.jacobi5(g, 0) == g).all()
    out = oracle.jacobi5(g, 5)
    for sl in (np.s_[0, :], np.s_[-1, :], np.s_[:, 0], np.s_[:, -1]):
        assert (out[sl] == g[sl]).all()


def test_jacobi_single_sweep_bruteforce():
    # one sweep written out point by point from the north_star formula
    g = synth.jacobi_init(6, 7).astype(np.float64)
    out = oracle.jacobi5(g.astype(np.float32), 1)
    for i in range(1, 5):
        for j in range(1, 6):
            assert out[i, j] == 0.25 * ((g[i - 1, j] + g[i + 1, j]) + (g[i, j - 1] + g[i, j + 1]))


def test_jacobi_eigenmode_decay():
    # sin(k pi i/(N-1)) sin(l pi j/(N-1)) with zero boundary decays by
    # lambda = (cos(k pi/(N-1)) + cos(l pi/(N-1)))/2 per sweep
    N, k, l, S = 65, 5, 3, 40
    i = np.arange(N)[:, None]
    j = np.arange(N)[None, :]
    g = np.sin(k * np.pi * i / (N - 1)) * np.sin(l * np.pi * j / (N - 1))
    g32 = g.astype(np.float32)
    lam = (np.cos(k * np.pi / (N - 1)) + np.cos(l * np.pi / (N - 1))) / 2
    out = oracle.jacobi5(g32, S)
    exact = g32.astype(np.float64) * lam ** S
    # the fp32 rounding of the initial field is not an exact eigenvector:
    # its residual component decays at most at rate 1 (bounded by 2^-24 scale)
    assert np.abs(out - exact).max() < 1e-6


def test_jacobi_max_principle_and_transpose_symmetry():
    g = synth.jacobi_init(40, 40)
    out = oracle.jacobi5(g, 30)
    assert out.min() >= g.min() and out.max() <= g.max()
    sym = (g + g.T) / 2
    sym = sym.astype(np.float32)
    o2 = oracle.jacobi5(sym, 9)
    assert (o2 == o2.T).all()


def test_jacobi_window_matches_full():
    ny, nx, S = 48, 52, 6
    g = synth.jacobi_init(ny, nx)
    full = oracle.jacobi5(g, S)
    for (r0, r1, c0, c1) in ((10, 20, 12, 30), (0, 8, 0, 9), (40, 48, 45, 52)):
        wr0, wr1 = max(0, r0 - S), min(ny, r1 + S)
        wc0, wc1 = max(0, c0 - S), min(nx, c1 + S)
        w = oracle.jacobi5_window(ny, nx, S, wr0, wc0, g[wr0:wr1, wc0:wc1])
        core = w[r0 - wr0:r1 - wr0, c0 - wc0:c1 - wc0]
        assert (core == full[r0:r1, c0:c1]).all()


# ---- o7 matmul ----------------------------------------------------------------
def test_matmul_spec_identity():
    ex = SPEC["matmul_identity"]
    C = oracle.matmul(np.array(ex["A"], np.float32), np.array(ex["B"], np.float32))
    assert C.tolist() == ex["expect_C"]


def test_matmul_numpy_float64():
    # library routine: numpy float64 matmul (BLAS dgemm) on the same values
    A = synth.f32_sym(3, 0, 37 * 53).reshape(37, 53)
    B = synth.f32_sym(4, 0, 53 * 29).reshape(53, 29)
    C = oracle.matmul(A, B)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.abs(C - ref).max() <= 1e-13


def test_matmul_small_integers_exact():
    rng = np.random.default_rng(5)
    A = rng.integers(-2, 3, (20, 64)).astype(np.float32)
    B = rng.integers(-2, 3, (64, 24)).astype(np.float32)
    ref = A.astype(np.int64) @ B.astype(np.int64)
    assert (oracle.matmul(A, B) == ref).all()


def test_matmul_rank1_closed_form_and_rows():
    K = 50
    u = synth.f32_sym(1, 0, 12)
    v = synth.f32_sym(2, 0, 9)
    A = np.repeat(u[:, None], K, axis=1)          # A = u 1^T
    B = np.repeat(v[None, :], K, axis=0)          # B = 1 v^T
    C = oracle.matmul(A, B)
    assert np.allclose(C, K * np.outer(u.astype(np.float64), v.astype(np.float64)), rtol=0, atol=1e-12)
    rows = np.array([11, 0, 5])
    assert (oracle.matmul_rows(A, B, rows) == C[rows]).all()


# ---- matvec (NEXT #2) ---------------------------------------------------------------
def test_matvec_numpy_and_identity():
    A = synth.f32_sym(3, 0, 41 * 67).reshape(41, 67)
    x = synth.f32_sym(1, 0, 67)
    assert np.abs(oracle.matvec(A, x) - A.astype(np.float64) @ x.astype(np.float64)).max() <= 1e-13
    eye = np.eye(16, dtype=np.float32)
    v = synth.f32_sym(2, 0, 16)
    assert (oracle.matvec(eye, v) == v).all()


def test_matvec_small_integers_rows_and_rank1():
    rng = np.random.default_rng(3)
    A = rng.integers(-3, 4, (30, 50)).astype(np.float32)
    x = rng.integers(-3, 4, 50).astype(np.float32)
    y0 = np.full(30, 9.0)
    y = oracle.matvec(A, x, lb=4, ub=20, y_in=y0)
    assert (y[4:20] == (A.astype(np.int64) @ x.astype(np.int64))[4:20]).all()
    assert (y[:4] == 9).all() and (y[20:] == 9).all()
    u = synth.f32_sym(1, 0, 12)
    B = np.repeat(u[:, None], 40, axis=1)            # rows u_i * 1^T
    assert np.allclose(oracle.matvec(B, np.ones(40, np.float32)), 40 * u.astype(np.float64), rtol=0, atol=1e-12)


# ---- 2-D filter stencil, radius 3 (NEXT #4) -----------------------------------------
def _w7():
    # symmetric dyadic weights summing to exactly 1
    v = np.array([1, 2, 3, 4, 3, 2, 1], np.float64)
    return (np.outer(v, v) / 256.0).astype(np.float32)


def test_stencil_library_routine_correlate2d():
    from scipy.signal import correlate2d
    g = synth.jacobi_init(30, 41)
    w = synth.f32_sym(9, 0, 49).reshape(7, 7)
    out = oracle.stencil2d(g, w)
    ref = correlate2d(g.astype(np.float64), w.astype(np.float64), mode="valid")
    assert np.abs(out[3:-3, 3:-3] - ref).max() <= 1e-12
    mask = np.ones_like(g, bool)
    mask[3:-3, 3:-3] = False
    assert (out[mask] == g[mask]).all()


def test_stencil_delta_and_shift_and_fixed_points():
    g = synth.jacobi_init(20, 25)
    d = np.zeros((7, 7), np.float32)
    d[3, 3] = 1
    assert (oracle.stencil2d(g, d, 3) == g).all()            # identity
    sh = np.zeros((7, 7), np.float32)
    sh[3, 5] = 1                                              # reads in[i][j+2]
    out = oracle.stencil2d(g, sh)
    assert (out[3:-3, 3:-3] == g[3:-3, 5:-1]).all()
    i = np.arange(40)[:, None].astype(np.float64)
    j = np.arange(40)[None, :].astype(np.float64)
    lin = (2 * i - 3 * j + 5).astype(np.float32)              # linear field, symmetric weights summing to 1
    assert (oracle.stencil2d(lin, _w7(), 4) == lin).all()


def test_reduce_stream_matches_array_oracle():
    # the oracle's in-place generator + reduction == generator module + array oracle
    for start, n in ((0, 5000), (123_456, 777)):
        xi = synth.i64_sym(6, start, n)
        xf = synth.f32_unit(7, start, n)
        assert oracle.reduce_stream(oracle.SUM, 2, 6, start, n) == oracle.reduce_i64(oracle.SUM, xi)
        assert oracle.reduce_stream(oracle.MAX, 2, 6, start, n) == int(xi.max())
        assert oracle.reduce_stream(oracle.SUM, 0, 7, start, n) == math.fsum(xf.astype(np.float64))
        assert oracle.reduce_stream(oracle.MAX, 0, 7, start, n) == float(xf.max())

"""CPU oracle of the UPIR data-parallel loop path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
(``paper_2209_10643_b200``) never imports it, and this package never imports
the product: they share no code.

Sequential, fp64 / exact int64.  Every function cites the passage it follows
(see upir_oracle.c).  Pins live in tests/test_oracle_*.py.

Parity status per function:
  trip_count, delinearize, schedule_chunks(static, static+chunk), owner_map,
  axpy, reduce_i64, reduce_f32, jacobi5, jacobi5_window, matmul_rows,
  tile_owner, tiled_owner (row-major c24 and column-major c35 tile ids),
  schedule_chunks(guided), matvec, stencil2d, simdlen groups (c33),
  MapSpace: pinned.
  schedule_chunks(dynamic): chunk partition pinned; the unit assignment is
  "parity unpinned (several results correct)" -- the GPU's assignment is
  checked for validity, not equality (reading c8).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "upir_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

STATIC, DYNAMIC, GUIDED, RUNTIME, AUTO = 0, 1, 2, 3, 4
SUM, MAX, MIN = 0, 1, 2


def build(force=False):
    """Compile the C oracle with gcc (plain -O2, no fast-math)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
           "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"]
    subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        sig = {
            "orc_trip_count": (i64, [i64, i64, i64]),
            "orc_delinearize": (None, [i32, vp, i64, vp]),
            "orc_schedule_chunks": (i64, [i32, i64, i64, i64, i64, vp, vp, i64]),
            "orc_owner_map": (i32, [i32, i64, i64, i64, vp]),
            "orc_schedule_chunks_simd": (i64, [i32, i64, i64, i64, i64, i64, vp, vp, i64]),
            "orc_owner_map_simd": (i32, [i32, i64, i64, i64, i64, vp]),
            "orc_axpy": (i32, [i64, i64, i64, i64, dbl, vp, vp, vp]),
            "orc_reduce_i64": (i32, [i32, i64, i64, i64, i64, i32, i64, i64, vp, i64, vp, vp]),
            "orc_reduce_f32": (i32, [i32, i64, i64, i64, i64, i32, i64, i64, vp, dbl, vp, vp]),
            "orc_jacobi5": (i32, [i64, i64, i64, vp, vp]),
            "orc_jacobi5_window": (i32, [i64, i64, i64, i64, i64, i64, i64, vp, vp]),
            "orc_matmul_rows": (i32, [i64, i64, i64, vp, vp, vp, i64, vp]),
            "orc_tile_owner": (i32, [i64, i64, i64, i64, i32, i64, i64, vp]),
            "orc_tiled_owner": (i64, [i64, i64, i64, i64, i64, i64, i32, i64, i64, i64, i64, vp, vp]),
            "orc_tiled_owner_order": (i64, [i64, i64, i64, i64, i64, i64, i32, i64, i64, i64, i64, i32, vp, vp]),
            "orc_matvec": (i32, [i64, i64, i64, i64, i64, vp, vp, vp, vp]),
            "orc_stencil2d": (i32, [i64, i64, i64, i64, vp, vp, vp]),
            "orc_reduce_stream": (i32, [i32, i32, ctypes.c_uint64, i64, i64, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


# ---- o1 ---------------------------------------------------------------------
def trip_count(lb, ub, step):
    return int(lib().orc_trip_count(lb, ub, step))


def delinearize(T, t):
    T = np.ascontiguousarray(T, dtype=np.int64)
    k = np.zeros(len(T), dtype=np.int64)
    lib().orc_delinearize(len(T), _p(T), t, _p(k))
    return tuple(int(v) for v in k)


# ---- o2/o3 ------------------------------------------------------------------
def schedule_chunks(policy, chunk, T, p, u, simdlen=1):
    """Chunks [lo, hi) of unit u (o2/o3); simdlen > 1: the schedule of the
    SIMD groups of simdlen iterations (reading c33)."""
    cap = 1
    while True:
        lo = np.zeros(cap, dtype=np.int64)
        hi = np.zeros(cap, dtype=np.int64)
        n = lib().orc_schedule_chunks_simd(policy, chunk, simdlen, T, p, u, _p(lo), _p(hi), cap)
        if n < 0:
            raise ValueError("invalid schedule")
        if n <= cap:
            return [(int(a), int(b)) for a, b in zip(lo[:n], hi[:n])]
        cap = n


def owner_map(policy, chunk, T, p, simdlen=1):
    owner = np.zeros(max(T, 1), dtype=np.int64)
    _check(lib().orc_owner_map_simd(policy, chunk, simdlen, T, p, _p(owner)), "owner_map")
    return owner[:T]


def tile_owner(R, C, tm, tn, policy, chunk, p):
    nt = ((R + tm - 1) // tm) * ((C + tn - 1) // tn)
    owner = np.zeros(max(nt, 1), dtype=np.int64)
    _check(lib().orc_tile_owner(R, C, tm, tn, policy, chunk, p, _p(owner)), "tile_owner")
    return owner[:nt]


def tiled_owner(lb0, ub0, lb1, ub1, BM, BN, policy, chunk, p_teams, ic, units, colmajor=False, reverse=False):
    """(team, unit) of every box position of a tiled collapse(2) nest (c24);
    colmajor: tile ids enumerate the tile grid column-major (c35); reverse:
    id k is the tile the un-reversed order numbers nt - 1 - k (c38)."""
    if ub0 <= lb0 or ub1 <= lb1:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    nt = (((ub0 + BM - 1) // BM) - lb0 // BM) * (((ub1 + BN - 1) // BN) - lb1 // BN)
    team = np.zeros(nt * BM * BN, dtype=np.int64)
    unit = np.zeros(nt * BM * BN, dtype=np.int64)
    r = lib().orc_tiled_owner_order(lb0, ub0, lb1, ub1, BM, BN, policy, chunk, p_teams, ic, units,
                                    (1 if colmajor else 0) | (2 if reverse else 0), _p(team), _p(unit))
    if r != nt:
        raise ValueError("tiled_owner failed")
    return team, unit


# ---- o4 ---------------------------------------------------------------------
def axpy(a, x, y, lb=0, ub=None, step=1):
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    n = len(y)
    ub = n if ub is None else ub
    out = np.zeros(n, dtype=np.float64)
    _check(lib().orc_axpy(n, lb, ub, step, float(a), _p(x), _p(y), _p(out)), "axpy")
    return out


# ---- o5 ---------------------------------------------------------------------
def reduce_i64(op, x, init=None, lb=0, ub=None, step=1, policy=STATIC, chunk=0, p=1,
               want_partials=False):
    x = np.ascontiguousarray(x, dtype=np.int64)
    n = len(x)
    ub = n if ub is None else ub
    if init is None:
        init = {SUM: 0, MAX: -(1 << 63), MIN: (1 << 63) - 1}[op]
    res = np.zeros(1, dtype=np.int64)
    parts = np.zeros(p, dtype=np.int64) if want_partials else None
    rc = lib().orc_reduce_i64(op, n, lb, ub, step, policy, chunk, p, _p(x), int(init),
                              _p(parts) if want_partials else None, _p(res))
    _check(rc, "reduce_i64")
    return (int(res[0]), parts) if want_partials else int(res[0])


def reduce_f32(op, x, init=None, lb=0, ub=None, step=1, policy=STATIC, chunk=0, p=1,
               want_partials=False):
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = len(x)
    ub = n if ub is None else ub
    if init is None:
        init = {SUM: 0.0, MAX: -np.inf, MIN: np.inf}[op]
    res = np.zeros(1, dtype=np.float64)
    parts = np.zeros(p, dtype=np.float64) if want_partials else None
    rc = lib().orc_reduce_f32(op, n, lb, ub, step, policy, chunk, p, _p(x), float(init),
                              _p(parts) if want_partials else None, _p(res))
    _check(rc, "reduce_f32")
    return (float(res[0]), parts) if want_partials else float(res[0])


def reduce_stream(op, dist, stream, start, n):
    """Sequential reduction of elements [start, start+n) of the synthetic
    stream, generated inside the oracle (its own copy of the recipe):
    dist 2 = int64 (exact), dist 0 = fp32 U[0,1) (fp64 accumulation)."""
    rf = np.zeros(1, np.float64)
    ri = np.zeros(1, np.int64)
    _check(lib().orc_reduce_stream(op, dist, stream, start, n, _p(rf), _p(ri)), "reduce_stream")
    return int(ri[0]) if dist == 2 else float(rf[0])


def world_reduce(op, rank_results):
    """o8: combine per-rank results in ascending rank order (PAPER.md:889
    'allreduce'; reading c10).  Integers wrap (c12); floats in fp64."""
    acc = None
    for r in rank_results:
        if acc is None:
            acc = r
        elif op == SUM:
            acc = acc + r
            if isinstance(acc, int):
                acc = ((acc + (1 << 63)) % (1 << 64)) - (1 << 63)
        elif op == MAX:
            acc = max(acc, r)
        else:
            acc = min(acc, r)
    return acc


# ---- o6 ---------------------------------------------------------------------
def jacobi5(grid, S):
    g = np.ascontiguousarray(grid, dtype=np.float32)
    ny, nx = g.shape
    out = np.zeros((ny, nx), dtype=np.float64)
    _check(lib().orc_jacobi5(ny, nx, S, _p(g), _p(out)), "jacobi5")
    return out


def jacobi5_window(ny, nx, S, wr0, wc0, win):
    w = np.ascontiguousarray(win, dtype=np.float32)
    wy, wx = w.shape
    out = np.zeros((wy, wx), dtype=np.float64)
    _check(lib().orc_jacobi5_window(ny, nx, S, wr0, wc0, wy, wx, _p(w), _p(out)),
           "jacobi5_window")
    return out


def stencil2d(grid, w, S=1):
    """2-D filter stencil of radius R = (len(w)-1)/2 (NEXT #4; reading c28)."""
    g = np.ascontiguousarray(grid, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    F = w.shape[0]
    assert w.shape == (F, F) and F % 2 == 1
    ny, nx = g.shape
    out = np.zeros((ny, nx), dtype=np.float64)
    _check(lib().orc_stencil2d(ny, nx, (F - 1) // 2, S, _p(w), _p(g), _p(out)), "stencil2d")
    return out


# ---- o7 ---------------------------------------------------------------------
def matmul_rows(A, B, rows):
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    C = np.zeros((len(rows), N), dtype=np.float64)
    _check(lib().orc_matmul_rows(M, N, K, _p(A), _p(B), _p(rows), len(rows), _p(C)),
           "matmul_rows")
    return C


def matvec(A, x, lb=0, ub=None, y_in=None):
    """y = A x over rows [lb, ub) in fp64 (NEXT #2 body)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    M, K = A.shape
    ub = M if ub is None else ub
    yi = np.zeros(M) if y_in is None else np.ascontiguousarray(y_in, dtype=np.float64)
    y = np.zeros(M, dtype=np.float64)
    _check(lib().orc_matvec(M, K, K, lb, ub, _p(A), _p(x), _p(yi), _p(y)), "matvec")
    return y


def matmul(A, B):
    return matmul_rows(A, B, np.arange(np.asarray(A).shape[0]))


# ---- o9: data map (Fig. 5 mapping, 843-854 Fig. 6) --------
from .mapspace import MapSpace  # noqa: E402,F401

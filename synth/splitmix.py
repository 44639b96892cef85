"""Counter-based splitmix64 input generator (numpy, host side).

Recipe: SURVEY.md §8(d) "Input generator"; restated in DESIGN.md.
Value maps (all exact in their target type):
  f32 U[0,1)      : (x >> 40) * 2^-24              (on the 2^-24 grid)
  f32 U[-1,1)     : 2 * f32_unit - 1
  i64 U[-2^28,2^28): int64(x >> 35) - 2^28
  bf16 U[-1,1)    : ((x >> 57) * 2^-7) * 2 - 1     (on the 2^-6 grid, exact in bf16)
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# stream ids (one per logical input array)
STREAMS = {"x": 1, "y": 2, "A": 3, "B": 4, "jacobi": 5, "i64": 6, "f32": 7}

# Test vectors of the recipe, used by tests to pin
# both this module and the CUDA fill kernel.
GOLDEN = {
    (1, "raw"): [0xE9D45DEC413FE5DB, 0xD5B8699E45F4FD81],
    (1, "f32"): [0.9133966565132141, 0.8348451256752014, 0.6024439930915833,
                 0.3780694603919983],
    (6, "i64"): [193051221, -102165435, 243335293, 138854209],
    (3, "bf16"): [0.90625, -0.4375, -0.09375, -0.78125],
}


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def raw(stream, start, n):
    """uint64 words for global element indices [start, start+n)."""
    seed = np.uint64(((2209 << 16) | int(stream)) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        i = np.arange(start, start + n, dtype=np.uint64)
        z = seed + (i + np.uint64(1)) * _GOLDEN
        return _mix(z)


def f32_unit(stream, start, n):
    return ((raw(stream, start, n) >> np.uint64(40)).astype(np.float64)
            * 2.0 ** -24).astype(np.float32)


def f32_sym(stream, start, n):
    u = (raw(stream, start, n) >> np.uint64(40)).astype(np.float64) * 2.0 ** -24
    return (2.0 * u - 1.0).astype(np.float32)


def i64_sym(stream, start, n):
    return (raw(stream, start, n) >> np.uint64(35)).astype(np.int64) - (1 << 28)


def bf16_sym_as_f32(stream, start, n):
    """bf16-representable values in U[-1,1), returned as float32."""
    m = (raw(stream, start, n) >> np.uint64(57)).astype(np.float64)
    return ((m * 2.0 ** -7) * 2.0 - 1.0).astype(np.float32)


def jacobi_init_rows(ny, nx, r0, r1, stream=STREAMS["jacobi"]):
    """Rows [r0, r1) of the Jacobi initial grid (fp32, row-major).

    Interior: U[0,1) of stream 5 at the global row-major index i*nx + j.
    Boundary (Dirichlet, fixed): top row (i = 0) = 1.0, every other boundary
    point = 0.0.
    """
    rows = r1 - r0
    g = f32_unit(stream, r0 * nx, rows * nx).reshape(rows, nx)
    ii = np.arange(r0, r1)[:, None]
    jj = np.arange(nx)[None, :]
    boundary = (ii == 0) | (ii == ny - 1) | (jj == 0) | (jj == nx - 1)
    g = np.where(boundary, np.float32(0.0), g)
    if r0 == 0:
        g[0, :] = 1.0
    return g.astype(np.float32)


def jacobi_init(ny, nx, stream=STREAMS["jacobi"]):
    return jacobi_init_rows(ny, nx, 0, ny, stream)


# ---- C twin for large inputs (same recipe; tests pin it against the above) ----
import ctypes as _ct
import os as _os
import subprocess as _sp

_CSRC = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "splitmix.c")
_CLIB = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "libsynth.so")
_clib = None


def build_c(force=False):
    if force or not _os.path.exists(_CLIB) or _os.path.getmtime(_CLIB) < _os.path.getmtime(_CSRC):
        _sp.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _CLIB, _CSRC])
    return _CLIB


def _c():
    global _clib
    if _clib is None:
        _clib = _ct.CDLL(build_c())
        for n in ("synth_raw", "synth_f32_unit", "synth_i64_sym"):
            getattr(_clib, n).argtypes = [_ct.c_uint64, _ct.c_int64, _ct.c_int64, _ct.c_void_p]
            getattr(_clib, n).restype = None
    return _clib


def c_f32_unit(stream, start, n):
    out = np.empty(n, dtype=np.float32)
    _c().synth_f32_unit(stream, start, n, out.ctypes.data)
    return out


def c_i64_sym(stream, start, n):
    out = np.empty(n, dtype=np.int64)
    _c().synth_i64_sym(stream, start, n, out.ctypes.data)
    return out


def c_raw(stream, start, n):
    out = np.empty(n, dtype=np.uint64)
    _c().synth_raw(stream, start, n, out.ctypes.data)
    return out

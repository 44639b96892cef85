"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NONE of the method's arithmetic (no schedule, no loop
body, no reduction).  It only produces input values, with a counter-based
generator so that any element can be produced independently:

    mix(z) : z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
             z = (z ^ (z >> 27)) * 0x94D049BB133111EB
             return z ^ (z >> 31)                     (splitmix64 finaliser)
    seed_s = (2209 << 16) | stream
    x_i    = mix(seed_s + (i + 1) * 0x9E3779B97F4A7C15)   (uint64 wrap-around)

The CUDA fill kernel (``upir_synth_fill`` in the C-ABI) is a second,
independent implementation of the same recipe; tests check the two agree
bit for bit.  See DESIGN.md "Input recipe".
"""
from .splitmix import (  # noqa: F401
    STREAMS, raw, f32_unit, f32_sym, i64_sym, bf16_sym_as_f32, jacobi_init,
    jacobi_init_rows, GOLDEN, c_f32_unit, c_i64_sym, c_raw, build_c,
)

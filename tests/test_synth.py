"""The shared input generator reproduces the recipe's test vectors
 and its value maps are exact."""
import numpy as np

import synth


def test_golden_vectors():
    assert [int(v) for v in synth.raw(1, 0, 2)] == synth.GOLDEN[(1, "raw")]
    assert synth.f32_unit(1, 0, 4).tolist() == synth.GOLDEN[(1, "f32")]
    assert synth.i64_sym(6, 0, 4).tolist() == synth.GOLDEN[(6, "i64")]
    assert synth.bf16_sym_as_f32(3, 0, 4).tolist() == synth.GOLDEN[(3, "bf16")]


def test_counter_based_offsets():
    a = synth.raw(5, 0, 100)
    b = synth.raw(5, 37, 20)
    assert (a[37:57] == b).all()


def test_ranges_and_grids():
    u = synth.f32_unit(7, 0, 1 << 16)
    assert u.min() >= 0 and u.max() < 1
    assert ((u.astype(np.float64) * 2 ** 24) % 1 == 0).all()
    i = synth.i64_sym(6, 0, 1 << 16)
    assert i.min() >= -(1 << 28) and i.max() < (1 << 28)
    b = synth.bf16_sym_as_f32(3, 0, 1 << 12)
    # exactly representable in bf16: low 16 bits of the fp32 pattern are zero
    assert ((b.view(np.uint32) & 0xFFFF) == 0).all()


def test_jacobi_init_boundary():
    g = synth.jacobi_init(9, 11)
    assert (g[0] == 1.0).all() and (g[-1] == 0).all()
    assert (g[1:, 0] == 0).all() and (g[1:, -1] == 0).all()
    rows = synth.jacobi_init_rows(9, 11, 3, 6)
    assert (rows == g[3:6]).all()

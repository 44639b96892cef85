"""Pins of o9 (upir.data map semantics) by invariants (SURVEY §8(c) 'Map')."""
import numpy as np
import pytest

from oracle.mapspace import MapSpace, TO, FROM, TOFROM, ALLOC, POISON


def test_to_from_round_trip_byte_identical():
    m = MapSpace()
    data = np.arange(100, dtype=np.float32)
    m.host_buffer("x", data)
    m.enter("x", TOFROM)
    assert (m.device("x") == m.host["x"]).all()
    m.exit("x")
    assert m.host["x"].tobytes() == data.tobytes()
    assert m.h2d == 400 and m.d2h == 400 and m.live() == 0


def test_alloc_no_copy_poison_visible():
    m = MapSpace()
    m.host_buffer("t", np.zeros(16, np.uint8))
    m.enter("t", ALLOC)
    assert m.h2d == 0 and (m.device("t") == POISON).all()
    m.exit("t")
    assert m.d2h == 0 and (m.host["t"] == 0).all()


def test_from_copies_back_only():
    m = MapSpace()
    m.host_buffer("y", np.zeros(8, np.uint8))
    m.enter("y", FROM)
    assert m.h2d == 0
    m.device("y")[:] = 7
    m.exit("y")
    assert (m.host["y"] == 7).all() and m.d2h == 8


def test_nested_map_copies_once():
    m = MapSpace()
    m.host_buffer("x", np.ones(10, np.float64))
    m.enter("x", TO)
    m.enter("x", TO)
    assert m.h2d == 80
    m.exit("x")
    assert m.live() == 1
    m.exit("x")
    assert m.live() == 0 and m.d2h == 0


def test_update_directions():
    m = MapSpace()
    m.host_buffer("x", np.zeros(4, np.uint8))
    m.enter("x", TO)
    m.host["x"][:] = 3
    m.update("x", backward=False)            # forward = host -> device (c19)
    assert (m.device("x") == 3).all()
    m.device("x")[:] = 9
    m.update("x", backward=True)
    assert (m.host["x"] == 9).all()
    with pytest.raises(KeyError):
        m.exit("nope")

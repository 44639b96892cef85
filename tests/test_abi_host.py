"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/upir.h declares, and its host-only logic (normalisation, validation,
schedule mirror, block distribution) agrees with the oracle.  No compute call
is made here (no GPU)."""
import ctypes
import os
import re

import pytest

import oracle
import paper_2209_10643_b200 as U
from conftest import ROOT


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "upir.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(upir_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = U.lib()
    names = _declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(U._abi.DECLARED)


def test_header_flag_macros_match_the_binding():
    """Every `#define UPIR_<NAME> <n>u` flag of include/upir.h has the same
    value under the binding's name (argument marshalling must not drift)."""
    src = open(os.path.join(ROOT, "include", "upir.h")).read()
    defs = dict(re.findall(r"#define UPIR_([A-Z_0-9]+) (\d+)u?\b", src))
    flags = {k: v for k, v in defs.items() if k not in ("H",) and not k.endswith("_H")}
    assert {"NOWAIT", "WORLD_REDUCE", "TILE_COLMAJOR", "WORLD_VIA_COMM", "TILE_REVERSE", "HALO_EXPLICIT"} <= set(flags)
    for k, v in flags.items():
        if hasattr(U, k):
            assert getattr(U, k) == int(v), k
    vals = [int(flags[k]) for k in ("NOWAIT", "WORLD_REDUCE", "TILE_COLMAJOR", "WORLD_VIA_COMM", "TILE_REVERSE",
                                    "HALO_EXPLICIT")]
    assert len(set(vals)) == len(vals) and all(v & (v - 1) == 0 for v in vals)   # distinct single bits


def test_header_enum_values_match_the_binding():
    """Every enumerator `UPIR_<NAME> = <n>` of include/upir.h's enums has the
    same value under the binding's name (the binding drops the UPIR_ prefix;
    statuses are E_*, bodies BODY_*, and so on), and none is missing."""
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "upir.h")).read(), flags=re.S)
    enums = re.findall(r"typedef enum\s*\{(.*?)\}", src, flags=re.S)
    vals = {}
    for body in enums:
        for name, v in re.findall(r"UPIR_([A-Z_0-9]+)\s*=\s*(\d+)", body):
            vals[name] = int(v)
    assert len(vals) >= 40
    for name, v in vals.items():
        assert hasattr(U, name), name
        assert getattr(U, name) == v, name


def test_version():
    assert "sm_100a" in U.upir_version()


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(U.UpirError) as ei:
        U.upir_init(0)
    assert ei.value.status in (U.E_CUDA, U.E_UNSUPPORTED)
    assert "no CPU fallback" in str(ei.value) or "CUDA" in str(ei.value)


@pytest.mark.parametrize("lb,ub,step", [(0, 10, 1), (0, 10, 3), (10, 0, -1), (10, 0, -3), (5, 5, 1),
                                        (-7, 20, 4), (0, 1 << 34, 1)])
def test_normalize_matches_oracle(lb, ub, step):
    T, Td = U.upir_loop_normalize(U.loop_desc(lb, ub, step))
    assert T == oracle.trip_count(lb, ub, step) == Td[0]


def test_normalize_collapse2():
    T, Td = U.upir_loop_normalize(U.loop_desc([1, 1], [8191, 8191]))
    assert T == 8190 * 8190 and Td[:2] == (8190, 8190)
    with pytest.raises(U.UpirError):
        U.upir_loop_normalize(U.loop_desc(0, 10, 0))


def test_schedule_mirror_matches_oracle():
    for T in (0, 1, 7, 10, 64, 1000):
        for p in (1, 2, 3, 7, 64):
            for c in (0, 1, 2, 5):
                for u in range(p):
                    assert U.upir_schedule_chunks(U.SCHED_STATIC, c, T, p, u) == \
                        oracle.schedule_chunks(oracle.STATIC, c, T, p, u)


def test_dist_owned_rows_matches_block_rule():
    # reading c20: the static block rule of o2 applied over ranks
    for n in (0, 1, 7, 32768, 32766):
        for R in (1, 2, 3, 4, 8):
            for r in range(R):
                lo, hi = U.upir_dist_owned_rows(n, r, R)
                exp = oracle.schedule_chunks(oracle.STATIC, 0, n, R, r)
                assert [(lo, hi)] == exp or (lo == hi and exp == [])


def _st(spmd, loop, kind, reds=None):
    return U.upir_loop_validate(spmd, loop, kind, reds)


def test_validation_error_paths():
    ok_spmd = U.spmd_desc(148, 256)
    loop = U.loop_desc(0, 1000)
    red = U.reduction(U.OP_SUM, U.F32, 0)
    assert _st(ok_spmd, loop, U.BODY_REDUCE, [red]) == U.OK
    # geometry honoured or rejected, never clamped
    assert _st(U.spmd_desc(1, 1025), loop, U.BODY_REDUCE, [red]) == U.E_INVALID
    assert _st(U.spmd_desc(0, 256), loop, U.BODY_REDUCE, [red]) == U.E_INVALID
    assert _st(U.spmd_desc(1, 0), loop, U.BODY_REDUCE, [red]) == U.E_INVALID
    assert _st(U.spmd_desc(1, 1024), loop, U.BODY_REDUCE, [red]) == U.OK
    # guided is built for 1-D loops
    assert _st(ok_spmd, U.loop_desc(0, 10, policy=U.SCHED_GUIDED), U.BODY_REDUCE, [red]) == U.OK
    assert _st(ok_spmd, U.loop_desc(0, 10, policy=9), U.BODY_REDUCE, [red]) == U.E_INVALID
    # distribute(units) with several teams would replicate (reading c7)
    assert _st(ok_spmd, U.loop_desc(0, 10, distribute=U.DIST_UNITS), U.BODY_REDUCE, [red]) == U.E_INVALID
    assert _st(U.spmd_desc(1, 64), U.loop_desc(0, 10, distribute=U.DIST_UNITS), U.BODY_REDUCE, [red]) == U.OK
    # REDUCE needs a reduction; at most two
    assert _st(ok_spmd, loop, U.BODY_REDUCE, []) == U.E_INVALID
    assert _st(ok_spmd, loop, U.BODY_REDUCE, [red, red, red]) == U.E_INVALID
    # step 0, negative chunk, bad collapse
    assert _st(ok_spmd, U.loop_desc(0, 10, 0), U.BODY_REDUCE, [red]) == U.E_INVALID
    assert _st(ok_spmd, U.loop_desc(0, 10, chunk=-1), U.BODY_REDUCE, [red]) == U.E_INVALID
    assert _st(ok_spmd, U.loop_desc([0, 0], [4, 4]), U.BODY_REDUCE, [red]) == U.E_INVALID
    # Jacobi needs a tiled collapse(2) nest over teams
    j = U.loop_desc([1, 1], [63, 63], tile=[32, 256], distribute=U.DIST_TEAMS, inner_chunk=4)
    assert _st(ok_spmd, j, U.BODY_JACOBI5) == U.OK
    assert _st(ok_spmd, U.loop_desc([1, 1], [63, 63]), U.BODY_JACOBI5) == U.E_INVALID


def test_failed_validation_sets_message():
    assert _st(U.spmd_desc(1, 2000), U.loop_desc(0, 1), U.BODY_REDUCE, [U.reduction(0, U.I64, 0)]) == U.E_INVALID
    assert "num_units" in U.upir_last_error()


def test_simdlen_validation_host():
    """simdlen (reading c33) is validated without a device."""
    reds = [U.reduction(U.OP_SUM, U.I64, 0)]
    ok = U.loop_desc(0, 100, simdlen=8)
    assert U.upir_loop_validate(U.spmd_desc(1, 32), ok, U.BODY_REDUCE, reds) == U.OK
    bad = U.loop_desc(0, 100, simdlen=5000)
    assert U.upir_loop_validate(U.spmd_desc(1, 32), bad, U.BODY_REDUCE, reds) == U.E_INVALID

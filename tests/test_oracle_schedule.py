"""Pins of the oracle's iteration space and schedule (o1, o2, o3).

Each pin is something other than the oracle itself: SPEC.md's worked
examples (tests/golden/spec_examples.json), GCC libgomp's static schedules
(tests/golden/libgomp_static.json, an independent OpenMP runtime), closed
forms, brute-force enumeration and partition invariants.
"""
import itertools
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

SPEC = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


# ---- o1 trip count ------------------------------------------------------------
@pytest.mark.parametrize("lb,ub,step", [(0, 10, 1), (0, 10, 3), (5, 5, 1), (7, 3, 1),
                                        (10, 0, -1), (10, 0, -3), (-4, 9, 2), (3, 7, -1),
                                        (0, 1, 100), (-10, -20, -4)])
def test_trip_count_bruteforce(lb, ub, step):
    # brute force: count the induction values a C for-loop would visit
    cnt, i = 0, lb
    while (i < ub) if step > 0 else (i > ub):
        cnt += 1
        i += step
    assert oracle.trip_count(lb, ub, step) == cnt


def test_trip_count_zero_step_invalid():
    assert oracle.trip_count(0, 10, 0) == -1


def test_trip_count_large_int64():
    # reading c2: int64 everywhere; T = 2^34 (C5) must not overflow
    assert oracle.trip_count(0, 1 << 34, 1) == 1 << 34
    assert oracle.trip_count(0, (1 << 34) + 1, 2) == (1 << 33) + 1


# ---- o1 collapse --------------------------------------------------------------
def test_collapse_spec_example():
    T = SPEC["collapse_4x3"]["T"]
    seq = [oracle.delinearize(T, t) for t in range(12)]
    assert seq == list(itertools.product(range(4), range(3)))


@pytest.mark.parametrize("T", [(3, 5), (1, 7), (2, 3, 4), (5, 1, 2), (6,)])
def test_collapse_lexicographic_bruteforce(T):
    n = math.prod(T)
    seq = [oracle.delinearize(list(T), t) for t in range(n)]
    assert seq == list(itertools.product(*[range(d) for d in T]))


# ---- o2 static: SPEC worked examples -----------------------------------------
@pytest.mark.parametrize("key", ["static_T10_p3", "static_chunk2_T8_p2", "static_p1"])
def test_static_spec_examples(key):
    ex = SPEC[key]
    for u, exp in enumerate(ex["expect"]):
        got = oracle.schedule_chunks(oracle.STATIC, ex["chunk"], ex["T"], ex["p"], u)
        assert [list(c) for c in got] == exp, ex["cite"]


def test_empty_T0():
    ex = SPEC["empty_T0"]
    for policy, c in ((oracle.STATIC, 0), (oracle.STATIC, 2), (oracle.DYNAMIC, 1)):
        for u in range(ex["p"]):
            assert oracle.schedule_chunks(policy, c, 0, ex["p"], u) == []


# ---- o2 static vs GCC libgomp (independent library) --------------------------
def test_static_matches_libgomp():
    data = json.load(open(os.path.join(GOLDEN, "libgomp_static.json")))
    assert len(data["cases"]) > 1000
    for T, p, c, own in data["cases"]:
        got = oracle.owner_map(oracle.STATIC, c, T, p)
        assert got.tolist() == own, (T, p, c)


def test_runtime_auto_resolve_to_static():
    for pol in (oracle.RUNTIME, oracle.AUTO):
        assert (oracle.owner_map(pol, 0, 37, 5) == oracle.owner_map(oracle.STATIC, 0, 37, 5)).all()


# ---- o2/o3 partition invariants (SPEC.md:363 property) -----------------------
def _check_partition(policy, c, T, p):
    seen = np.zeros(T, dtype=np.int64)
    for u in range(p):
        chunks = oracle.schedule_chunks(policy, c, T, p, u)
        prev = -1
        for lo, hi in chunks:
            assert 0 <= lo < hi <= T
            assert lo > prev            # each unit's chunks strictly increasing
            prev = lo
            seen[lo:hi] += 1
    assert (seen == 1).all()           # disjoint, union = [0, T)


def test_partition_exhaustive_small():
    for T in range(0, 65):
        for p in range(1, 10):
            for c in (0, 1, 2, 3, 7, 17):
                _check_partition(oracle.STATIC, c, T, p)
                if c:
                    _check_partition(oracle.DYNAMIC, c, T, p)


def test_partition_sampled_large():
    rng = random.Random(2209)
    for _ in range(60):
        T = rng.randrange(0, 10_001)
        p = rng.randrange(1, 65)
        c = rng.randrange(0, 18)
        _check_partition(oracle.STATIC, c, T, p)


def test_static_block_sizes_closed_form():
    # static without chunk: first T mod p units get ceil(T/p), rest floor(T/p)
    for T, p in ((10, 3), (1000, 7), (5, 8), (2 ** 20 + 3, 148 * 256)):
        for u in (0, p // 2, p - 1):
            ch = oracle.schedule_chunks(oracle.STATIC, 0, T, p, u)
            length = sum(h - l for l, h in ch)
            assert length == (T // p + (1 if u < T % p else 0))


# ---- o3 dynamic ---------------------------------------------------------------
def test_dynamic_spec_example():
    ex = SPEC["dynamic_c1_T4_p2"]
    got = oracle.owner_map(oracle.DYNAMIC, ex["chunk"], ex["T"], ex["p"])
    assert got.tolist() == ex["expect_owner"], ex["cite"]


def test_dynamic_default_chunk_is_one():
    assert (oracle.owner_map(oracle.DYNAMIC, 0, 9, 4) == oracle.owner_map(oracle.DYNAMIC, 1, 9, 4)).all()


def test_dynamic_chunk_boundaries():
    # the chunk partition of dynamic,c is {[kc, min((k+1)c, T))}
    T, p, c = 103, 5, 8
    allchunks = sorted(ch for u in range(p) for ch in oracle.schedule_chunks(oracle.DYNAMIC, c, T, p, u))
    assert allchunks == [(k * c, min((k + 1) * c, T)) for k in range((T + c - 1) // c)]


# ---- guided ---------------------------------------------
def _guided_bounds(T, p, c):
    return sorted(lo for u in range(p) for lo, hi in oracle.schedule_chunks(oracle.GUIDED, c, T, p, u))


def test_guided_boundaries_vs_libgomp():
    # independent runtime: every run start libgomp shows is a chunk boundary of
    # the oracle, and across 12 runs most boundaries are observed
    data = json.load(open(os.path.join(GOLDEN, "libgomp_guided.json")))
    seen = total = 0
    for T, p, c, starts in data["cases"]:
        b = set(_guided_bounds(T, p, c))
        assert set(starts) <= b, (T, p, c)
        seen += len(starts)
        total += len(b)
    assert seen >= 0.6 * total


def test_guided_partition_and_special_cases():
    for T in (0, 1, 10, 97, 1000):
        for p in (1, 2, 5, 16):
            for c in (0, 1, 3, 50):
                _check_partition(oracle.GUIDED, c, T, p)
    # p = 1: one chunk [0, T); c >= T: one chunk
    assert oracle.schedule_chunks(oracle.GUIDED, 1, 37, 1, 0) == [(0, 37)]
    assert _guided_bounds(37, 4, 100) == [0]
    # first chunk is ceil(T/p); chunk sizes never grow
    b = _guided_bounds(1000, 7, 1) + [1000]
    sizes = [b[i + 1] - b[i] for i in range(len(b) - 1)]
    assert sizes[0] == 143 and all(sizes[i] >= sizes[i + 1] for i in range(len(sizes) - 1))


def test_tile_owner_static1_round_robin():
    # tile loop static,1 over p teams: tile tau -> team tau mod p (chunk rule)
    own = oracle.tile_owner(10, 20, 3, 7, oracle.STATIC, 1, 4)
    ntiles = 4 * 3
    assert own.tolist() == [t % 4 for t in range(ntiles)]


def test_tiled_owner_bruteforce():
    # brute force from the reading: tiles anchored at 0, tile loop static,1
    # over teams, box positions static,ic over units, out-of-space positions -1
    lb0, ub0, lb1, ub1, BM, BN = 1, 10, 1, 13, 4, 8
    team, unit = oracle.tiled_owner(lb0, ub0, lb1, ub1, BM, BN, oracle.STATIC, 1, 3, 4, 5)
    tiles = [(ti, tj) for ti in range(0, 3) for tj in range(0, 2)]
    t = 0
    for tid, (ti, tj) in enumerate(tiles):
        for pos in range(BM * BN):
            i, j = ti * BM + pos // BN, tj * BN + pos % BN
            if lb0 <= i < ub0 and lb1 <= j < ub1:
                assert team[t] == tid % 3 and unit[t] == (pos // 4) % 5
            else:
                assert team[t] == -1 and unit[t] == -1
            t += 1
    assert t == len(team)
    # every iteration appears exactly once
    assert (team >= 0).sum() == (ub0 - lb0) * (ub1 - lb1)


@pytest.mark.parametrize("policy,chunk,p", [(0, 1, 3), (0, 0, 4), (0, 2, 5)])
def test_tiled_owner_colmajor_bruteforce(policy, chunk, p):
    """Reading c35: tile ids enumerate the tile grid column-major; the tile
    loop schedule and the intra-tile rule are unchanged.  Brute force of the
    reading (static block / static,c written out), and the set of executed
    (i, j) equals the row-major enumeration's."""
    lb0, ub0, lb1, ub1, BM, BN, ic, units = 1, 10, 1, 13, 4, 8, 4, 5
    team, unit = oracle.tiled_owner(lb0, ub0, lb1, ub1, BM, BN, oracle.STATIC, chunk, p, ic, units, colmajor=True)
    ntr, ntc = 3, 2
    nt = ntr * ntc
    tiles = [(ti, tj) for tj in range(ntc) for ti in range(ntr)]     # column-major ids

    def tile_team(tid):
        if chunk == 0:       # static block: first nt % p teams get one more
            q, r = divmod(nt, p)
            lo = 0
            for u in range(p):
                n = q + (u < r)
                if lo <= tid < lo + n:
                    return u
                lo += n
        return (tid // chunk) % p
    t = 0
    seen = set()
    for tid, (ti, tj) in enumerate(tiles):
        for pos in range(BM * BN):
            i, j = ti * BM + pos // BN, tj * BN + pos % BN
            if lb0 <= i < ub0 and lb1 <= j < ub1:
                assert team[t] == tile_team(tid) and unit[t] == (pos // ic) % units
                seen.add((i, j))
            else:
                assert team[t] == -1 and unit[t] == -1
            t += 1
    assert seen == {(i, j) for i in range(lb0, ub0) for j in range(lb1, ub1)}
    # a row-major run gives the same per-position unit map within each tile
    team_r, unit_r = oracle.tiled_owner(lb0, ub0, lb1, ub1, BM, BN, oracle.STATIC, chunk, p, ic, units)
    P = BM * BN
    for tid, (ti, tj) in enumerate(tiles):
        rid = ti * ntc + tj
        assert (unit[tid * P:(tid + 1) * P] == unit_r[rid * P:(rid + 1) * P]).all()


# ---- simd(simdlen) combined with worksharing (reading c33) -------------------------
SIMD_CASES = [(T, p, s) for T in (0, 1, 7, 64, 100, 1001) for p in (1, 3, 8) for s in (2, 4, 8)]


@pytest.mark.parametrize("T,p,s", SIMD_CASES)
def test_simd_static_chunk_is_openmp_simd_modifier(T, p, s):
    # OpenMP 4.5 2.7.1 'simd' schedule modifier: chunk_size becomes
    # simd_width * ceil(chunk_size / simd_width) -- a plain static,c' schedule
    for c in (1, 3, 5, 8, 13):
        c2 = s * math.ceil(c / s)
        for u in range(p):
            assert oracle.schedule_chunks(oracle.STATIC, c, T, p, u, simdlen=s) == \
                oracle.schedule_chunks(oracle.STATIC, c2, T, p, u)


@pytest.mark.parametrize("T,p,s", SIMD_CASES)
def test_simd_dynamic_partition_and_default_chunk(T, p, s):
    # chunk partition of dynamic,c under simd = that of dynamic,s*ceil(c/s);
    # the default chunk (1 iteration) becomes one SIMD group of s iterations
    for c, c2 in ((0, s), (1, s), (5, s * math.ceil(5 / s))):
        got = sorted(ch for u in range(p) for ch in oracle.schedule_chunks(oracle.DYNAMIC, c, T, p, u, simdlen=s))
        want = [(k, min(k + c2, T)) for k in range(0, T, c2)]
        assert got == want


@pytest.mark.parametrize("T,p,s", SIMD_CASES)
def test_simd_static_block_over_groups(T, p, s):
    # brute force of the strip-mined block rule: G = ceil(T/s) groups, the
    # first G mod p units own one group more; boundaries are multiples of s
    G = -(-T // s)
    q, r = divmod(G, p)
    for u in range(p):
        g0 = u * q + min(u, r)
        g1 = g0 + q + (1 if u < r else 0)
        want = [(g0 * s, min(g1 * s, T))] if g1 > g0 else []
        assert oracle.schedule_chunks(oracle.STATIC, 0, T, p, u, simdlen=s) == want
    if T % (s * p) == 0:   # groups split evenly: the plain block rule
        for u in range(p):
            assert oracle.schedule_chunks(oracle.STATIC, 0, T, p, u, simdlen=s) == \
                oracle.schedule_chunks(oracle.STATIC, 0, T, p, u)


@pytest.mark.parametrize("T,p,s", SIMD_CASES)
def test_simd_every_policy_partitions_on_group_boundaries(T, p, s):
    for pol, c in ((oracle.STATIC, 0), (oracle.STATIC, 3), (oracle.DYNAMIC, 2), (oracle.GUIDED, 0),
                   (oracle.GUIDED, 5)):
        owner = oracle.owner_map(pol, c, T, p, simdlen=s)
        assert (owner >= 0).all() and (owner < p).all()
        # each SIMD group (s consecutive iterations) is executed by one unit
        for g0 in range(0, T, s):
            assert len(set(owner[g0:g0 + s].tolist())) == 1
        chunks = [ch for u in range(p) for ch in oracle.schedule_chunks(pol, c, T, p, u, simdlen=s)]
        assert all(a % s == 0 and (b % s == 0 or b == T) for a, b in chunks)


@pytest.mark.parametrize("T,p,s", [(1000, 3, 4), (4099, 8, 8), (17, 5, 2)])
def test_simd_guided_group_sizes(T, p, s):
    # guided over groups: chunk = max(ceil(remaining groups / p), ceil(c/s)) groups
    c = 6
    chunks = sorted(ch for u in range(p) for ch in oracle.schedule_chunks(oracle.GUIDED, c, T, p, u, simdlen=s))
    G, g = -(-T // s), 0
    for a, b in chunks:
        assert a == g * s
        n = max(-(-(G - g) // p), -(-c // s))
        n = min(n, G - g)
        assert b == min((g + n) * s, T)
        g += n
    assert g == G


def test_simdlen_one_is_plain():
    for pol, c in ((oracle.STATIC, 0), (oracle.STATIC, 7), (oracle.DYNAMIC, 3), (oracle.GUIDED, 2)):
        for u in range(4):
            assert oracle.schedule_chunks(pol, c, 99, 4, u, simdlen=1) == oracle.schedule_chunks(pol, c, 99, 4, u)


@pytest.mark.parametrize("colmajor", [False, True])
@pytest.mark.parametrize("chunk,p", [(1, 3), (0, 4), (2, 5)])
def test_tiled_owner_reverse_bruteforce(colmajor, chunk, p):
    """Reading c38: with the reversed tile order, id k is the tile the plain
    (row- or column-major) order numbers nt - 1 - k; the tile-loop schedule
    maps ids to teams unchanged and the intra-tile rule is unchanged.  Brute
    force of the reading, and every iteration executed exactly once."""
    lb0, ub0, lb1, ub1, BM, BN, ic, units = 1, 10, 1, 13, 4, 8, 4, 5
    team, unit = oracle.tiled_owner(lb0, ub0, lb1, ub1, BM, BN, oracle.STATIC, chunk, p, ic, units,
                                    colmajor=colmajor, reverse=True)
    ntr, ntc = 3, 2
    nt = ntr * ntc
    plain = ([(ti, tj) for tj in range(ntc) for ti in range(ntr)] if colmajor
             else [(ti, tj) for ti in range(ntr) for tj in range(ntc)])
    tiles = [plain[nt - 1 - k] for k in range(nt)]

    def tile_team(tid):
        if chunk == 0:
            q, r = divmod(nt, p)
            lo = 0
            for u in range(p):
                n = q + (u < r)
                if lo <= tid < lo + n:
                    return u
                lo += n
        return (tid // chunk) % p
    t = 0
    seen = []
    for tid, (ti, tj) in enumerate(tiles):
        for pos in range(BM * BN):
            i, j = ti * BM + pos // BN, tj * BN + pos % BN
            if lb0 <= i < ub0 and lb1 <= j < ub1:
                assert team[t] == tile_team(tid) and unit[t] == (pos // ic) % units
                seen.append((i, j))
            else:
                assert team[t] == -1 and unit[t] == -1
            t += 1
    assert sorted(seen) == [(i, j) for i in range(lb0, ub0) for j in range(lb1, ub1)]

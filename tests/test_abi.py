"""The C ABI without a GPU: the library loads, exports every symbol
include/bz.h declares, its host-only work planner partitions each round's
combination space exactly (across any number of shards), and compute
entry points fail loudly when no device is present."""

from __future__ import annotations

import ctypes
import itertools
import os
import re
from math import comb

import pytest

from oracle import oracle
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.errors import InvalidArity, NoDevice, TooLarge

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "bz.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*(bz_\w+)\s*\(",
                                 text, re.M)))


def test_header_symbols_exported():
    L = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    assert set(syms) == set(_native.SYMBOLS)
    for s in syms:
        assert hasattr(L, s), s
    assert L.bz_abi_version() == _native.ABI_VERSION


@pytest.mark.parametrize("engine", ["auto", "popc", "imma", "umma", "mxf4", "mxf4p", "mxf4t", "mxf4q",
                                    "mxf4w", "mxf4f"])
def test_plan_counts(engine):
    for (m, k, g) in [(1, 5, 1), (2, 24, 3), (2, 80, 8), (3, 40, 8), (1, 64, 6), (2, 128, 4)]:
        groups, nchunks = _native.plan(m, k, g, engine)
        assert sum(gr[5] for gr in groups) == m * comb(k, g)
        assert nchunks >= 1
        starts = [gr[0] for gr in groups]
        assert starts == sorted(starts) and starts[0] == 0
        for gr in groups:
            begin, nprefix, gamma, ell, ppl, combos, depth, lanes, spc, nsb, sfloor, sl = gr
            assert nsb >= 1 and (depth < 3 or spc * nsb >= comb(k - sfloor, depth))
            # (K5 family: sl = 0 marks a merged group -- every prefix below a
            # level's floor, the (g - depth)-subsets of [0, ell + 1))
            assert sl in (1, 2, 4, 8, 16, 32) if depth < 3 else sl in (0, 1)
            merged = depth >= 3 and sl == 0
            assert lanes == ({"imma": 256}.get(engine, 128) if depth >= 3 else 32)
            want = 3 if (engine != "popc" and g >= 4) else (2 if g >= 4 else 1)
            if engine in ("auto", "mxf4", "mxf4p", "mxf4t", "mxf4q", "mxf4w", "mxf4f") and g >= 4:
                # K5 suffix levels: depth 3..5, floors above ell + 1
                assert 3 <= depth <= min(5, g - 1) and sfloor >= ell + 1
            else:
                assert depth == want and sfloor == ell + 1
            assert nprefix == (1 if g == 1 else comb(ell + 1, g - depth) if merged
                               else comb(ell, g - 1 - depth))
            assert not merged or depth > 3
            assert combos == nprefix * comb(k - sfloor, depth)


@pytest.mark.parametrize("engine", ["auto", "popc", "imma", "umma", "mxf4", "mxf4p", "mxf4t", "mxf4q",
                                    "mxf4w", "mxf4f"])
@pytest.mark.parametrize("m,k,g", [(1, 6, 1), (1, 7, 2), (2, 9, 3), (1, 12, 5),
                                   (2, 10, 10), (1, 40, 3), (1, 34, 4), (1, 20, 6)])
def test_plan_partitions_rank_space(m, k, g, engine):
    """Every g-combination of every Gamma is visited exactly once, for any
    shard count, by the device's chunk/lane/colex walk."""
    import random

    rng = random.Random(k * 100 + g)
    n = 2 * k + 5
    gammas = [[rng.getrandbits(n) for _ in range(k)] for _ in range(m)]
    expect = sorted(oracle.all_combinations(m, k, g))
    for nshards in (1, 2, 3, 8):
        groups, nchunks = _native.plan(m, k, g, engine, nshards)
        seen = []
        mins = [None] * m
        for s in range(nshards):
            mn, _, got = oracle.enumerate_chunks(gammas, k, g, groups, nchunks, s, nshards)
            seen += got
            mins = [a if b is None else (b if a is None else min(a, b))
                    for a, b in zip(mins, mn)]
        assert sorted(seen) == expect
        for j in range(m):
            assert mins[j] == oracle.min_weight(gammas[j], n, g)[0]


def test_plan_errors():
    with pytest.raises(InvalidArity):
        _native.plan(1, 5, 6)
    with pytest.raises(InvalidArity):
        _native.plan(1, 5, 0)
    with pytest.raises(TooLarge):
        _native.plan(1, 128, 40)


def test_no_device_fails_loudly():
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(NoDevice):
        _native.Context(0)


def test_colex_unrank_bijective():
    for ell in range(0, 12):
        for q in range(0, min(ell, 5) + 1):
            subs = [tuple(oracle.colex_unrank(r, q, ell)) for r in range(comb(ell, q))]
            assert sorted(subs) == sorted(itertools.combinations(range(ell), q))


@pytest.mark.parametrize("m,k,g,floors", [(1, 12, 6, "4,7"), (2, 10, 7, "4"), (1, 14, 8, "5,9"),
                                          (1, 12, 5, "6"), (1, 11, 9, "0,3")])
def test_plan_levels_partition(monkeypatch, m, k, g, floors):
    """K5 suffix levels (forced floors): the depth-3/4/5 groups still visit
    every g-combination exactly once, for any shard count."""
    import collections
    import random

    monkeypatch.setenv("BZ_K5_FLOORS", floors)
    rng = random.Random(k * 31 + g)
    n = 2 * k + 3
    gammas = [[rng.getrandbits(n) for _ in range(k)] for _ in range(m)]
    expect = sorted(oracle.all_combinations(m, k, g))
    groups, _ = _native.plan(m, k, g, "mxf4")
    assert max(collections.Counter(int(gr[6]) for gr in groups)) > 3  # deeper levels in use
    for engine, nshards in (("mxf4", 1), ("mxf4", 3), ("mxf4p", 1), ("mxf4p", 3), ("mxf4t", 3), ("mxf4q", 3),
                            ("mxf4w", 2), ("mxf4f", 2)):
        groups, nchunks = _native.plan(m, k, g, engine, nshards)
        seen = []
        for s in range(nshards):
            _, _, got = oracle.enumerate_chunks(gammas, k, g, groups, nchunks, s, nshards)
            seen += got
        assert sorted(seen) == expect


def test_plan_levels_auto_cfg5():
    """The cost model splits the cfg5 top round into levels and keeps the
    combination count exact."""
    groups, _ = _native.plan(2, 80, 8, "mxf4")
    depths = {int(gr[6]) for gr in groups}
    assert depths >= {3, 4}
    assert sum(int(gr[5]) for gr in groups) == 2 * comb(80, 8)


def test_k5q_offset_encoding():
    """Host-only (no device): K5q's producer threshold and e2m1 offset blocks
    over every prefix stored weight 0..128 and bound -4..128 stay in range
    (thr in [1, 128], offset x <= 238) and dot to their integers exactly
    (bz_k5q_selftest runs the kernel's own k5q_threshold / pad_chunk)."""
    bad, first = _native.k5q_selftest()
    assert bad == 0, first


def test_k5q_offset_encoding_restated():
    """Independent restatement of the same check in Python: the A offset
    block for T (6.0 on the table's 4.0 elements while 24 fit, the rest on
    the 1.0 elements) dots to T for every T in 0..238, and the producer's
    threshold keeps x = wt + 128 - thr in that range."""
    for T in range(239):
        k6 = min(8, T // 24)
        rest = T - 24 * k6           # on eight 1.0 elements: 6.0s then the remainder
        n6 = min(rest // 6, 8)
        rem = rest - 6 * n6
        assert 24 * k6 + 6 * n6 + rem == T and (n6 < 8 or rem == 0)
        assert rem <= 5 and (rem < 5 or n6 <= 6)  # 5 = 4.0 + 1.0 on the next element
    for wt in range(129):
        for rel in range(-4, 129):  # bounds start capped at the stored columns (<= 128)
            thr = max(wt - 110, max(1, min(128, rel)))
            x = wt + 128 - thr
            assert 1 <= thr <= 128 and 0 <= x <= 238
            assert thr >= rel and 128 + 128 - thr <= 255  # stored weight 128 still a byte

"""Row-level operation counters (row_additions / row_accesses,
m/enumeration.py:19-24): the device counts them (bz_counters) for its
prefix-sum + stored-row decomposition of every combination, and the oracle
(oracle.expected_counters) recounts them from the work plan alone.

CPU: closed forms of the counting model (one addition per codeword, the
partial sums of K1's depth-2 suffix loop, the walkers' colex updates) and the
ratios the paper is about -- additions per combination close to one, and
many combinations per row access.  GPU: the device's counts equal the
oracle's exactly, per Gamma, for every kernel family, batched rounds, shards
and minimum_distance reports."""

from __future__ import annotations

import random
from math import comb

import numpy as np
import pytest

from oracle import oracle
from paper_1603_06757_b200 import _native

ENGINES = ("popc", "mxf4", "mxf4q", "mxf4w", "mxf4f")


def _plan(m, k, g, engine, nshards=1):
    return _native.plan(m, k, g, engine, nshards)


def test_counters_closed_forms_k1():
    """K1 plans: g = 1 and 2 cost one addition per codeword (Lemma 2/3
    with a stored single row), g = 3 adds one partial sum per (prefix, e1);
    the prefix {ell} needs no walker additions."""
    k = 29
    for g, want_adds in ((1, comb(k, 1)), (2, comb(k, 2)), (3, comb(k, 3) + comb(k - 1, 2))):
        groups, nch = _plan(1, k, g, "popc")
        adds, accs = oracle.expected_counters(1, k, g, groups, nch)
        assert adds[0] == want_adds, (g, adds[0], want_adds)
        assert 0 < accs[0] < adds[0] + 64 * len(groups)


def test_counters_walker_cost():
    """A walker over the whole colex order of the q-subsets of [0, ell)
    does q additions for its first subset and 2 or 3 per successor."""
    q, ell = 3, 12
    n = comb(ell, q)
    cost = oracle._walk_cost(0, n, q, ell)
    assert 3 + 2 * (n - 1) <= cost <= 3 + 3 * (n - 1)
    # splitting the range re-pays the second half's init (q) instead of the
    # successor step from rank 99 to 100
    step99 = oracle._walk_cost(99, 2, q, ell) - q
    assert oracle._walk_cost(0, 100, q, ell) + oracle._walk_cost(100, n - 100, q, ell) \
        == cost + q - step99
    assert oracle._walk_cost(100, 1, q, ell) == q


@pytest.mark.parametrize("engine", ENGINES)
def test_counters_ratios(engine):
    """Additions per combination stay within a few percent of one (each
    codeword is one prefix sum combined with one stored row), and every row
    access serves many codewords -- up to 64 per suffix-row load in K1 (32
    lanes x 2 walkers; every lane's walker also reads its own prefix-table
    rows), up to 128 per stored-row load in K5/K5q: the paper's "more
    additions per row access" (section 3.5) at GPU scale."""
    k, g = 48, 6
    groups, nch = _plan(2, k, g, engine)
    adds, accs = oracle.expected_counters(2, k, g, groups, nch)
    combos = 2 * comb(k, g)
    assert combos <= sum(adds) <= 1.25 * combos
    assert sum(accs) * (8 if engine == "popc" else 30) < combos


def test_counters_shards_partition():
    """Shard counts sum to the whole round's (chunk c -> shard c % n)."""
    k, g = 30, 5
    for engine in ENGINES:
        groups, nch = _plan(2, k, g, engine)
        whole = oracle.expected_counters(2, k, g, groups, nch)
        for nshards in (2, 3):
            gs3, n3 = _plan(2, k, g, engine, nshards)
            parts = [oracle.expected_counters(2, k, g, gs3, n3, s, nshards) for s in range(nshards)]
            assert [sum(p[0][j] for p in parts) for j in range(2)] == whole[0]
            assert [sum(p[1][j] for p in parts) for j in range(2)] == whole[1]


# ------------------------------------------------------------------------ GPU

gpu = pytest.mark.gpu


def _family(m, k, n, seed):
    rng = random.Random(seed)
    return [[rng.getrandbits(n) for _ in range(k)] for _ in range(m)]


def _load(ctx, fam, n):
    words = np.stack([oracle.words64(rows, n) for rows in fam]).astype(np.uint64)
    ctx.set_elision(False)
    ctx.load(words, n)


@gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_device_counters_match_oracle(engine):
    ctx = _native.context(0)
    m, k, n = 2, 26, 80
    fam = _family(m, k, n, 11)
    try:
        with ctx.lock:
            ctx.set_engine(engine)
            _load(ctx, fam, n)
            for g in range(1, 7):
                mins, combos = ctx.round(g, -1, 1 << 20)
                adds, accs = ctx.counters(1)
                groups, nch = _plan(m, k, g, engine)
                want = oracle.expected_counters(m, k, g, groups, nch)
                assert combos == [comb(k, g)] * m
                assert adds[0] == want[0], (engine, g)
                assert accs[0] == want[1], (engine, g)
            # a round too small to split runs whole on one rank (bz.cu
            # run_batch: shard 0 here), the others report nothing
            groups, nch = _plan(m, k, 5, engine)
            whole = oracle.expected_counters(m, k, 5, groups, nch)
            for shard in range(3):
                ctx.round(5, -1, 1 << 20, shard, 3)
                adds, accs = ctx.counters(1)
                assert (adds[0], accs[0]) == (whole if shard == 0 else ([0] * m, [0] * m))
            # a batch of rounds (fused launches) reports every round's counts
            res = ctx.rounds(1, [-1] * 6, 1 << 20)
            adds, accs = ctx.counters(6)
            for i in range(6):
                groups, nch = _plan(m, k, i + 1, engine)
                assert (adds[i], accs[i]) == oracle.expected_counters(m, k, i + 1, groups, nch)
            assert len(res) == 6
            # a round large enough to be split over 2 shards (2 C(60,7) =
            # 7.7e8 combinations): each shard's counts of its own chunks
            big = _family(2, 60, 100, 12)
            _load(ctx, big, 100)
            groups, nch = _plan(2, 60, 7, engine, 2)
            for shard in range(2):
                ctx.round(7, -1, 1 << 20, shard, 2)
                adds, accs = ctx.counters(1)
                assert (adds[0], accs[0]) == \
                    oracle.expected_counters(2, 60, 7, groups, nch, shard, 2), (engine, shard)
    finally:
        ctx.set_engine("auto")
        ctx.set_elision(True)


@gpu
def test_report_counters_through_minimum_distance():
    """minimum_distance sums the device counters over its rounds; the
    enumerate_gpu drop-in reports the pass's own."""
    from paper_1603_06757_b200 import BitMatrix, EngineConfig, enumerate_gpu, minimum_distance

    rng = random.Random(5)
    G = BitMatrix([rng.getrandbits(60) for _ in range(22)], 60)
    rep = minimum_distance(G, EngineConfig(engine="popc"))
    c = rep.counters
    assert c.combinations <= c.row_additions <= 1.5 * c.combinations
    assert 0 < c.row_accesses < c.row_additions
    res = enumerate_gpu(G, 4)
    assert res.combinations == comb(22, 4)
    assert res.combinations <= res.row_additions <= 1.5 * res.combinations
    assert 0 < res.row_accesses < res.row_additions

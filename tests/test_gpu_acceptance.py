"""Acceptance-style checks of the GPU path (the reference's acceptance
criteria, t/test_acceptance.py: random codes against brute force, known
codes, reproducibility; its hypothesis property tests, t/test_gf2.py): the
whole minimum_distance loop on the B200 against the C oracle's Gray-code
brute force, for every engine."""

from __future__ import annotations

import random
from math import comb

import pytest

from oracle import oracle
from paper_1603_06757_b200 import (BitMatrix, EngineConfig, RankDeficient, enumerate_gpu,
                                   minimum_distance)
from paper_1603_06757_b200.constructions import cyclic_code_generator, extend_code

pytestmark = pytest.mark.gpu


def _random_codes(count: int, seed: int):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        k = rng.randint(1, 14)
        n = rng.randint(k + 1, 3 * k + 12)
        density = rng.choice((0.2, 0.5, 0.8))
        rows = [sum(1 << b for b in range(n) if rng.random() < density) for _ in range(k)]
        out.append((rows, n))
    return out


@pytest.mark.parametrize("engine", ["auto", "popc", "mxf4", "mxf4q", "mxf4w", "mxf4f"])
def test_random_codes_match_brute_force(engine):
    """500 random codes (k <= 14, sparse / balanced / dense rows): the GPU
    distance equals the brute force over all 2^k - 1 messages, the status
    is exact and the trace obeys the BZ discipline; rank-deficient
    generators raise RankDeficient like the reference."""
    checked = deficient = 0
    for rows, n in _random_codes(500, 2026 + len(engine)):
        G = BitMatrix(rows, n)
        try:
            rep = minimum_distance(G, EngineConfig(engine=engine))
        except RankDeficient:
            deficient += 1
            continue
        assert rep.distance == oracle.brute_distance(rows, n), (rows, n)
        assert rep.exact
        ls = [L for _, L, _ in rep.bounds_trace]
        us = [U for _, _, U in rep.bounds_trace]
        assert ls == sorted(ls) and us == sorted(us, reverse=True)
        assert rep.distance <= n - len(rows) + 1
        checked += 1
    assert checked >= 300 and deficient > 0


def test_known_codes():
    """Hamming [7,4,3] (cyclic, g(x) = 1 + x + x^3), the binary Golay code
    [23,12,7] (g(x) = 1 + x^2 + x^4 + x^5 + x^6 + x^10 + x^11) and its
    extension [24,12,8], a repetition code [9,1,9] and a single-parity-check
    code [12,11,2]."""
    hamming = cyclic_code_generator(0b1011, 7)
    golay = cyclic_code_generator(0b110001110101, 23)
    cases = [(hamming, 3), (golay, 7), (extend_code(golay), 8),
             (BitMatrix([(1 << 9) - 1], 9), 9),
             (BitMatrix([(1 << i) | (1 << 11) for i in range(11)], 12), 2)]
    for G, d in cases:
        for engine in ("auto", "popc"):
            rep = minimum_distance(G, EngineConfig(engine=engine))
            assert rep.distance == d and rep.exact, (G.num_cols, G.num_rows, engine)


def test_reproducible_reports():
    """The same generator twice (and on another engine): identical
    distance, trace, status, pivots and counters."""
    rng = random.Random(77)
    G = BitMatrix([rng.getrandbits(70) for _ in range(30)], 70)
    a = minimum_distance(G, EngineConfig())
    b = minimum_distance(G, EngineConfig())
    c = minimum_distance(G, EngineConfig(engine="popc"))
    for r in (b, c):
        assert (r.distance, r.status, r.g_reached, r.bounds_trace, r.pivot_sets) == \
            (a.distance, a.status, a.g_reached, a.bounds_trace, a.pivot_sets)
        assert r.counters.combinations == a.counters.combinations
    assert (b.counters.row_additions, b.counters.row_accesses) == \
        (a.counters.row_additions, a.counters.row_accesses)


def test_property_enumerate_matches_oracle():
    """Property test (hypothesis, as the reference's t/test_gf2.py:85-93):
    for random (k, n, g, rows, ubound) the GPU pass equals the oracle's
    enumerate_stack restatement, clipped to ubound."""
    hyp = pytest.importorskip("hypothesis")
    st = hyp.strategies

    @hyp.settings(max_examples=60, deadline=None, derandomize=True)
    @hyp.given(st.integers(1, 24), st.integers(1, 200), st.integers(1, 6),
               st.integers(0, 2**31 - 1), st.one_of(st.none(), st.integers(0, 120)))
    def check(k, n, g, seed, ubound):
        g = min(g, k)
        rng = random.Random(seed)
        rows = [rng.getrandbits(n) for _ in range(k)]
        res = enumerate_gpu(BitMatrix(rows, n), g, ubound)
        want = oracle.min_weight(rows, n, g)[0]
        assert res.min_weight == (want if ubound is None else min(want, ubound))
        assert res.combinations == comb(k, g)

    check()


@pytest.mark.parametrize("batch", [2_000_000_000, 0])
def test_native_loop_equals_python_loop(batch):
    """The loop on one rank runs natively (bz_advance); the Python loop it
    replaces (EngineConfig(native_loop=False)) gives the same report: trace,
    status, g_reached, every counter and each round's combinations -- with
    batching on and off, under max_g, and resumed from start_g /
    start_upper."""
    from paper_1603_06757_b200.configs import code

    rng = random.Random(5)
    cases = [code(name, seed)[0] for name, seed in (("cfg1", 1), ("cfg1", 2), ("cfg2", 1),
                                                     ("cfg3", 1), ("cfg5", 7))]
    cases += [BitMatrix([rng.getrandbits(n) for _ in range(k)], n)
              for k, n in ((9, 30), (20, 47), (33, 70), (60, 61))]
    extra = [dict(), dict(max_g=2), dict(max_g=1), dict(start_g=3, start_upper=30)]
    for G in cases:
        for kw in extra:
            try:
                a = minimum_distance(G, EngineConfig(batch_combinations=batch, **kw))
            except RankDeficient:
                break
            b = minimum_distance(G, EngineConfig(batch_combinations=batch, native_loop=False,
                                                 **kw))
            assert (a.distance, a.status, a.g_reached, a.bounds_trace) == \
                (b.distance, b.status, b.g_reached, b.bounds_trace), (G.num_rows, kw)
            assert (a.counters.combinations, a.counters.row_additions,
                    a.counters.row_accesses) == (b.counters.combinations,
                                                 b.counters.row_additions,
                                                 b.counters.row_accesses)
            assert [(r.g, r.combinations) for r in a.rounds] == \
                [(r.g, r.combinations) for r in b.rounds]

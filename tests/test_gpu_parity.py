"""Parity of the sm_100a kernels (through the C ABI) with the CPU oracle
and with the reference's golden outputs.  Needs a B200: run via gpurun
with `pytest -m gpu`.  Integer work, so every comparison is exact."""

from __future__ import annotations

import hashlib
import random
from math import comb

import numpy as np
import pytest

from conftest import CFG4_HIST_SHA256, hexrows
from oracle import oracle
from paper_1603_06757_b200 import (BitMatrix, EngineConfig, InvalidArity, TooLarge,
                                   enumerate_gpu, minimum_distance, weight_histogram_gpu)
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.configs import code, microbench_gamma
from paper_1603_06757_b200.enumeration import family_words

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return _native.context(0)


@pytest.fixture(params=["popc", "mxf4", "mxf4q", "mxf4w", "mxf4f"])
def engine(request):
    """Every kernel of the library: K1 (XOR+POPC), K5 (tcgen05 kind::mxf4,
    g >= 4), K5q (kind::mxf4nvf4, two codewords per accumulator as bytes;
    W <= 4 and <= 128 stored columns -- other shapes run K5) and K5w
    (kind::mxf4, two codewords as 11-bit fields; W >= 2); K5f (K5q's bytes from
    folded MMAs, odd W <= 3 whose last stored word holds <= 16 columns -- other
    shapes run K5q / K5)."""
    _native.context(0).set_engine(request.param)
    yield request.param
    _native.context(0).set_engine("auto")


def test_small_enum_fixtures(goldens, engine):
    for fx in goldens["small"]["enum"]:
        M = BitMatrix(hexrows(fx["rows"]), fx["n"])
        for g, expect in enumerate(fx["min_by_g"], start=1):
            res = enumerate_gpu(M, g)
            assert res.min_weight == expect, (fx["src"], g)
            assert res.combinations == comb(fx["k"], g)


def test_clipping_semantics():
    M = BitMatrix([random.Random(19).getrandbits(16) | (1 << i) for i in range(6)], 22)
    true_min = enumerate_gpu(M, 3).min_weight
    assert enumerate_gpu(M, 3, ubound=true_min - 1).min_weight == true_min - 1
    assert enumerate_gpu(M, 3, ubound=true_min + 5).min_weight == true_min
    assert enumerate_gpu(M, 3, ubound=true_min - 1).combinations == comb(6, 3)


def test_bad_arity():
    M = BitMatrix([1, 2, 4, 8], 5)
    with pytest.raises(InvalidArity):
        enumerate_gpu(M, 0)
    with pytest.raises(InvalidArity):
        enumerate_gpu(M, 5)


@pytest.mark.parametrize("n", [1, 7, 31, 32, 33, 64, 65, 100, 127, 160, 192, 200, 255, 256])
def test_word_widths(n, engine):
    """Every W = ceil(n/32) instantiation (1..8), padded and exact sizes."""
    rng = random.Random(n)
    k = min(12, n) if n > 1 else 1
    rows = [rng.getrandbits(n) for _ in range(k)]
    M = BitMatrix(rows, n)
    for g in range(1, k + 1):
        assert enumerate_gpu(M, g).min_weight == oracle.min_weight(rows, n, g)[0], (n, g)


@pytest.mark.parametrize("k,g", [(1, 1), (2, 2), (33, 3), (64, 4), (65, 3), (100, 3),
                                 (127, 2), (128, 3), (128, 128), (70, 69)])
def test_row_counts(k, g, engine):
    """Masks cross the 64-bit word boundary; g = k and g = k-1 edges."""
    rng = random.Random(k * 7 + g)
    n = 150
    rows = [rng.getrandbits(n) for _ in range(k)]
    M = BitMatrix(rows, n)
    assert enumerate_gpu(M, g).min_weight == oracle.min_weight(rows, n, g)[0]


def test_random_sweep_vs_oracle(engine):
    rng = random.Random(2024)
    for _ in range(40):
        k = rng.randint(2, 40)
        n = rng.randint(k, 256)
        rows = [rng.getrandbits(n) for _ in range(k)]
        M = BitMatrix(rows, n)
        for g in sorted({1, 2, min(k, 3), min(k, 4), min(k, 5), k}):
            if comb(k, g) > 3_000_000:
                continue
            assert enumerate_gpu(M, g).min_weight == oracle.min_weight(rows, n, g)[0], (k, n, g)


def test_zero_rows_and_duplicates(engine):
    rows = [0, 0, 5, 5, 7]
    M = BitMatrix(rows, 3)
    for g in range(1, 6):
        assert enumerate_gpu(M, g).min_weight == oracle.min_weight(rows, 3, g)[0]


def test_round_sharded_equals_whole(ctx, engine):
    G, gs, _ = code("cfg2", 1)
    ctx.load(family_words(gs.gammas, 96), 96)
    for g in (1, 2, 3, 4, 5, 6):
        whole_min, whole_c = ctx.round(g, 0, 10**6)
        for nshards in (2, 3, 8):
            mins = [10**9] * 2
            cs = [0, 0]
            for s in range(nshards):
                mn, c = ctx.round(g, 0, 10**6, s, nshards)
                mins = [min(a, b) for a, b in zip(mins, mn)]
                cs = [a + b for a, b in zip(cs, c)]
            assert mins == whole_min and cs == whole_c == [comb(48, g)] * 2
        assert whole_min == [oracle.min_weight(list(gm.rows), 96, g)[0] for gm in gs.gammas]


@pytest.mark.parametrize("idx", range(6))
def test_minimum_distance_configs(goldens, idx, engine):
    fx = goldens["configs"][idx]
    rep = minimum_distance(BitMatrix(hexrows(fx["rows"]), fx["n"]), EngineConfig(engine=engine))
    assert rep.distance == fx["distance"]
    assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]]
    assert (rep.status, rep.g_reached, rep.m, rep.k_m) == \
        (fx["status"], fx["g_reached"], fx["m"], fx["k_m"])
    assert [list(p) for p in rep.pivot_sets] == fx["pivot_sets"]
    assert rep.counters.combinations == fx["combinations"]


def test_early_exit_fixture(goldens):
    """cfg1 seed 2 round 3: U reaches L_prev = 6, the only exit that keeps
    the trace bit-exact (SURVEY.md 8(a) invariant 5)."""
    fx = [c for c in goldens["configs"] if (c["name"], c["seed"]) == ("cfg1", 2)][0]
    G = BitMatrix(hexrows(fx["rows"]), fx["n"])
    fast = minimum_distance(G, EngineConfig(early_exit=True))
    full = minimum_distance(G)  # default: full passes, the reference's counts
    for rep in (fast, full):
        assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]]
        assert rep.distance == 6
    assert full.counters.combinations == fx["combinations"]
    assert fast.counters.combinations <= full.counters.combinations


def test_small_codes(goldens, engine):
    for fx in goldens["small"]["codes"]:
        rep = minimum_distance(BitMatrix(hexrows(fx["rows"]), fx["n"]), EngineConfig(engine=engine))
        assert rep.distance == fx["distance"] == fx["brute"], fx["src"]
        assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]], fx["src"]


def test_cfg4_histogram(goldens):
    fx = goldens["cfg4"]
    M = microbench_gamma(1)
    assert [format(r, "x") for r in M.rows] == fx["rows"]
    hist, mn, combos = weight_histogram_gpu(M, 6)
    assert combos == comb(64, 6) == int(hist.sum())
    assert mn == fx["min_weight"] == 39
    assert hashlib.sha256(hist.astype("<u8").tobytes()).hexdigest() == CFG4_HIST_SHA256
    assert np.array_equal(hist, oracle.histogram(list(M.rows), 192, 6))
    assert enumerate_gpu(M, 6).min_weight == 39


def test_histogram_small_vs_oracle():
    rng = random.Random(11)
    for (k, n, g) in [(10, 40, 3), (20, 70, 4), (30, 256, 3), (16, 16, 5), (9, 33, 1)]:
        rows = [rng.getrandbits(n) for _ in range(k)]
        hist, mn, c = weight_histogram_gpu(BitMatrix(rows, n), g)
        assert np.array_equal(hist, oracle.histogram(rows, n, g)), (k, n, g)


@pytest.mark.gpu
def test_histogram_outside_window():
    """K1h keeps private counters for a window of 64 weights around the
    expected weight and sends the rest through its exact slow path: rows of
    very different densities spread the weights over the whole range."""
    rng = random.Random(23)
    for (k, n, g) in [(18, 200, 3), (16, 250, 4), (14, 130, 2), (12, 256, 3)]:
        full = (1 << n) - 1
        rows = []
        for i in range(k):
            r = rng.getrandbits(n)
            if i % 3 == 0:
                r &= rng.getrandbits(n) & rng.getrandbits(n)  # sparse
            elif i % 3 == 1:
                r |= rng.getrandbits(n) | rng.getrandbits(n)  # dense
            rows.append(r & full)
        rows[0] = 0
        rows[1] = full
        hist, mn, c = weight_histogram_gpu(BitMatrix(rows, n), g)
        want = oracle.histogram(rows, n, g)
        assert np.array_equal(hist, want), (k, n, g)
        assert c == comb(k, g) and mn == int(np.flatnonzero(want)[0])
        nz = np.flatnonzero(want)
        assert nz[-1] - nz[0] >= 64  # wider than the window


def test_cfg5_full(cfg5_golden, engine):
    fx = cfg5_golden
    G, gs, draws = code("cfg5", 7)
    assert [format(r, "x") for r in G.rows] == fx["rows"]
    rep = minimum_distance(G, EngineConfig(engine=engine))
    assert rep.distance == fx["distance"]
    assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]]
    assert rep.counters.combinations == fx["combinations"]


@pytest.mark.parametrize("mirror", [False, True])
@pytest.mark.parametrize("nshards", [2, 8])
def test_cfg5_batch_sharded(cfg5_golden, ctx, nshards, mirror):
    """BASELINE's multi-GPU configuration at full size, one rank at a time on
    this device: rounds 1..8 of config 5 as shard s of N in one batch each
    (what rank s launches), folded like the host exchange -- min of the
    minima, sum of the counts per round -- must reproduce the reference's U
    trajectory and combination count.  With the shared-bound mirror mapped
    (this context's own memory) every shard also thresholds with the finds of
    the shards before it and does not report minima at or above them: the
    fold must not change."""
    fx = cfg5_golden
    G, gs, _ = code("cfg5", 7)
    trace = [tuple(t) for t in fx["bounds_trace"]]
    lp = [0] + [t[1] for t in trace[:-1]]
    u0 = 160 - 80 + 1
    with ctx.lock:
        ctx.set_engine("auto")
        ctx.load(family_words(gs.gammas, 160), 160)
        if mirror:
            ctx.shared_bound_export()
            ctx.shared_bound_open(None)
            ctx.shared_bound_epoch(0x5000 + nshards)
        try:
            res = [ctx.rounds(1, lp, u0, s, nshards) for s in range(nshards)]
        finally:
            if mirror:
                ctx.shared_bound_close()
    run_min, total = u0, 0
    for g, (_, _, u_ref) in enumerate(trace):
        run_min = min([run_min] + [min(r[g][0]) for r in res])
        total += sum(sum(r[g][1]) for r in res)
        assert run_min == u_ref, (g + 1, run_min, u_ref)
    assert total == fx["combinations"]


def test_too_large(ctx):
    M = BitMatrix([(1 << i) for i in range(128)], 200)
    with pytest.raises(TooLarge):
        enumerate_gpu(M, 40)


_WIDE: dict = {}


@pytest.mark.parametrize("k,n", [(28, 280), (32, 288), (36, 290)])
def test_codes_wider_than_256(k, n, engine):
    """n up to 384: every Gamma keeps n - k <= 256 columns after identity
    elision (the remainder Gamma too), so the device rows still fit 8 words."""
    rng = random.Random(1000 * k + n)
    rows = [rng.getrandbits(n) for _ in range(k)]
    if (k, n) not in _WIDE:  # the C oracle, once per code (~5 s for k = 36)
        _WIDE[(k, n)] = oracle.minimum_distance(rows, n)
    want = _WIDE[(k, n)]
    try:
        rep = minimum_distance(BitMatrix(rows, n), EngineConfig(engine=engine))
    except TooLarge:
        raise
    assert rep.distance == want["distance"]
    assert rep.bounds_trace == [tuple(t) for t in want["bounds_trace"]]
    assert (rep.m, rep.k_m) == (want["m"], want["k_m"])
    assert rep.counters.combinations == want["combinations"]


def test_stored_columns_limit():
    """More than 256 stored columns, or n > 384, fail loudly."""
    rng = random.Random(5)
    rows = [rng.getrandbits(290) for _ in range(28)]  # n - k = 262 stored
    with pytest.raises(TooLarge):
        minimum_distance(BitMatrix(rows, 290))
    rows = [rng.getrandbits(400) for _ in range(128)]
    with pytest.raises(TooLarge):
        minimum_distance(BitMatrix(rows, 400))
    with pytest.raises(TooLarge):  # not systematic: every column is stored
        enumerate_gpu(BitMatrix([rng.getrandbits(300) for _ in range(20)], 300), 2)


@pytest.mark.parametrize("k,n,g", [(4, 9, 4), (5, 40, 4), (128, 256, 4), (100, 200, 5),
                                   (40, 224, 6), (30, 33, 7)])
def test_tensor_engine_shapes(k, n, g, engine):
    """Tensor-engine edge shapes: smallest suffix tables (k = 4, 5), wide
    rows (W = 7, 8), k = 128, slices smaller than one tile."""
    rng = random.Random(k * 1000 + n + g)
    rows = [rng.getrandbits(n) for _ in range(k)]
    M = BitMatrix(rows, n)
    # (100, 200, 5): 7.5e7 combinations, ~1 s in the threaded C oracle
    assert enumerate_gpu(M, g).min_weight == oracle.min_weight(rows, n, g)[0], (k, n, g)


def test_round_many_shards(ctx, engine):
    G, gs, _ = code("cfg2", 2)
    ctx.load(family_words(gs.gammas, 96), 96)
    for g in (4, 5, 6):
        whole_min, whole_c = ctx.round(g, 0, 10**6)
        mins, cs = [10**9] * 2, [0, 0]
        for s in range(5):
            mn, c = ctx.round(g, 0, 10**6, s, 5)
            mins = [min(a, b) for a, b in zip(mins, mn)]
            cs = [a + b for a, b in zip(cs, c)]
        assert mins == whole_min and cs == whole_c == [comb(48, g)] * 2


def test_early_exit_all_engines(ctx, engine):
    """With the in-round early exit on, once the running minimum reaches
    lower_prev the round stops; its result is then exactly lower_prev and
    fewer combinations are visited.  Off (the default), the same call visits
    every combination."""
    G, gs, _ = code("cfg2", 1)
    ctx.load(family_words(gs.gammas, 96), 96)
    for g in (4, 5):
        full_min, full_c = ctx.round(g, 0, 10**6)
        true_min = min(full_min)
        mins, combos = ctx.round(g, true_min, 10**6)
        assert (mins, combos) == (full_min, full_c) == (full_min, [comb(48, g)] * 2)
        ctx.set_early_exit(True)
        try:
            mins, combos = ctx.round(g, true_min, 10**6)
        finally:
            ctx.set_early_exit(False)
        assert min(mins) == true_min
        assert sum(combos) <= sum(full_c)


@pytest.mark.parametrize("k,g,floors", [(12, 6, "4,7"), (14, 8, "5,9"), (12, 5, "6"),
                                        (20, 7, "8,13"), (11, 9, "0,3")])
@pytest.mark.parametrize("n", [20, 37, 70, 88, 96, 160, 230])
@pytest.mark.parametrize("kernel", ["mxf4", "mxf4q", "mxf4w", "mxf4f"])
def test_mxf4_levels(monkeypatch, ctx, k, g, floors, n, kernel):
    """K5 / K5p with forced suffix levels (depth-4/5 tables): exact minima and
    combination counts per Gamma against the oracle (K5p runs at n = 20, 70,
    96; the other widths fall back to K5)."""
    monkeypatch.setenv("BZ_K5_FLOORS", floors)
    rng = random.Random(k * 1000 + g * 10 + n)
    gammas = [[rng.getrandbits(n) for _ in range(k)] for _ in range(2)]
    ctx.set_engine(kernel)
    try:
        ctx.load(family_words([BitMatrix(r, n) for r in gammas], n), n)
        mins, combos = ctx.round(g, -1, 1 << 30)
    finally:
        ctx.set_engine("auto")
    for j in range(2):
        want = oracle.min_weight(gammas[j], n, g)[0]
        assert mins[j] == want, (j, mins, want)
        assert combos[j] == comb(k, g)


@pytest.mark.parametrize("name,seed,mask", [("cfg1", 2, 0b11), ("cfg2", 1, 0b11),
                                            ("cfg3", 1, 0b111), ("cfg3", 2, 0b111)])
def test_identity_elision(ctx, name, seed, mask):
    """Gammas with a unit column per row are stored without those columns
    (+g on every weight).  That includes cfg3's remainder: k_m counts its new
    pivots, but like every Gamma it spans the full row space and keeps the
    earlier pivots' unit columns.  The whole BZ run is identical with
    elision on and off, for every engine."""
    G, gs, _ = code(name, seed)
    reports = {}
    for elide in (True, False):
        for eng in ("auto", "mxf4", "popc"):
            rep = minimum_distance(G, EngineConfig(engine=eng, elide_identity=elide))
            if elide:
                assert ctx.elided() == mask
            reports[(elide, eng)] = (rep.distance, tuple(map(tuple, rep.bounds_trace)),
                                     rep.counters.combinations)
    assert len(set(reports.values())) == 1, reports
    _native.context(0).set_elision(True)


def test_identity_elision_systematic_histogram(ctx):
    """[I | A] (cfg4's generator): elided min and histogram equal the
    un-elided ones, bin for bin (the histogram is shifted by g)."""
    gm = microbench_gamma(3)  # random_systematic_matrix(64, 192, 3)
    out = {}
    for elide in (True, False):
        ctx.set_elision(elide)
        words = family_words([gm], gm.num_cols)
        ctx.load(words, gm.num_cols)
        assert ctx.elided() == (1 if elide else 0)
        for g in (3, 4):
            hist, mn, c = ctx.histogram(0, g)
            out[(elide, g)] = (list(hist), mn, c)
    ctx.set_elision(True)
    for g in (3, 4):
        assert out[(True, g)] == out[(False, g)]
        assert out[(True, g)][1] == min(i for i, v in enumerate(out[(True, g)][0]) if v)


def test_brute_force_goldens(goldens):
    """GPU brute force (bz_brute_force) against the reference's
    brute_force_distance on every golden code that has one."""
    from paper_1603_06757_b200 import brute_force_distance

    n_checked = 0
    for fx in goldens["small"]["codes"]:
        if "brute" in fx:
            M = BitMatrix(hexrows(fx["rows"]), fx["n"])
            assert brute_force_distance(M) == fx["brute"], fx["src"]
            n_checked += 1
    for fx in goldens["configs"]:
        if fx["name"] == "cfg1":
            M = BitMatrix(hexrows(fx["rows"]), fx["n"])
            assert brute_force_distance(M) == fx["distance"]
            n_checked += 1
    assert n_checked >= 3


@pytest.mark.parametrize("k,n", [(1, 5), (7, 31), (12, 33), (20, 100), (29, 64), (30, 256)])
def test_brute_force_vs_oracle(k, n):
    """Word widths 1..8; k = 29, 30 are beyond the reference's default cap
    (max_k raised), checked against the C oracle's Gray walk."""
    from paper_1603_06757_b200 import brute_force_distance

    rng = random.Random(k * 1000 + n)
    rows = [rng.getrandbits(n) for _ in range(k)]
    M = BitMatrix(rows, n)
    want = oracle.brute_distance(rows, n)
    assert brute_force_distance(M, max_k=40) == want
    if k > 28:
        with pytest.raises(TooLarge):
            brute_force_distance(M)


def test_brute_force_rank_deficient():
    from paper_1603_06757_b200 import brute_force_distance

    M = BitMatrix([0b1011, 0b0110, 0b1101], 4)  # row 3 = row 1 ^ row 2
    assert brute_force_distance(M) == 0


@pytest.mark.parametrize("n", [1, 17, 32, 33, 64, 80, 95, 96, 110, 111, 120, 127, 128])
@pytest.mark.parametrize("density", [0.05, 0.5, 0.97])
def test_k5q_weight_range(ctx, n, density):
    """K5q packs two codewords as bytes x = wt + 128 - thr of one fp32
    accumulator: every stored weight from 0 to n <= 127 must come back exact,
    including all-zero and all-one codewords, dense rows (prefix weights up
    to 128), slices crossing the 480-row tile and both parts of a column."""
    rng = random.Random(n * 100 + int(density * 100))
    k = 24
    rows = [sum(1 << b for b in range(n) if rng.random() < density) for _ in range(k)]
    rows[3] = rows[4]                      # a zero codeword at every even g >= 2
    rows[5] = (1 << n) - 1                 # an all-ones row
    ctx.set_engine("mxf4q")
    try:
        ctx.load(family_words([BitMatrix(rows, n), BitMatrix(rows[::-1], n)], n), n)
        for g in (4, 5, 6, 7):
            want = oracle.min_weight(rows, n, g)[0]
            for upper in (1 << 30, want + 1, want, max(want - 2, 0)):
                mins, combos = ctx.round(g, -1, upper)
                assert mins == [min(want, upper)] * 2 and combos == [comb(k, g)] * 2, \
                    (g, upper, mins, want)
    finally:
        ctx.set_engine("auto")


@pytest.mark.parametrize("n", [40, 96, 111, 127, 128])
def test_k5q_all_heavy(ctx, n):
    """Every codeword heavy (odd g over identical all-ones rows: weight n),
    so the minimum is the largest value a byte field carries -- up to a
    stored weight of 128 with no bound (the start bound is capped at the
    stored columns, so the threshold stays <= 128)."""
    k = 15
    rows = [(1 << n) - 1] * k
    ctx.set_engine("mxf4q")
    try:
        ctx.load(family_words([BitMatrix(rows, n)], n), n)
        for g in (5, 7, 9):
            mins, _ = ctx.round(g, -1, 1 << 30)
            assert mins == [n], (g, mins)
            mn, c = ctx.enumerate(0, g)
            assert (mn, c) == (n, comb(k, g)), (g, mn, c)
        for g in (4, 6):
            mins, _ = ctx.round(g, -1, 1 << 30)
            assert mins == [0], (g, mins)
    finally:
        ctx.set_engine("auto")


def test_k5q_dense_prefix_small_bound(ctx):
    """A prefix of stored weight 127 (an all-ones row) under a small bound:
    the offset x = wt + 128 - thr would pass 238, past what an e2m1 offset
    block encodes, unless the producer raises its threshold (k5q_threshold).
    The bound must come back unchanged (no codeword is that light) and the
    unbounded pass must give the oracle minimum."""
    rng = random.Random(2024)
    n, k = 127, 20
    rows = [rng.getrandbits(n) for _ in range(k)]
    rows[0] = (1 << n) - 1
    want = oracle.min_weight(rows, n, 4)[0]
    ctx.set_engine("mxf4q")
    try:
        ctx.load(family_words([BitMatrix(rows, n)], n), n)
        for upper in (0, 1, 5, 16, 17, want, want + 1):
            mins, combos = ctx.round(4, -1, upper)
            assert mins == [min(upper, want)] and combos == [comb(k, 4)], (upper, mins, want)
        mins, _ = ctx.round(4, -1, 1 << 30)
        assert mins == [want]
    finally:
        ctx.set_engine("auto")


def _dense_systematic(k: int, seed: int, light: int, r: int | None = None):
    """[I_k | A] with A (k x r, r = k by default) random, A's row 0 all ones
    (stored weight r in Gamma_1) and row 1 of weight `light` - 1 (a planted
    codeword of weight `light`); at least two full information sets (exactly
    two, no remainder, when r = k)."""
    rng = random.Random(seed)
    r = k if r is None else r
    n = k + r
    while True:
        A = [rng.getrandbits(r) for _ in range(k)]
        A[0] = (1 << r) - 1
        A[1] = sum(1 << b for b in rng.sample(range(r), light - 1))
        rows = [(1 << i) | (a << k) for i, a in enumerate(A)]
        try:
            from paper_1603_06757_b200.gf2 import build_gamma_set

            gs = build_gamma_set(BitMatrix(rows, n))
        except Exception:
            continue
        if gs.full_rank_count == 2 and (gs.remainder_rank == 0 or r > k):
            return rows, n


def test_k5q_dense_row_minimum_distance():
    """BZ on a code whose Gammas keep 127 stored columns, with a dense row
    and a planted light codeword (U = 12 after round 1, so round 4 runs with
    thr = U - g = 8 against a prefix of stored weight 127): distance, trace,
    status and counts equal the C oracle's, K5q forced for every g >= 4."""
    rows, n = _dense_systematic(127, 11, 12)
    want = oracle.minimum_distance(rows, n, max_g=4)
    rep = minimum_distance(BitMatrix(rows, n), EngineConfig(engine="mxf4q", max_g=4))
    assert rep.bounds_trace == [tuple(t) for t in want["bounds_trace"]]
    assert rep.distance == want["distance"] == 12
    assert rep.counters.combinations == want["combinations"]
    assert _native.context(0).elided() == 0b11  # both Gammas store n - k = 127 columns


@pytest.mark.parametrize("n", [129, 160, 185, 192, 193, 224, 255, 256])
@pytest.mark.parametrize("density", [0.05, 0.5, 0.97])
def test_k5w_weight_range(ctx, n, density):
    """K5w packs two codewords as 11-bit fields x = w + 1024 - thr of one
    fp32 accumulator (rows wider than K5q's 128 stored columns): every stored
    weight from 0 to 256 must come back exact -- zero codewords, all-one rows,
    dense prefixes (R = w(P) - thr up to 450 in the offset chunk), slices
    crossing the 480-row tile and both parts of a column -- under loose,
    exact and too-tight bounds."""
    rng = random.Random(n * 100 + int(density * 100))
    k = 22
    rows = [sum(1 << b for b in range(n) if rng.random() < density) for _ in range(k)]
    rows[3] = rows[4]                      # a zero codeword at every even g >= 2
    rows[5] = (1 << n) - 1                 # an all-ones row
    ctx.set_engine("mxf4w")
    try:
        ctx.load(family_words([BitMatrix(rows, n), BitMatrix(rows[::-1], n)], n), n)
        for g in (4, 5, 6, 7):
            want = oracle.min_weight(rows, n, g)[0]
            for upper in (1 << 30, want + 1, want, max(want - 2, 0)):
                mins, combos = ctx.round(g, -1, upper)
                assert mins == [min(want, upper)] * 2 and combos == [comb(k, g)] * 2, \
                    (g, upper, mins, want)
    finally:
        ctx.set_engine("auto")


@pytest.mark.parametrize("n", [150, 200, 256])
def test_k5w_all_heavy(ctx, n):
    """Odd g over identical all-ones rows: every codeword has stored weight
    n (up to 256, the widest field value); even g: weight 0."""
    k = 15
    rows = [(1 << n) - 1] * k
    ctx.set_engine("mxf4w")
    try:
        ctx.load(family_words([BitMatrix(rows, n)], n), n)
        for g in (5, 7, 9):
            mins, _ = ctx.round(g, -1, 1 << 30)
            assert mins == [n], (g, mins)
            mn, c = ctx.enumerate(0, g)
            assert (mn, c) == (n, comb(k, g)), (g, mn, c)
        for g in (4, 6):
            mins, _ = ctx.round(g, -1, 1 << 30)
            assert mins == [0], (g, mins)
    finally:
        ctx.set_engine("auto")


@pytest.mark.parametrize("engine_name", ["auto", "mxf4w"])
def test_k5w_dense_row_minimum_distance(engine_name):
    """BZ on a [280, 100] code whose Gammas keep 180 stored columns (AUTO
    runs K5 there, mxf4w forces K5w for g >= 4; two full information sets and
    a remainder), with an all-ones row and a planted light codeword: trace,
    distance and counts equal the C oracle's."""
    rows, n = _dense_systematic(100, 13, 14, r=180)
    want = oracle.minimum_distance(rows, n, max_g=4)
    rep = minimum_distance(BitMatrix(rows, n), EngineConfig(engine=engine_name, max_g=4))
    assert rep.bounds_trace == [tuple(t) for t in want["bounds_trace"]]
    assert rep.distance == want["distance"] == 14
    assert rep.counters.combinations == want["combinations"]


@pytest.mark.parametrize("engine_name", ["auto", "mxf4", "popc"])
def test_batched_rounds_chain_u(ctx, engine_name):
    """bz_rounds: round g0 starts from `upper`, each later round from the U
    its predecessor ended with -- exactly the per-round calls with the
    running U (no early exit here: lower_prev = 0)."""
    G, gs, _ = code("cfg2", 1)
    ctx.set_engine(engine_name)
    try:
        ctx.load(family_words(gs.gammas, 96), 96)
        res = ctx.rounds(1, [0] * 6, 10**6)
        U = 10**6
        for i, (mins, combos) in enumerate(res):
            want_min, want_c = ctx.round(1 + i, 0, U)
            assert (mins, combos) == (want_min, want_c), (1 + i, mins, want_min)
            U = min([U] + mins)
    finally:
        ctx.set_engine("auto")


def test_batched_rounds_past_termination_exit(ctx):
    """A batch that runs ahead of termination: the rounds after the one
    where L >= U start from (or, launched as programmatic dependents, watch)
    the predecessor's U, find it already <= their L_prev and stop at once,
    while the rounds up to termination are exact."""
    G, gs, _ = code("cfg2", 1)  # trace (1,4,16) (2,6,15) (3,8,12) (4,10,12) (5,12,11)
    ctx.set_engine("auto")
    ctx.load(family_words(gs.gammas, 96), 96)
    k, m = 48, 2
    lps = [0] + [2 * (g + 1) for g in range(1, 8)]  # L after round g (m = 2 full sets)
    res = ctx.rounds(1, lps, 10**6)
    U = 10**6
    for g, (mins, combos) in enumerate(res[:5], start=1):
        U = min([U] + mins)
        assert combos == [comb(k, g)] * m or U <= lps[g - 1], (g, combos)
    assert U == 11
    for g, (mins, combos) in enumerate(res[5:], start=6):
        assert min(mins) <= 11
        assert sum(combos) < 0.05 * m * comb(k, g), (g, combos)

"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference package itself (tests/golden/make_golden.py) and against the
reference's own known answers.  CPU only."""

from __future__ import annotations

import hashlib
import itertools
from math import comb

import numpy as np
import pytest

from conftest import CFG4_HIST_SHA256, hexrows
from oracle import oracle


def fold_min(rows, g):
    best = None
    for c in itertools.combinations(range(len(rows)), g):
        acc = 0
        for i in c:
            acc ^= rows[i]
        w = acc.bit_count()
        best = w if best is None or w < best else best
    return best


def test_small_enum_fixtures(goldens):
    """Per-(matrix, g) minima of the reference's test matrices
    (t/test_enumeration.py:65-76, :285-302)."""
    for fx in goldens["small"]["enum"]:
        rows = hexrows(fx["rows"])
        for g, expect in enumerate(fx["min_by_g"], start=1):
            mn, combos = oracle.min_weight(rows, fx["n"], g, threads=2)
            assert mn == expect, (fx["src"], g)
            assert combos == comb(fx["k"], g)


def test_fold_restatement_agrees():
    """The C walk against a direct fold (t/test_enumeration.py:31-40)."""
    import random

    rng = random.Random(5)
    for _ in range(20):
        k = rng.randint(2, 11)
        n = rng.randint(k, 140)
        rows = [rng.getrandbits(n) for _ in range(k)]
        for g in range(1, k + 1):
            assert oracle.min_weight(rows, n, g, threads=3)[0] == fold_min(rows, g)


def test_codes_and_known_answers(goldens):
    """Full BZ loop on the reference's engine-test codes: distance, status,
    g_reached, m, k_m and the (g, L, U) trace (t/test_engine.py:88-152)."""
    for fx in goldens["small"]["codes"]:
        rows = hexrows(fx["rows"])
        rep = oracle.minimum_distance(rows, fx["n"], threads=2)
        assert rep["distance"] == fx["distance"] == fx["brute"], fx["src"]
        assert rep["bounds_trace"] == [tuple(t) for t in fx["bounds_trace"]], fx["src"]
        assert (rep["m"], rep["k_m"], rep["g_reached"], rep["status"]) == \
            (fx["m"], fx["k_m"], fx["g_reached"], fx["status"]), fx["src"]
        if fx["k"] <= 20:
            assert oracle.brute_distance(rows, fx["n"]) == fx["brute"]


@pytest.mark.parametrize("idx", range(6))
def test_configs_1_to_3(goldens, idx):
    fx = goldens["configs"][idx]
    rows = hexrows(fx["rows"])
    rep = oracle.minimum_distance(rows, fx["n"])
    for key in ("distance", "status", "g_reached", "m", "k_m", "combinations"):
        assert rep[key] == fx[key], (fx["name"], fx["seed"], key)
    assert rep["bounds_trace"] == [tuple(t) for t in fx["bounds_trace"]]
    assert rep["pivot_sets"] == fx["pivot_sets"]


def test_gamma_family_matches_reference(goldens):
    for fx in goldens["configs"]:
        gammas, piv, full, rem = oracle.gamma_family(hexrows(fx["rows"]), fx["n"])
        assert [[format(r, "x") for r in gm] for gm in gammas] == fx["gammas"]
        assert [list(p) for p in piv] == fx["pivot_sets"]


def test_cfg1_brute_force(goldens):
    for fx in goldens["configs"]:
        if fx["name"] == "cfg1":
            assert oracle.brute_distance(hexrows(fx["rows"]), fx["n"]) == fx["distance"]


def test_cfg4_min_and_histogram(goldens):
    fx = goldens["cfg4"]
    rows = hexrows(fx["rows"])
    hist = oracle.histogram(rows, fx["n"], fx["g"])
    assert int(hist.sum()) == comb(64, 6) == fx["combinations"]
    nz = np.flatnonzero(hist)
    assert int(nz[0]) == fx["min_weight"] == 39
    assert hashlib.sha256(hist.astype("<u8").tobytes()).hexdigest() == CFG4_HIST_SHA256
    assert oracle.min_weight(rows, fx["n"], fx["g"])[0] == fx["min_weight"]


def test_cfg5_rounds_up_to_6(cfg5_golden):
    """Rounds g <= 6 of the reference's cfg5 seed-7 trace (the full run is
    6.5e10 combinations; the GPU tests check all of it)."""
    fx = cfg5_golden
    rep = oracle.minimum_distance(hexrows(fx["rows"]), fx["n"], max_g=6)
    assert rep["bounds_trace"] == [tuple(t) for t in fx["bounds_trace"][:6]]


@pytest.mark.parametrize("name,seed", [("cfg1", 1), ("cfg1", 2), ("cfg2", 2), ("cfg3", 1),
                                       ("cfg5", 7)])
def test_oracle_draw_matches_configs(name, seed):
    """bench.py's CPU arm draws its matrix through oracle.draw_code (no
    product import): the rows equal the product's configs.code draw."""
    from paper_1603_06757_b200.configs import CONFIGS, code

    c = CONFIGS[name]
    G, _, _ = code(name, seed)
    assert oracle.draw_code(c.k, c.n, seed, c.target) == list(G.rows)

"""The boundary tested from the reference's side: the unmodified reference
package (baseline/_ref, installed from the reference's pkg/) with the
"gpu" strategy of paper_1603_06757_b200/reference_plugin.py installed --
STRATEGIES (m/engine.py:29) plus the _Runner.run seam (m/engine.py:136-150)
bound to libbz.so by ctypes.  The reference's own engine loop then drives
the device.

The GPU cases restate the reference's strategy-parametrised engine tests
(t/test_engine.py:88-227: repetition and Hamming codes, the full-space
shortcut, rank-deficient input, strategies vs brute force, the bounds-trace
discipline, two information sets, max_g, the running U within a round,
interrupt + resume, terminal resume, the report round trip) with
strategy="gpu", and compare whole DistanceReports with the reference's own
"saved" strategy and with the goldens of configs 1-3."""

from __future__ import annotations

import os
import sys

import pytest

from conftest import hexrows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

if not os.path.isdir(os.path.join(REF, "mindist")):
    pytest.skip("baseline/_ref (the installed reference package) is missing",
                allow_module_level=True)
if REF not in sys.path:
    sys.path.insert(0, REF)

from mindist import engine as ref_engine  # noqa: E402
from mindist import errors as ref_errors  # noqa: E402
from mindist.gf2 import BitMatrix as RefMatrix  # noqa: E402
from mindist.gf2 import random_systematic_matrix  # noqa: E402

from paper_1603_06757_b200 import reference_plugin  # noqa: E402

PASSES = reference_plugin.install(ref_engine)
EngineConfig = ref_engine.EngineConfig
minimum_distance = ref_engine.minimum_distance


def _gpu(**kw):
    return EngineConfig(strategy="gpu", **kw)


def test_install_is_idempotent_and_keeps_reference_strategies():
    again = reference_plugin.install(ref_engine)
    assert again is PASSES
    assert ref_engine.STRATEGIES.count("gpu") == 1
    assert ref_engine.STRATEGIES[:5] == ("basic", "optimized", "stack", "saved",
                                        "saved-unrolled")
    # the reference's own strategies still run the reference code (CPU)
    M = random_systematic_matrix(6, 15, seed=3)
    rep = minimum_distance(M, EngineConfig(strategy="stack"))
    assert rep.distance == ref_engine.brute_force_distance(M)


def test_unknown_strategy_still_rejected():
    with pytest.raises(ref_errors.InvalidArity):
        minimum_distance(RefMatrix([1, 2], 3), EngineConfig(strategy="gpu2"))


def test_no_cpu_fallback_without_device():
    """Off a GPU box the strategy fails loudly with the reference's own
    MindistError -- it never drops back to a CPU enumeration."""
    if PASSES.lib.bz_device_count() > 0:
        pytest.skip("a device is visible")
    with pytest.raises(ref_errors.MindistError):
        minimum_distance(RefMatrix([0b111, 0b1010], 4), _gpu())


# --------------------------------------------------------------------------- GPU

gpu = pytest.mark.gpu


def _launches():
    import ctypes
    total = 0
    for ctx, _ in PASSES.ctxs.values():
        c = ctypes.c_uint64()
        PASSES.lib.bz_launch_count(ctx, ctypes.byref(c))
        total += c.value
    return total


@gpu
def test_repetition_and_hamming():
    rep = minimum_distance(RefMatrix([0b11111], 5), _gpu())
    assert rep.distance == 5 and rep.exact
    H = RefMatrix.from_bits([[1, 0, 0, 0, 1, 1, 0], [0, 1, 0, 0, 1, 0, 1],
                             [0, 0, 1, 0, 0, 1, 1], [0, 0, 0, 1, 1, 1, 1]])
    rep = minimum_distance(H, _gpu())
    assert rep.distance == 3 and rep.exact and rep.m == 2 and rep.k_m == 3
    text = ref_engine.format_report(rep)
    parsed = ref_engine.parse_report(text)
    assert parsed["distance"] == 3 and parsed["bounds_trace"] == rep.bounds_trace
    assert parsed["combinations"] == rep.counters.combinations
    # the device's row counters ride along (one addition per codeword at
    # least; rows are loaded once for many codewords)
    assert rep.counters.row_additions >= rep.counters.combinations > 0
    assert rep.counters.row_accesses > 0


@gpu
def test_full_space_and_rank_deficient():
    rep = minimum_distance(RefMatrix([1, 2, 4, 8], 4), _gpu())
    assert rep.distance == 1 and rep.g_reached == 0 and rep.bounds_trace == []
    with pytest.raises(ref_errors.RankDeficient):
        minimum_distance(RefMatrix.from_bits([[1, 1, 0], [1, 1, 0]]), _gpu())


@gpu
def test_gpu_matches_brute_force():
    before = _launches()
    for seed in range(5):
        M = random_systematic_matrix(5 + seed, 13 + 3 * seed, seed=40 + seed)
        rep = minimum_distance(M, _gpu())
        assert rep.distance == ref_engine.brute_force_distance(M), seed
        assert rep.exact
    assert _launches() > before  # the passes ran on the device


@gpu
def test_bounds_trace_discipline_and_two_sets():
    M = random_systematic_matrix(9, 28, seed=5)
    rep = minimum_distance(M, _gpu())
    ls = [L for _, L, _ in rep.bounds_trace]
    us = [U for _, _, U in rep.bounds_trace]
    assert ls == sorted(ls) and len(set(ls)) == len(ls)
    assert us == sorted(us, reverse=True) and rep.distance == us[-1]
    g_final, L_final, U_final = rep.bounds_trace[-1]
    assert L_final >= U_final or g_final == M.num_rows
    M = random_systematic_matrix(4, 14, seed=11)
    d = ref_engine.brute_force_distance(M)
    rep = minimum_distance(M, _gpu())
    assert rep.distance == d and rep.g_reached < d - 1


@gpu
def test_max_g_upper_bound_only():
    M = random_systematic_matrix(14, 30, seed=29)
    full = minimum_distance(M, _gpu())
    assert full.g_reached >= 2
    rep = minimum_distance(M, _gpu(max_g=1))
    assert rep.status == ref_engine.STATUS_UPPER_BOUND_ONLY and not rep.exact
    assert rep.distance >= ref_engine.brute_force_distance(M)


@gpu
def test_running_upper_bound_within_round(monkeypatch):
    M = random_systematic_matrix(5, 15, seed=8)
    seen = []
    real = PASSES.run

    def spy(idx, gamma, g, ubound):
        seen.append(ubound)
        return real(idx, gamma, g, ubound)

    monkeypatch.setattr(PASSES, "run", spy)
    rep = minimum_distance(M, _gpu())
    assert rep.m >= 2 and seen
    for i in range(1, len(seen)):
        if i % rep.m:
            assert seen[i] <= seen[i - 1]


@gpu
def test_interrupt_and_resume(monkeypatch):
    M = random_systematic_matrix(8, 26, seed=9)
    expected = ref_engine.brute_force_distance(M)
    real = PASSES.run

    def bomb(idx, gamma, g, ubound):
        if g == 2:
            raise KeyboardInterrupt
        return real(idx, gamma, g, ubound)

    monkeypatch.setattr(PASSES, "run", bomb)
    with pytest.raises(ref_errors.Interrupted) as exc:
        minimum_distance(M, _gpu())
    partial = exc.value.report
    assert partial.status == ref_engine.STATUS_INTERRUPTED and partial.g_reached == 1
    monkeypatch.setattr(PASSES, "run", real)
    resumed = minimum_distance(M, _gpu(start_g=partial.g_reached + 1,
                                       start_upper=partial.distance))
    assert resumed.distance == expected and resumed.exact
    again = minimum_distance(M, _gpu(start_g=resumed.g_reached + 1,
                                     start_upper=resumed.distance))
    assert again.distance == resumed.distance and again.counters.combinations == 0


def _same_report(a, b):
    assert (a.distance, a.status, a.g_reached, a.m, a.k_m) == \
        (b.distance, b.status, b.g_reached, b.m, b.k_m)
    assert a.pivot_sets == b.pivot_sets
    assert a.bounds_trace == b.bounds_trace
    assert a.counters.combinations == b.counters.combinations


@gpu
@pytest.mark.parametrize("k,n,seed", [(6, 20, 1), (10, 30, 77), (12, 40, 3), (16, 44, 5),
                                      (20, 60, 2), (33, 70, 4)])
def test_gpu_report_equals_reference_saved(k, n, seed):
    """Whole reports: the gpu strategy and the reference's own default
    strategy (saved, s=3) on the same seeded systematic codes."""
    M = random_systematic_matrix(k, n, seed=seed)
    _same_report(minimum_distance(M, _gpu()), minimum_distance(M, EngineConfig()))


@gpu
def test_configs_1_to_3_against_goldens(goldens):
    """BASELINE configs 1-3 (two seeds each) through the reference's loop
    with the gpu strategy: distance, status, trace, pivots and the
    combination count the reference recorded."""
    for c in goldens["configs"]:
        if c["name"] not in ("cfg1", "cfg2", "cfg3"):
            continue
        M = RefMatrix(hexrows(c["rows"]), c["n"])
        rep = minimum_distance(M, _gpu())
        assert rep.distance == c["distance"], c["name"]
        assert rep.status == c["status"] and rep.g_reached == c["g_reached"]
        assert [list(t) for t in rep.bounds_trace] == c["bounds_trace"]
        assert [list(p) for p in rep.pivot_sets] == c["pivot_sets"]
        assert (rep.m, rep.k_m) == (c["m"], c["k_m"])
        assert rep.counters.combinations == c["combinations"]

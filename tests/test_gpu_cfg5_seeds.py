"""Config 5 at scale: eight random [160,80] codes (seeds 1..8).

The reference's own traces for rounds g <= 6 (tests/golden/cfg5_traces.json,
tests/golden/make_cfg5_traces.py) pin the GPU path on every seed: the same
generator matrix and pivot sets, the same (g, L, U) trace, status and
combination count.  The full runs to d (g = 8 or 9, up to 5e11
combinations, beyond what the reference can run here) must then agree
across kernel families and stop only when L >= U.
"""

from __future__ import annotations

import pytest

from conftest import hexrows
from paper_1603_06757_b200 import EngineConfig, minimum_distance
from paper_1603_06757_b200.configs import code

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine", ["auto", "mxf4", "popc"])
def test_cfg5_seed_traces_vs_reference(cfg5_traces, engine):
    for fx in cfg5_traces:
        G, gs, draws = code("cfg5", fx["seed"])
        assert [format(r, "x") for r in G.rows] == fx["rows"], fx["seed"]
        assert draws == fx["draws"]
        assert [list(p) for p in gs.pivot_sets] == fx["pivot_sets"]
        rep = minimum_distance(G, EngineConfig(engine=engine, max_g=fx["max_g"]))
        assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]], fx["seed"]
        assert (rep.status, rep.distance, rep.g_reached) == \
            (fx["status"], fx["upper"], fx["g_reached"]), fx["seed"]
        assert rep.counters.combinations == fx["combinations"], fx["seed"]


def test_cfg5_seeds_full_runs(cfg5_traces):
    """Every seed to its exact distance with K5q and K5: identical traces,
    the reference's prefix, termination exactly when L >= U."""
    for fx in cfg5_traces:
        G, _, _ = code("cfg5", fx["seed"])
        reps = [minimum_distance(G, EngineConfig(engine=e)) for e in ("auto", "mxf4")]
        assert reps[0].bounds_trace == reps[1].bounds_trace, fx["seed"]
        assert reps[0].counters.combinations == reps[1].counters.combinations
        rep = reps[0]
        prefix = [tuple(t) for t in fx["bounds_trace"]]
        assert rep.bounds_trace[:len(prefix)] == prefix, fx["seed"]
        g, L, U = rep.bounds_trace[-1]
        assert rep.status == "exact" and L >= U == rep.distance
        assert all(l < u for (_, l, u) in rep.bounds_trace[:-1])
        print(f"seed {fx['seed']}: d = {rep.distance} at g = {g}, "
              f"{rep.counters.combinations} combinations")

"""Host layer of the package on CPU: GF(2) family construction, bounds,
report format, and the engine loop driven through the backend seam with
the oracle standing in for the device (the reference tests swap strategy
functions the same way, t/test_engine.py:165-208)."""

from __future__ import annotations

import pytest

from conftest import hexrows
from oracle import oracle
from paper_1603_06757_b200 import (BitMatrix, EngineConfig, Interrupted, InvalidArity,
                                   InvalidDimensions, MatrixFormatError, RankDeficient,
                                   build_gamma_set, engine, format_matrix_text,
                                   format_report, initial_bounds, lower_bound_update,
                                   minimum_distance, parse_matrix_text, parse_report,
                                   random_systematic_matrix)
from paper_1603_06757_b200.configs import CONFIGS, code


class OracleRounds:
    """Test double for engine.GpuRounds backed by the C oracle."""

    calls: list = []

    def __init__(self, config, comm):
        self.comm = comm

    def load(self, gs, n):
        self.gammas = [list(gm.rows) for gm in gs.gammas]
        self.n = n

    def run(self, g, lower_prev, upper):
        OracleRounds.calls.append((g, lower_prev, upper))
        res = [oracle.min_weight(rows, self.n, g, threads=2) for rows in self.gammas]
        mins = [min(mn, upper) for mn, _ in res]
        return mins, [c for _, c in res], 0.0


@pytest.fixture
def oracle_backend(monkeypatch):
    OracleRounds.calls = []
    monkeypatch.setattr(engine, "make_backend", lambda cfg, comm: OracleRounds(cfg, comm))
    return OracleRounds


def test_gamma_family_matches_reference(goldens):
    for fx in goldens["configs"]:
        G = BitMatrix(hexrows(fx["rows"]), fx["n"])
        gs = build_gamma_set(G)
        assert [[format(r, "x") for r in gm.rows] for gm in gs.gammas] == fx["gammas"]
        assert [list(p) for p in gs.pivot_sets] == fx["pivot_sets"]
        assert gs.matrix_count == fx["m"] and gs.remainder_rank == fx["k_m"]


def test_config_generator_matches_goldens(goldens):
    for fx in goldens["configs"]:
        G, gs, draws = code(fx["name"], fx["seed"])
        assert [format(r, "x") for r in G.rows] == fx["rows"]
        assert draws == fx["draws"]


def test_random_systematic_matches_reference(goldens):
    fx = goldens["cfg4"]
    assert [format(r, "x") for r in random_systematic_matrix(64, 192, 1).rows] == fx["rows"]
    for e in goldens["small"]["enum"]:
        if e["src"].startswith("random_systematic_matrix"):
            k, n, seed = (int(v) for v in e["src"].split("(")[1].rstrip(")").split(","))
            assert [format(r, "x") for r in random_systematic_matrix(k, n, seed).rows] == e["rows"]


def test_bounds_examples():
    assert initial_bounds(150, 50) == engine.Bounds(1, 101)
    assert initial_bounds(6, 6) == engine.Bounds(1, 1)
    with pytest.raises(InvalidDimensions):
        initial_bounds(4, 5)
    assert lower_bound_update(1, 3, 50, 10) == 4
    assert lower_bound_update(2, 1, 9, 9) == 3
    assert lower_bound_update(5, 2, 50, 0) == 6


def test_rank_deficient_and_bad_rows():
    with pytest.raises(RankDeficient):
        minimum_distance(BitMatrix.from_bits([[1, 1, 0], [1, 1, 0]]))
    with pytest.raises(InvalidDimensions):
        BitMatrix([0b1000], 3)
    with pytest.raises(InvalidArity):
        minimum_distance(random_systematic_matrix(4, 9, 1), EngineConfig(strategy="saved"))


def test_matrix_text_roundtrip():
    M = random_systematic_matrix(7, 19, 3)
    assert parse_matrix_text(format_matrix_text(M, ["c"])) == M
    with pytest.raises(MatrixFormatError):
        parse_matrix_text("2 3\n101\n")


def test_full_space_terminates_immediately(oracle_backend):
    rep = minimum_distance(BitMatrix([1, 2, 4, 8], 4))
    assert rep.distance == 1 and rep.exact and rep.g_reached == 0 and rep.bounds_trace == []
    assert oracle_backend.calls == []


@pytest.mark.parametrize("idx", range(6))
def test_engine_loop_configs(goldens, oracle_backend, idx):
    fx = goldens["configs"][idx]
    rep = minimum_distance(BitMatrix(hexrows(fx["rows"]), fx["n"]))
    assert rep.distance == fx["distance"]
    assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]]
    assert (rep.status, rep.g_reached, rep.m, rep.k_m) == \
        (fx["status"], fx["g_reached"], fx["m"], fx["k_m"])
    assert rep.counters.combinations == fx["combinations"]
    # the previous round's L is the early-exit threshold handed to the device
    Ls = [1] + [t[1] for t in fx["bounds_trace"]]
    assert [c[1] for c in oracle_backend.calls] == Ls[:len(oracle_backend.calls)]


def test_engine_small_codes(goldens, oracle_backend):
    for fx in goldens["small"]["codes"]:
        rep = minimum_distance(BitMatrix(hexrows(fx["rows"]), fx["n"]))
        assert rep.distance == fx["distance"], fx["src"]
        assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]], fx["src"]


def test_max_g_and_resume(oracle_backend):
    M = random_systematic_matrix(14, 30, 29)
    full = minimum_distance(M)
    rep = minimum_distance(M, EngineConfig(max_g=1))
    assert rep.status == "upper_bound_only" and not rep.exact
    again = minimum_distance(M, EngineConfig(start_g=rep.g_reached + 1,
                                             start_upper=rep.distance))
    assert again.distance == full.distance


def test_interrupt_and_resume(monkeypatch):
    M = random_systematic_matrix(8, 26, 9)

    class Bomb(OracleRounds):
        def run(self, g, lower_prev, upper):
            if g == 2:
                raise KeyboardInterrupt
            return super().run(g, lower_prev, upper)

    monkeypatch.setattr(engine, "make_backend", lambda cfg, comm: Bomb(cfg, comm))
    with pytest.raises(Interrupted) as exc:
        minimum_distance(M)
    part = exc.value.report
    assert part.status == "interrupted" and part.g_reached == 1
    monkeypatch.setattr(engine, "make_backend", lambda cfg, comm: OracleRounds(cfg, comm))
    rep = minimum_distance(M, EngineConfig(start_g=2, start_upper=part.distance))
    assert rep.distance == oracle.brute_distance(list(M.rows), M.num_cols)


def test_report_roundtrip(oracle_backend):
    H = BitMatrix.from_bits([[1, 0, 0, 0, 1, 1, 0], [0, 1, 0, 0, 1, 0, 1],
                             [0, 0, 1, 0, 0, 1, 1], [0, 0, 0, 1, 1, 1, 1]])
    rep = minimum_distance(H)
    assert rep.distance == 3 and rep.m == 2 and rep.k_m == 3
    parsed = parse_report(format_report(rep))
    assert parsed["distance"] == 3 and parsed["bounds_trace"] == rep.bounds_trace
    assert parsed["combinations"] == rep.counters.combinations


def test_configs_table():
    assert CONFIGS["cfg5"].k == 80 and CONFIGS["cfg5"].n == 160


class OracleBatchRounds(OracleRounds):
    """Adds the batched-rounds seam (GpuRounds.run_batch) on the oracle."""

    batches: list = []

    def run_batch(self, g0, lower_prevs, upper):
        """Mirrors bz_rounds: round i > 0 starts from the U round i-1 ended
        with and exits at once when that U already meets its lower_prev
        (a round past termination)."""
        OracleBatchRounds.batches.append((g0, len(lower_prevs)))
        out = []
        U = upper
        for i in range(len(lower_prevs)):
            if i > 0 and U <= lower_prevs[i]:
                out.append(([U] * len(self.gammas), [0] * len(self.gammas)))
                continue
            res = [oracle.min_weight(rows, self.n, g0 + i, threads=2) for rows in self.gammas]
            out.append(([min(mn, U) for mn, _ in res], [c for _, c in res]))
            U = min([U] + out[-1][0])
        return out, 0.0


@pytest.mark.parametrize("idx", range(6))
def test_engine_batched_rounds(goldens, monkeypatch, idx):
    """Rounds batched ahead of the bound check give the reference's trace,
    status and combination count (rounds past termination are dropped)."""
    OracleBatchRounds.batches = []
    monkeypatch.setattr(engine, "make_backend", lambda cfg, comm: OracleBatchRounds(cfg, comm))
    fx = goldens["configs"][idx]
    rep = minimum_distance(BitMatrix(hexrows(fx["rows"]), fx["n"]),
                           EngineConfig(batch_combinations=10**9))
    assert rep.distance == fx["distance"]
    assert rep.bounds_trace == [tuple(t) for t in fx["bounds_trace"]]
    assert rep.counters.combinations == fx["combinations"]
    assert OracleBatchRounds.batches and OracleBatchRounds.batches[0][0] == 1

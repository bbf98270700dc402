"""Generate the committed golden fixtures from the REFERENCE package.

Test infrastructure only.  Runs in the build container, where the
read-only reference lives at /root/reference; it imports the reference's
own `mindist` package (pure Python + numpy) and records its outputs as
JSON.  Nothing on the GPU box reads /root/reference: the tests there use
the JSON written by this script.

    python tests/golden/make_golden.py            # configs 1-4 + small fixtures
    python tests/golden/make_golden.py --cfg5     # cfg5 seed 7 (long: ~45 min)

Input generation follows SURVEY.md Appendix A: `random.Random(seed)`,
`getrandbits(n)` per row (bit j = column j), redraw until
`build_gamma_set` yields the target (full_rank_count, remainder_rank);
cfg4 uses the reference's `random_systematic_matrix(64, 192, seed)`.
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import random
import sys
import time

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from mindist import (  # noqa: E402  (reference package)
    BitMatrix, EngineConfig, brute_force_distance, build_gamma_set,
    build_saved_store, enumerate_basic, enumerate_saved, minimum_distance,
    random_systematic_matrix)
from mindist.errors import RankDeficient  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CONFIGS = {
    "cfg1": dict(k=24, n=48, target=(2, 0), seeds=(1, 2)),
    "cfg2": dict(k=48, n=96, target=(2, 0), seeds=(1, 2)),
    "cfg3": dict(k=40, n=100, target=(2, 20), seeds=(1, 2)),
    "cfg5": dict(k=80, n=160, target=(2, 0), seeds=(7,)),
}


def draw(k, n, seed, target):
    rng = random.Random(seed)
    draws = 0
    while True:
        draws += 1
        rows = [rng.getrandbits(n) for _ in range(k)]
        M = BitMatrix(rows, n)
        try:
            gs = build_gamma_set(M)
        except RankDeficient:
            continue
        if (gs.full_rank_count, gs.remainder_rank) == target:
            return M, gs, draws


def hexrows(M):
    return [format(r, "x") for r in M.rows]


def run_config(name, seed, s=3):
    c = CONFIGS[name]
    M, gs, draws = draw(c["k"], c["n"], seed, c["target"])
    per_round = []
    t_last = [time.perf_counter()]

    def progress(g, L, U):
        now = time.perf_counter()
        per_round.append(dict(g=g, L=L, U=U, seconds=round(now - t_last[0], 3)))
        t_last[0] = now
        print(f"  {name} seed={seed} g={g} L={L} U={U} ({per_round[-1]['seconds']} s)",
              flush=True)

    rep = minimum_distance(M, EngineConfig(strategy="saved", s=s, progress=progress))
    return dict(
        name=name, seed=seed, k=c["k"], n=c["n"], draws=draws, rows=hexrows(M),
        m=rep.m, k_m=rep.k_m, pivot_sets=[list(p) for p in rep.pivot_sets],
        gammas=[hexrows(gm) for gm in gs.gammas],
        distance=rep.distance, status=rep.status, g_reached=rep.g_reached,
        bounds_trace=[list(t) for t in rep.bounds_trace],
        combinations=rep.counters.combinations, elapsed=round(rep.elapsed, 3),
        rounds=per_round, reference_strategy=f"saved s={s}")


def small_fixtures():
    """Per-(matrix, g) minimum weights from the reference's own test
    matrices (t/test_enumeration.py:285-302 sweep, :65-76 known answers,
    t/test_engine.py:113-120 brute-force codes)."""
    out = {"enum": [], "codes": []}
    for seed in range(4):  # test_all_strategies_agree
        rng = random.Random(100 + seed)
        k = rng.randint(4, 12)
        n = rng.randint(k + 1, 34)
        M = random_systematic_matrix(k, n, seed)
        mins = [enumerate_basic(M, g).min_weight for g in range(1, k + 1)]
        out["enum"].append(dict(k=k, n=n, rows=hexrows(M), min_by_g=mins,
                                src=f"random_systematic_matrix({k},{n},{seed})"))
    for (k, n, seed) in [(7, 19, 2), (7, 15, 3), (8, 21, 12), (9, 24, 16),
                         (10, 26, 17), (6, 16, 19), (12, 30, 13)]:
        M = random_systematic_matrix(k, n, seed)
        mins = [enumerate_basic(M, g).min_weight for g in range(1, k + 1)]
        out["enum"].append(dict(k=k, n=n, rows=hexrows(M), min_by_g=mins,
                                src=f"random_systematic_matrix({k},{n},{seed})"))
    # known answers (t/test_enumeration.py:65-76)
    out["enum"].append(dict(k=3, n=3, rows=["1", "2", "4"], min_by_g=[1, 2, 3],
                            src="I3"))
    codes = []
    for seed in range(5):  # t/test_engine.py:113-120
        codes.append((5 + seed, 13 + 3 * seed, 40 + seed))
    codes += [(10, 30, 77), (9, 28, 5), (4, 14, 11), (14, 30, 29), (8, 26, 9),
              (7, 21, 10)]
    for (k, n, seed) in codes:
        M = random_systematic_matrix(k, n, seed)
        rep = minimum_distance(M, EngineConfig(strategy="stack"))
        out["codes"].append(dict(
            k=k, n=n, rows=hexrows(M), src=f"random_systematic_matrix({k},{n},{seed})",
            brute=brute_force_distance(M), distance=rep.distance, m=rep.m,
            k_m=rep.k_m, g_reached=rep.g_reached, status=rep.status,
            bounds_trace=[list(t) for t in rep.bounds_trace]))
    # known codes (t/conftest.py:9-29, t/test_engine.py:88-104)
    ham = BitMatrix.from_bits([[1, 0, 0, 0, 1, 1, 0], [0, 1, 0, 0, 1, 0, 1],
                               [0, 0, 1, 0, 0, 1, 1], [0, 0, 0, 1, 1, 1, 1]])
    for label, M in (("hamming74", ham), ("repetition5", BitMatrix([0b11111], 5)),
                     ("I4", BitMatrix([1, 2, 4, 8], 4))):
        rep = minimum_distance(M)
        out["codes"].append(dict(
            k=M.num_rows, n=M.num_cols, rows=hexrows(M), src=label,
            brute=brute_force_distance(M), distance=rep.distance, m=rep.m,
            k_m=rep.k_m, g_reached=rep.g_reached, status=rep.status,
            bounds_trace=[list(t) for t in rep.bounds_trace]))
    return out


def cfg4(seed=1):
    M = random_systematic_matrix(64, 192, seed)
    t0 = time.perf_counter()
    res = enumerate_saved(build_saved_store(M, 3), 6)
    return dict(name="cfg4", seed=seed, k=64, n=192, g=6, rows=hexrows(M),
                min_weight=res.min_weight, combinations=res.combinations,
                seconds=round(time.perf_counter() - t0, 3),
                reference_call="enumerate_saved(build_saved_store(G,3),6)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg5", action="store_true")
    args = ap.parse_args()
    if args.cfg5:
        res = run_config("cfg5", 7, s=4)
        with open(os.path.join(HERE, "cfg5_seed7.json"), "w") as fh:
            json.dump(res, fh, indent=1)
        return
    out = {"configs": [], "small": small_fixtures(), "cfg4": cfg4(1)}
    for name in ("cfg1", "cfg2", "cfg3"):
        for seed in CONFIGS[name]["seeds"]:
            out["configs"].append(run_config(name, seed))
    with open(os.path.join(HERE, "goldens.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()

"""Reference traces of config 5 for seeds 1..8, rounds g <= MAX_G.

Test infrastructure only (build container): imports the reference package
from /root/reference, draws each seed's [160,80] code with the Appendix-A
generator (make_golden.draw), runs the reference's minimum_distance with
max_g = MAX_G (strategy "saved", s = 4) and
records rows, pivot sets, the (g, L, U) trace and the combination count in
tests/golden/cfg5_traces.json.  One process per seed.

    python tests/golden/make_cfg5_traces.py     # ~8 min on 8 cores
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
MAX_G = 7


def one(seed: int) -> dict:
    from make_golden import CONFIGS, EngineConfig, draw, minimum_distance

    c = CONFIGS["cfg5"]
    M, gs, draws = draw(c["k"], c["n"], seed, c["target"])
    t0 = time.perf_counter()
    rep = minimum_distance(M, EngineConfig(strategy="saved", s=4, max_g=MAX_G))
    return {"seed": seed, "draws": draws, "k": c["k"], "n": c["n"], "max_g": MAX_G,
            "rows": [format(r, "x") for r in M.rows],
            "pivot_sets": [list(p) for p in gs.pivot_sets],
            "bounds_trace": [list(t) for t in rep.bounds_trace],
            "status": rep.status, "upper": rep.distance, "g_reached": rep.g_reached,
            "combinations": rep.counters.combinations,
            "reference_seconds": round(time.perf_counter() - t0, 1)}


def main():
    with ProcessPoolExecutor(max_workers=8) as ex:
        out = list(ex.map(one, range(1, 9)))
    with open(os.path.join(HERE, "cfg5_traces.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for r in out:
        print(r["seed"], r["bounds_trace"], r["combinations"], r["reference_seconds"], "s")


if __name__ == "__main__":
    main()

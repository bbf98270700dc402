"""The paper's section-6 codes on the GPU: exact minimum distances of
C1 = [234,51], C2 = [234,52] and their extended / punctured relatives
(tests/golden/section6_codes.json), with the time to d.

    python tools/section6.py [NAME ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_06757_b200 import BitMatrix, EngineConfig, minimum_distance  # noqa: E402

fx = json.load(open(os.path.join(ROOT, "tests", "golden", "section6_codes.json")))
want = set(sys.argv[1:])
for c in fx["codes"]:
    if want and c["name"] not in want:
        continue
    G = BitMatrix([int(r, 16) for r in c["rows"]], c["n"])
    minimum_distance(BitMatrix([int(r, 16) for r in c["rows"]][:c["k"]], c["n"]),
                     EngineConfig(max_g=2))  # warm-up (module load, tables)
    t0 = time.perf_counter()
    rep = minimum_distance(G, EngineConfig())
    dt = time.perf_counter() - t0
    print(json.dumps({"name": c["name"], "n": c["n"], "k": c["k"], "d": rep.distance,
                      "paper_d": c["paper_d"], "status": rep.status, "m": rep.m,
                      "k_m": rep.k_m, "g_reached": rep.g_reached,
                      "combinations": rep.counters.combinations, "seconds": round(dt, 3),
                      "rate": rep.counters.combinations / dt,
                      "trace": rep.bounds_trace,
                      "round_ms": [(r.g, round(r.kernel_ms, 3)) for r in rep.rounds]}),
          flush=True)

"""Section-6 code C1 = [234,51]: the g = 12 round alone on K5 (mxf4) and K5w
(mxf4w) against the live fp4 MAC roofline, then the full run to d on the
default engine (wall time).

    python tools/s6_rates.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_06757_b200 import BitMatrix, EngineConfig, _native, minimum_distance  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402
from paper_1603_06757_b200.gf2 import build_gamma_set  # noqa: E402

fx = [c for c in json.load(open(os.path.join(ROOT, "tests/golden/section6_codes.json")))["codes"]
      if c["name"] == "C1"][0]
G = BitMatrix([int(r, 16) for r in fx["rows"]], fx["n"])
gs = build_gamma_set(G)
ctx = _native.context(0)
ctx.load(family_words(gs.gammas, G.num_cols), G.num_cols)
n_eff = G.num_cols - G.num_rows
w = (n_eff + 31) // 32
peaks = ctx.measure_int_peaks(w)
mac = peaks["mxf4_mac_per_s"]
g = 12
for eng in ("mxf4", "mxf4w"):
    ctx.set_engine(eng)
    ms = []
    for i in range(3):
        mins, combos = ctx.round(g, 0, fx["paper_d"] + 1)
        if i:
            ms.append(ctx.last_kernel_ms())
    t = min(ms)
    rate = sum(combos) / (t * 1e-3)
    issued = 64 * ((w + 1) // 2) + (64 if w % 2 == 0 else 0)
    print(json.dumps({"code": "C1 [234,51]", "g": g, "engine": eng, "ms": round(t, 3),
                      "combinations": sum(combos), "rate": rate,
                      "frac_algorithmic": rate / (mac / n_eff), "frac_issued": rate / (mac / issued),
                      "stored_columns": n_eff, "macs_issued": issued}), flush=True)
ctx.set_engine("auto")
minimum_distance(G, EngineConfig(max_g=9))  # warm
t0 = time.perf_counter()
rep = minimum_distance(G, EngineConfig())
dt = time.perf_counter() - t0
print(json.dumps({"code": "C1 [234,51]", "d": rep.distance, "paper_d": fx["paper_d"],
                  "g_final": rep.g_reached, "combinations": rep.counters.combinations,
                  "wall_s": round(dt, 3), "rate": rep.counters.combinations / dt}))

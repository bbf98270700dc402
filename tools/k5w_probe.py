"""K5 vs K5w on wide rows: a random systematic [k + r, k] code (stored
columns r after identity elision), one round g alone per engine.

    python tools/k5w_probe.py [k r g]...
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_06757_b200 import BitMatrix, _native  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402
from paper_1603_06757_b200.gf2 import build_gamma_set  # noqa: E402

args = [int(x) for x in sys.argv[1:]] or [100, 200, 5, 51, 183, 8, 80, 180, 6]
ctx = _native.context(0)
for i in range(0, len(args), 3):
    k, r, g = args[i:i + 3]
    rng = random.Random(k * r + g)
    rows = [(1 << j) | (rng.getrandbits(r) << k) for j in range(k)]
    G = BitMatrix(rows, k + r)
    gs = build_gamma_set(G)
    ctx.load(family_words(gs.gammas, k + r), k + r)
    for eng in ("mxf4", "mxf4w"):
        ctx.set_engine(eng)
        ms = []
        for rep in range(3):
            mins, combos = ctx.round(g, 0, 40 + g)
            if rep:
                ms.append(ctx.last_kernel_ms())
        t = min(ms)
        print(f"[{k + r},{k}] m={len(combos)} g={g} {eng:6s} {t:8.3f} ms  "
              f"{sum(combos) / (t * 1e-3):.3e} comb/s  mins {mins}", flush=True)
ctx.set_engine("auto")

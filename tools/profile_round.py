"""One enumeration launch for ncu: the dominant round (g = 8) of the cfg5
workload, or any (config, g) given on the command line.

    python tools/profile_round.py [config] [g] [--hist] [--engine=NAME]
"""

from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import code, microbench_gamma  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "cfg5"
    g = int(args[1]) if len(args) > 1 else 8
    ctx = _native.context(0)
    for a in sys.argv[1:]:
        if a.startswith("--engine="):
            ctx.set_engine(a.split("=", 1)[1])
    if name == "cfg4":
        gm = microbench_gamma(1)
        ctx.load(family_words([gm], 192), 192)
    else:
        G, gs, _ = code(name)
        ctx.load(family_words(gs.gammas, G.num_cols), G.num_cols)
    t0 = time.perf_counter()
    if "--hist" in sys.argv:
        hist, mn, c = ctx.histogram(0, g)
        res = (mn, c)
    else:
        # --noexit: lower_prev = -1, so debug ablations that wreck the
        # minima never trigger the early exit
        upper = next((int(a.split("=", 1)[1]) for a in sys.argv[1:] if a.startswith("--upper=")),
                     1 << 30)
        lp = -(1 << 30) if "--noexit" in sys.argv else 0
        if "--cold" not in sys.argv:
            ctx.round(g, lp, upper)  # warm-up: lazy module loading, tables
            t0 = time.perf_counter()
        res = ctx.round(g, lp, upper)
    dt = time.perf_counter() - t0
    print(f"{name} g={g}: {res} kernel {ctx.last_kernel_ms():.3f} ms wall {dt*1e3:.1f} ms")


if __name__ == "__main__":
    main()

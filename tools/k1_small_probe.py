"""Device time of config 5's small rounds (g = 1..4): the fused K1 launch of
a BZ run, each round alone on K1, and g = 4 on the tensor-core kernels --
medians of 10 (bz_last_kernel_ms).

    python tools/k1_small_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

ctx = _native.context(0)
G, gs, _ = code("cfg5", int(sys.argv[1]) if len(sys.argv) > 1 else 7)
ctx.load(family_words(gs.gammas, 160), 160)


def timed(label, fn, reps=10):
    ms = []
    for r in range(reps + 1):
        res = fn()
        if r:
            ms.append(ctx.last_kernel_ms())
    ms.sort()
    print(f"{label}: median {ms[len(ms) // 2] * 1e3:.1f} us  min {ms[0] * 1e3:.1f} us  -> {res}",
          flush=True)


U = 21  # config 5's U after round 1 is about this
timed("fused g=1..4", lambda: [r[0] for r in ctx.rounds(1, [0, 4, 6, 8], 1 << 20)])
timed("fused g=1..4 tight", lambda: [r[0] for r in ctx.rounds(1, [0, 4, 6, 8], U)])
for g in (1, 2, 3, 4):
    timed(f"g={g} alone", lambda: ctx.round(g, 0, U))
for eng in ("mxf4q", "mxf4"):
    ctx.set_engine(eng)
    timed(f"g=4 {eng}", lambda: ctx.round(4, 0, U))
    timed(f"g=5 {eng}", lambda: ctx.round(5, 0, U))
ctx.set_engine("popc")
timed("g=5 popc", lambda: ctx.round(5, 0, U))

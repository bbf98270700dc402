"""Device time of batched rounds vs the same rounds alone (cfg5 seed 7):
how much of a batch is gaps between kernels.  python tools/gap_probe.py"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

G, gs, _ = code("cfg5", 7)
ctx = _native.context(0)
ctx.load(family_words(gs.gammas, G.num_cols), G.num_cols)
lps = [0] + [2 * (g + 1) for g in range(1, 8)]


def med(fn, reps=15):
    out = []
    for _ in range(reps):
        fn()
        out.append(ctx.last_kernel_ms())
    return statistics.median(out[3:])


U = 10**6
full = med(lambda: ctx.rounds(1, lps, U))
print(f"batch g=1..8: {full:.4f} ms  per-round {['%.4f' % x for x in ctx.round_ms(8)]}")
for g0, cnt in [(1, 4), (1, 5), (1, 6), (1, 7), (5, 1), (6, 1), (7, 1), (8, 1), (5, 4), (6, 3), (7, 2)]:
    t = med(lambda: ctx.rounds(g0, lps[g0 - 1:g0 - 1 + cnt], U))
    print(f"batch g={g0}..{g0 + cnt - 1}: {t:.4f} ms")

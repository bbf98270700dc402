"""Per-shard device time of config 5's run on one GPU (what rank s of an
N-GPU run executes): the whole batch g = 1..8 and round 8 alone, per-round
kernel times of one shard.

    python tools/shard_probe.py [N]      (env BZ_K5_CHUNK_SCALE etc. apply)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
MIRROR = "--mirror" in sys.argv  # map the shared-bound mirror (own memory) and pre-fill it
G, gs, _ = code("cfg5", 7)
ctx = _native.context(0)
ctx.load(family_words(gs.gammas, 160), 160)
lp = [0] + [2 * (g + 1) for g in range(1, 8)]


def t(fn, reps=5):
    ms = []
    for i in range(reps + 1):
        ctx.timer_start()
        fn()
        x = ctx.timer_stop()
        if i:
            ms.append(x)
    return sorted(ms)[len(ms) // 2]


if MIRROR:
    ctx.shared_bound_export()
    ctx.shared_bound_open(None)
    ctx.shared_bound_epoch(int(os.environ.get("EPOCH", "77")))
    for s in range(N):
        ctx.rounds(1, lp, 81, s, N)
full = t(lambda: ctx.rounds(1, lp, 81, 0, 1))
full8 = t(lambda: ctx.round(8, 16, 18, 0, 1))
print(f"unsharded: batch {full:.4f} ms  g=8 alone {full8:.4f} ms")
tb, t8 = [], []
for s in range(N):
    tb.append(t(lambda: ctx.rounds(1, lp, 81, s, N)))
    t8.append(t(lambda: ctx.round(8, 16, 18, s, N)))
print(f"N={N} batch per shard: " + " ".join(f"{x:.3f}" for x in tb) + f"  max {max(tb):.4f} -> x{full / max(tb):.2f}")
print(f"N={N} g=8   per shard: " + " ".join(f"{x:.3f}" for x in t8) + f"  max {max(t8):.4f} -> x{full8 / max(t8):.2f}")
ctx.rounds(1, lp, 81, 0, N)
print("shard 0 per-round kernel ms:", [round(x, 4) for x in ctx.round_ms(8)], "launches", ctx.launch_count())

"""K5f (folded MMAs) against K5q on config 5 seed 7: same minima and
combination counts per round, then the g = 8 round and the batch g = 1..8
timed interleaved on one box.

    python tools/k5f_probe.py [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
G, gs, _ = code("cfg5", 7)
ctx = _native.context(0)
engines = ("mxf4q", "mxf4f")
with ctx.lock:
    ctx.load(family_words(gs.gammas, 160), 160)
    ref = {}
    for eng in engines:
        ctx.set_engine(eng)
        for g in (4, 5, 6, 7):
            for upper in (1 << 30, 18, 17):
                got = ctx.round(g, 0, upper)
                ref.setdefault((g, upper), got)
                print(eng, g, upper, got, "OK" if got == ref[(g, upper)] else "MISMATCH")
    t = {e: {"g8": [], "batch": []} for e in engines}
    lp = [0] + [2 * (g + 1) for g in range(1, 8)]
    for _ in range(reps):
        for eng in engines:
            ctx.set_engine(eng)
            r8 = ctx.round(8, 0, 18)
            t[eng]["g8"].append(ctx.last_kernel_ms())
            rb = ctx.rounds(1, lp, 81)
            t[eng]["batch"].append(ctx.last_kernel_ms())
            ref.setdefault("g8", r8)
            ref.setdefault("batch", rb)
            if r8 != ref["g8"] or rb != ref["batch"]:
                print(eng, "MISMATCH", r8, rb)
    ctx.set_engine("auto")
print("g8", ref["g8"])
for eng in engines:
    g8 = sorted(t[eng]["g8"][1:])
    b = sorted(t[eng]["batch"][1:])
    print(f"{eng}: g8 alone {g8[len(g8) // 2]:.4f} ms (min {g8[0]:.4f})   "
          f"rounds 1..8 {b[len(b) // 2]:.4f} ms (min {b[0]:.4f})")

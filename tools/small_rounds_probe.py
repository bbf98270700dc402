"""Device time of the small tensor-core launches: config 4 (all C(64,6)
six-row combinations of one 64x192 [I | A]) and config 5's rounds g = 5..7
launched one at a time, then one per-chunk timeline of each
(BZ_K4_DEBUG & 32, summarised by tools/chunk_times.py).

    python tools/small_rounds_probe.py [out_dir]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import code, microbench_gamma  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
os.makedirs(out, exist_ok=True)
ctx = _native.context(0)


def timed(label, fn, reps=6):
    ms = []
    for r in range(reps):
        res = fn()
        if r:
            ms.append(ctx.last_kernel_ms())
    ms.sort()
    print(f"{label}: median {ms[len(ms) // 2] * 1e3:.1f} us  min {ms[0] * 1e3:.1f} us  -> {res}",
          flush=True)


gm = microbench_gamma(1)
ctx.load(family_words([gm], 192), 192)
for eng in ("auto", "mxf4", "popc"):
    ctx.set_engine(eng)
    timed(f"cfg4 g=6 {eng}", lambda: ctx.enumerate(0, 6))
ctx.set_engine("auto")
timed("cfg4 g=6 histogram (K1h)", lambda: ctx.histogram(0, 6)[1:])

G, gs, _ = code("cfg5", 7)
ctx.load(family_words(gs.gammas, 160), 160)
for g in (4, 5, 6, 7):
    timed(f"cfg5 g={g} auto", lambda: ctx.round(g, 0, 1 << 20))

if os.environ.get("BZ_K4_DEBUG"):
    sys.exit(0)
# chunk timelines (a child process per launch: the debug switch is read per call)
for label, script in (("cfg4", "ctx.load(family_words([microbench_gamma(1)], 192), 192); ctx.enumerate(0, 6)"),
                      ("cfg5g5", "G, gs, _ = code('cfg5', 7); ctx.load(family_words(gs.gammas, 160), 160); ctx.round(5, 0, 1 << 20)"),
                      ("cfg5g7", "G, gs, _ = code('cfg5', 7); ctx.load(family_words(gs.gammas, 160), 160); ctx.round(7, 0, 1 << 20)")):
    path = os.path.join(out, f"ct_{label}.bin")
    env = dict(os.environ, BZ_K4_DEBUG="32", BZ_K4_CTRACE=path)
    code_s = ("import sys; sys.path.insert(0, %r)\n" % ROOT +
              "from paper_1603_06757_b200 import _native\n"
              "from paper_1603_06757_b200.configs import code, microbench_gamma\n"
              "from paper_1603_06757_b200.enumeration import family_words\n"
              "ctx = _native.context(0)\n" + script + "\n")
    subprocess.run([sys.executable, "-c", code_s], env=env, check=True)
    print(f"-- chunk timeline {label}", flush=True)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "chunk_times.py"), path], check=True)

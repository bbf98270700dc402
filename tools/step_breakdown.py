"""Where the time of one config-5 BZ run goes on the host: the bench step
(start_state + run_rounds, family resident) against its device-timed span,
the bz_advance calls alone and the kernels' own device time -- medians of 30.

    python tools/step_breakdown.py [cfg5] [seed]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import EngineConfig, engine  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
G, gs, _ = code(name, seed)
k, n = G.num_rows, G.num_cols
cfg = EngineConfig()
backend = engine.make_backend(cfg, engine._make_comm(cfg))
backend.load(gs, n)
ctx = backend.ctx

calls = []
real_advance = ctx.advance


def timed_advance(*a, **kw):
    g0 = int(a[-1][0])
    t0 = time.perf_counter()
    r = real_advance(*a, **kw)
    calls.append((g0, len(r), time.perf_counter() - t0))
    return r


ctx.advance = timed_advance


def step():
    st = engine.start_state(gs, n, k, cfg)
    engine.run_rounds(backend, gs, k, cfg, st)
    return st


for _ in range(5):
    step()
wall, dev, kern, inner = [], [], [], []
for _ in range(30):
    calls.clear()
    ctx.timer_start()
    t0 = time.perf_counter()
    st = step()
    wall.append((time.perf_counter() - t0) * 1e3)
    dev.append(ctx.timer_stop())
    kern.append(sum(r.kernel_ms for r in st.rounds))
    inner.append(sum(c[2] for c in calls) * 1e3)
med = statistics.median
print(f"{name} seed {seed}: step wall {med(wall):.3f} ms, device span {med(dev):.3f} ms, "
      f"kernels {med(kern):.3f} ms, bz_advance calls {med(inner):.3f} ms "
      f"({len(calls)} calls: {[(c[0], c[1]) for c in calls]})")
print(f"  host outside bz_advance {med(wall) - med(inner):.3f} ms; "
      f"bz_advance beyond kernels {med(inner) - med(kern):.3f} ms")

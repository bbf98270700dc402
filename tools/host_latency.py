"""Host-side latency of the public path on tiny work: config 1 (k = 24; the
kernels run a few microseconds) through minimum_distance, the engine loop
with the family resident, and a bare bz_rounds call -- medians of 300.

    python tools/host_latency.py
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import EngineConfig, engine, minimum_distance  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402

G, gs, _ = code("cfg1", 2)
cfg = EngineConfig()


def med(fn, n=300):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


backend = engine.make_backend(cfg, engine._make_comm(cfg))
backend.load(gs, G.num_cols)
ctx = backend.ctx


def loop():
    st = engine.start_state(gs, G.num_cols, G.num_rows, cfg)
    engine.run_rounds(backend, gs, G.num_rows, cfg, st)


print(f"minimum_distance (cfg1): {med(lambda: minimum_distance(G, cfg)):.1f} us")
print(f"engine loop, family resident: {med(loop):.1f} us")
print(f"bare ctx.rounds(1..3): {med(lambda: ctx.rounds(1, [0, 4, 6], 25)):.1f} us")
print(f"bare ctx.round(1): {med(lambda: ctx.round(1, 0, 25)):.1f} us")

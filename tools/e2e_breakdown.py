"""Where the end-to-end time of minimum_distance(G) goes on config 5: the
Gamma family on the host, the upload, the rounds (suffix tables rebuilt
after every upload) and the rest -- medians of 30, against the same rounds
with the family already resident.

    python tools/e2e_breakdown.py [cfg5] [seed]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import EngineConfig, engine, minimum_distance  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402
from paper_1603_06757_b200.gf2 import build_gamma_set  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
G, _, _ = code(name, seed)
k, n = G.num_rows, G.num_cols
cfg = EngineConfig()
backend = engine.make_backend(cfg, engine._make_comm(cfg))
ctx = backend.ctx


def timed(fn, reps=30):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        ctx.synchronize() if hasattr(ctx, "synchronize") else None
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


gs = build_gamma_set(G)
t_md = timed(lambda: minimum_distance(G, cfg))
t_family = timed(lambda: build_gamma_set(G))
t_load = timed(lambda: backend.load(gs, n))


def load_and_run():
    backend.load(gs, n)
    st = engine.start_state(gs, n, k, cfg)
    engine.run_rounds(backend, gs, k, cfg, st)


def run_resident():
    st = engine.start_state(gs, n, k, cfg)
    engine.run_rounds(backend, gs, k, cfg, st)


t_load_run = timed(load_and_run)
backend.load(gs, n)
t_run = timed(run_resident)
print(f"{name} seed {seed}: minimum_distance {t_md:.3f} ms | family {t_family:.3f} | "
      f"load {t_load:.3f} | load + rounds {t_load_run:.3f} | rounds resident {t_run:.3f} ms")

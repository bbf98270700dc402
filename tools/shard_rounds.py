"""Per-round kernel times of one shard against the unsharded run (config 5,
any seed): python tools/shard_rounds.py [seed] [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import EngineConfig, _native, engine  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 2
G, gs, _ = code("cfg5", seed)
cfg = EngineConfig()
backend = engine.make_backend(cfg, engine._make_comm(cfg))
backend.load(gs, G.num_cols)
ctx = backend.ctx
st = engine.start_state(gs, G.num_cols, G.num_rows, cfg)
u0 = st.U
engine.run_rounds(backend, gs, G.num_rows, cfg, st)
lp = [0] + [t[1] for t in st.trace[:-1]]
n = len(lp)
for up, tag in ((u0, "loose start"), (st.U + 1, "start at d + 1")):
    for s, nsh in [(0, 1)] + [(s, N) for s in range(N)]:
        best = None
        for _ in range(3):
            ctx.timer_start()
            res = ctx.rounds(1, lp, up, s, nsh)
            ms = ctx.timer_stop()
            r = ctx.round_ms(n)
            if best is None or ms < best[0]:
                best = (ms, r, res)
        ms, r, res = best
        print(f"{tag:16s} shard {s}/{nsh}: {ms:8.4f} ms  rounds " + " ".join(f"{x:.3f}" for x in r) +
              "  mins " + str([min(x[0]) for x in res][-3:]))

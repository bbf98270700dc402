"""Per-round kernel vs wall time of one full BZ run (device-resident)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import EngineConfig, engine  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
G, gs, _ = code(name)
cfg = EngineConfig()
backend = engine.make_backend(cfg, engine._make_comm(cfg))
backend.load(gs, G.num_cols)
for rep in range(3):
    st = engine.start_state(gs, G.num_cols, G.num_rows, cfg)
    t0 = time.perf_counter()
    engine.run_rounds(backend, gs, G.num_rows, cfg, st)
    dt = (time.perf_counter() - t0) * 1e3
ksum = sum(r.kernel_ms for r in st.rounds)
print(f"{name}: wall {dt:.3f} ms, kernels {ksum:.3f} ms")
for r in st.rounds:
    print(f"  g={r.g}: kernel {r.kernel_ms:.3f} ms wall {r.wall_ms:.3f} ms combos {r.combinations}")

import sys, time, os
sys.path.insert(0, os.getcwd())
from paper_1603_06757_b200 import EngineConfig, minimum_distance, engine
from paper_1603_06757_b200.configs import code
from paper_1603_06757_b200.gf2 import build_gamma_set
G, gs, _ = code("cfg5", 7)
cfg = EngineConfig()
for _ in range(3): minimum_distance(G, cfg)
N=10
t=time.perf_counter()
for _ in range(N): gs2 = build_gamma_set(G)
print("build_gamma_set ms", (time.perf_counter()-t)/N*1e3)
backend = engine.make_backend(cfg, engine._make_comm(cfg))
t=time.perf_counter()
for _ in range(N): backend.load(gs, G.num_cols); backend.ctx.last_kernel_ms()
import ctypes
print("load ms", (time.perf_counter()-t)/N*1e3)
t=time.perf_counter()
for _ in range(N):
    st = engine.start_state(gs, G.num_cols, G.num_rows, cfg); engine.run_rounds(backend, gs, G.num_rows, cfg, st)
print("run_rounds ms", (time.perf_counter()-t)/N*1e3)
t=time.perf_counter()
for _ in range(N): minimum_distance(G, cfg)
print("minimum_distance ms", (time.perf_counter()-t)/N*1e3)
import cProfile, pstats
pr=cProfile.Profile(); pr.enable()
for _ in range(N): minimum_distance(G, cfg)
pr.disable(); pstats.Stats(pr).sort_stats('cumtime').print_stats(18)

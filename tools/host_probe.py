"""Host-side cost around one device-resident cfg5 run: the bench's timed
step vs the library call vs the kernels.  python tools/host_probe.py"""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1603_06757_b200 import EngineConfig, engine  # noqa: E402
from paper_1603_06757_b200.configs import code  # noqa: E402

G, gs, _ = code("cfg5", 7)
n, k = G.num_cols, G.num_rows
cfg = EngineConfig()
backend = engine.make_backend(cfg, engine._make_comm(cfg))
backend.load(gs, n)
ctx = backend.ctx
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda:0")
lps = [0] + [2 * (g + 1) for g in range(1, 8)]
for label, fl in (("no flush", False), ("L2 flushed", True)):
    rows = []
    for it in range(20):
        if fl:
            flush.zero_()
        torch.cuda.synchronize()
        ctx.timer_start()
        t0 = time.perf_counter()
        st = engine.start_state(gs, n, k, cfg)
        engine.run_rounds(backend, gs, k, cfg, st)
        t1 = time.perf_counter()
        dev = ctx.timer_stop()
        rows.append((dev, (t1 - t0) * 1e3, ctx.last_kernel_ms()))
    rows = rows[5:]
    print(label, "step dev %.4f  host wall %.4f  kernels(ev_k0..k1) %.4f ms" %
          tuple(statistics.median(r[i] for r in rows) for i in range(3)))
    rows = []
    for it in range(20):
        if fl:
            flush.zero_()
        torch.cuda.synchronize()
        ctx.timer_start()
        ctx.rounds(1, lps, 10**6)
        dev = ctx.timer_stop()
        rows.append((dev, ctx.last_kernel_ms()))
    rows = rows[5:]
    print(label, "bare ctx.rounds dev %.4f  kernels %.4f ms" %
          tuple(statistics.median(r[i] for r in rows) for i in range(2)))

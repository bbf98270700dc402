"""Benchmark: codeword combinations (XOR+popcount)/s and wall time to d.

Workload (BASELINE.json configs[4], the config its scaling target names):
the random binary [160,80] code of seed 7 (SURVEY.md Appendix A generator,
2 full information sets), full Brouwer-Zimmermann from g = 1 until L >= U
(d = 17 at g = 8, 6.5e10 combinations).  One *step* is one such run.

  value  -- combinations/s of the rounds with the Gamma family resident in
            HBM (device-timed with CUDA events on the library's stream, one
            event pair per step, L2 flushed before each step), summed over
            ranks / max-over-ranks time.
  e2e    -- the same metric through the public API minimum_distance(G, ...)
            from a host BitMatrix: Gamma construction, H2D of the rows and
            of every round's work plan, all rounds, D2H of every round's
            minima and counters, timed by the host clock.
  roofline -- the dominant kernel (the g = 8 round, K5q = tcgen05.mma
            kind::mxf4nvf4, two codewords as bytes of one fp32 TMEM
            accumulator) against the live fp4 MAC rate: `frac` per
            ALGORITHMIC MACs (the stored columns of a codeword, 80 for config
            5), `frac_issued` per MACs the kernel issues (its padded K plus
            the offset chunks, 128); "k5_mxf4" and "k1_popc" time the other
            two kernels of the library on the same launch.
  cfg4   -- BASELINE.json configs[3]: all C(64,6) six-row combinations of a
            64x192 [I | A], minimum (K5q) and the 193-bin weight histogram
            (K1h), each against its roofline.
  cpu_baseline -- the C oracle (oracle/, a restatement of the reference's
            enumerate_stack) on all host cores over a bounded sample.

  python bench.py [--gpus N --steps K --warmup W]   (N > 1: one rank per GPU,
                                                     spawned through torchrun
                                                     unless already under it)
  python bench.py --impl reference                  (CPU reference arm)
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "codeword combinations (XOR+popcount)/s, full BZ to d"
UNIT = "combinations/s"
WORKLOAD = "cfg5 random [160,80] seed 7, full BZ to d (g=1..8)"
# BASELINE.json configs (name -> k, n, (full-rank count, remainder rank), default seed)
CODES = {"cfg1": (24, 48, (2, 0), 1), "cfg2": (48, 96, (2, 0), 1),
         "cfg3": (40, 100, (2, 20), 1), "cfg5": (80, 160, (2, 0), 7)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="cfg5", choices=tuple(CODES))
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the side measurements")
    ap.add_argument("--cpu-sample-g", type=int, default=7)
    ap.add_argument("--ref-python-max-g", type=int, default=5,
                    help="reference arm: rounds of the reference package's own run")
    ap.add_argument("--cpu-selftest", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: launch N ranks of this
    script through torchrun (one process per GPU, 127.0.0.1 rendezvous) and
    pass their output through; rank 0 prints the JSON line.  NCCL reports
    its communicator setup (NCCL_DEBUG=INFO, INIT subsystem) unless the
    caller chose otherwise."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    if not args.cpu_selftest:
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region.

    nvidia-smi polls every 10 ms; a reader thread stamps each line with the
    host clock, entering waits for the first line (so the poller is running
    when the timed region starts) and the summary keeps the lines stamped
    inside the region (or the last one before it when the region is shorter
    than a poll period)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.stamped = []
        self.t0 = self.t1 = None

    def _read(self):
        for ln in self.proc.stdout:
            if ln.strip():
                self.stamped.append((time.perf_counter(), ln))

    def __enter__(self):
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
            deadline = time.perf_counter() + 5.0
            while not self.stamped and time.perf_counter() < deadline:
                time.sleep(0.002)
        except OSError:
            self.proc = None
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        self.t1 = time.perf_counter()
        if self.proc is not None:
            time.sleep(0.02)  # the poll that covers the region's last milliseconds
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.reader.join(timeout=5)

    def summary(self):
        inside = [ln for t, ln in self.stamped if self.t0 <= t <= self.t1 + 0.02]
        before = [ln for t, ln in self.stamped if t < self.t0]
        lines = inside or before[-1:]
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "samples_in_region": len(inside),
                "region_ms": None if self.t1 is None else round((self.t1 - self.t0) * 1e3, 2)}


def other_seeds(args, cfg, local, flush) -> dict:
    """Side measurement (not the headline): the same metric on config 5
    seeds 1 and 3, typical random [160,80] codes that need round g = 9
    (5.3e11 combinations per run, d = 19 / 20).  Device-resident, L2
    flushed before each run, median of 3 runs after one warm-up."""
    import torch

    from paper_1603_06757_b200 import engine
    from paper_1603_06757_b200.configs import code

    out = {}
    for seed in (1, 3):
        G, gs, _ = code("cfg5", seed)
        k, n = G.num_rows, G.num_cols
        backend = engine.make_backend(cfg, engine._make_comm(cfg))
        backend.load(gs, n)
        ctx = backend.ctx
        times, combos, st = [], 0, None
        for rep in range(4):
            flush.zero_()
            torch.cuda.synchronize(local)
            ctx.timer_start()
            st = engine.start_state(gs, n, k, cfg)
            engine.run_rounds(backend, gs, k, cfg, st)
            ms = ctx.timer_stop()
            if rep:
                times.append(ms)
            combos = st.counters.combinations
        ms = statistics.median(times)
        out[f"seed{seed}"] = {"value": combos / (ms * 1e-3), "unit": UNIT, "ms_per_run": ms,
                              "combinations": combos, "d": st.U, "g_final": st.g_reached}
        if seed == 1:
            # the same per-shard measurement as the headline's, on a typical
            # code (g = 9: 8x the work per run)
            out["seed1"]["shards_on_one_gpu"] = shard_times(
                ctx, st, engine.start_state(gs, n, k, cfg).U, gs.matrix_count, flush,
                lambda: torch.cuda.synchronize(local), reps=1)
    return out


def section6_c1(cfg) -> dict:
    """Side measurement: the paper's new code C1 = [234,51] (section 6;
    generator from tests/golden/section6_codes.json, built by the reference
    package) to its exact distance through minimum_distance, wall time
    (one warm-up run first)."""
    from paper_1603_06757_b200 import BitMatrix, minimum_distance

    path = os.path.join(ROOT, "tests", "golden", "section6_codes.json")
    if not os.path.exists(path):
        return {"skipped": "tests/golden/section6_codes.json missing"}
    with open(path) as fh:
        fx = [c for c in json.load(fh)["codes"] if c["name"] == "C1"][0]
    G = BitMatrix([int(r, 16) for r in fx["rows"]], fx["n"])
    minimum_distance(G, cfg)
    t0 = time.perf_counter()
    rep = minimum_distance(G, cfg)
    dt = time.perf_counter() - t0
    return {"code": f"[{fx['n']},{fx['k']}]", "d": rep.distance, "paper_d": fx["paper_d"],
            "status": rep.status, "g_final": rep.g_reached,
            "combinations": rep.counters.combinations, "wall_s": round(dt, 3),
            "value": rep.counters.combinations / dt, "unit": UNIT}


def configs_wall(cfg) -> dict:
    """Side measurement: wall time to d of BASELINE.json configs 1-3 (two
    seeds each, the Appendix-A generator) through the public API
    minimum_distance(G, ...) from a host BitMatrix -- Gamma family, upload,
    every round, read-back -- median of 5 after one warm-up.  These configs
    are launch-latency bound: the wall time to d, not the
    combination rate, is their number.  The reference reports the same
    `elapsed` (m/engine.py:168, :246)."""
    from paper_1603_06757_b200 import minimum_distance
    from paper_1603_06757_b200.configs import code

    out = {}
    for name in ("cfg1", "cfg2", "cfg3"):
        for seed in (1, 2):
            G, _, _ = code(name, seed)
            minimum_distance(G, cfg)
            walls = []
            for _ in range(5):
                t0 = time.perf_counter()
                rep = minimum_distance(G, cfg)
                walls.append(time.perf_counter() - t0)
            wall = statistics.median(walls)
            out[f"{name}_seed{seed}"] = {
                "n": G.num_cols, "k": G.num_rows, "d": rep.distance, "g_final": rep.g_reached,
                "trace": [list(t) for t in rep.bounds_trace],
                "combinations": rep.counters.combinations, "wall_ms": round(wall * 1e3, 3),
                "value": rep.counters.combinations / wall, "unit": UNIT}
    return out


def issued_macs(w: int) -> int:
    """MACs per combination the K5 family issues for W stored 32-bit words:
    ceil(W/2) K = 64 MMAs (the A/table offset chunk rides in the padding of
    the last one for odd W), plus one offset MMA for even W -- per codeword
    for K5 (one per accumulator column) and for K5q (two per column, two
    parts)."""
    return 64 * ((w + 1) // 2) + (64 if w % 2 == 0 else 0)


def cfg4_side(ctx, peaks, seed: int = 1) -> dict:
    """BASELINE.json configs[3]: the fixed-r microbenchmark.  All C(64,6) =
    74,974,368 six-row combinations of random_systematic_matrix(64, 192, 1)
    = [I_64 | A], no early exit: the minimum on the default engine (K5q:
    128 stored columns after identity elision, two codewords per
    accumulator) and the 193-bin weight histogram (K1h: XOR+POPC with
    per-thread shared-memory bins), device-timed (median of 5 after one
    warm-up), against their rooflines.  Reference: enumerate_saved /
    enumerate_parallel on the same Gamma (m/enumeration.py:305-313,
    :385-444), 3.6 s on one core."""
    import hashlib

    import numpy as np

    from paper_1603_06757_b200.configs import microbench_gamma
    from paper_1603_06757_b200.enumeration import family_words

    gm = microbench_gamma(seed)
    n, k, g = gm.num_cols, gm.num_rows, 6
    ctx.set_engine("auto")
    ctx.load(family_words([gm], n), n)
    stored = n - k if ctx.elided() & 1 else n
    w_st = (stored + 31) // 32
    ms_min, ms_hist = [], []
    for rep in range(6):
        mn, combos = ctx.enumerate(0, g)
        if rep:
            ms_min.append(ctx.last_kernel_ms())
    for rep in range(6):
        hist, hmn, hcombos = ctx.histogram(0, g)
        if rep:
            ms_hist.append(ctx.last_kernel_ms())
    t_min, t_hist = statistics.median(ms_min), statistics.median(ms_hist)
    sha = hashlib.sha256(np.asarray(hist, dtype="<u8").tobytes()).hexdigest()
    r_min = combos / (t_min * 1e-3)
    r_hist = hcombos / (t_hist * 1e-3)
    issued = issued_macs(w_st)
    mac = peaks["mxf4_mac_per_s"]
    popc_peak = peaks["popc_per_s"] / w_st
    return {
        "workload": "random_systematic_matrix(64,192,1), all C(64,6) combinations, no early exit",
        "combinations": combos, "min": mn, "hist_sha256": sha,
        "hist_checksum_ok": sha == "8d397da157d31b1e67746a3a522b01cb624e4d54d42a27b6fbd403a6da02252b",
        "stored_columns": stored,
        "min_k5q": {"ms": t_min, "value": r_min, "unit": UNIT,
                    "roofline_peak": mac / stored, "frac": r_min / (mac / stored),
                    "frac_issued": r_min / (mac / issued),
                    "note": f"algorithmic MACs = {stored} stored columns per combination; "
                            f"issued = {issued} (K5q, even W: one offset MMA per part)"},
        "histogram_k1h": {"ms": t_hist, "value": r_hist, "unit": UNIT,
                          "roofline_peak": popc_peak, "frac": r_hist / popc_peak,
                          "note": f"POPC roofline / {w_st} words per stored codeword"},
        "reference_1core_s": 3.6,
    }


_SHARD_EPOCH = itertools.count(0x7000)


def shard_times(ctx, st, u0: int, m: int, flush, sync, reps: int = 2) -> dict:
    """What one rank of an N-GPU run does, measured on THIS GPU: the run's
    rounds as shard s of N (bz_rounds(..., shard=s, nshards=N): the chunks
    with c % N == s; rounds too small to split go whole to one rank) for every
    s in turn, device time of each by CUDA events on the library stream.  The
    slowest shard is the device time a rank would need at N GPUs -- without
    the per-batch exchange (one all-gather of 4m int64) -- so t(1) / slowest
    is the device-side scaling the rank-space sharding allows, not a
    multi-GPU measurement.  Two brackets of what the ranks' shared bound (the
    CUDA-IPC mirror every rank's kernels publish to and tighten their
    thresholds from) does for a rank: "own_bound" -- no mirror, a shard only
    knows its own finds (the lower bracket); "shared_bound" -- the mirror
    mapped in this one process and filled by an untimed pass over all
    shards, so every timed shard starts from the job's minima as if another
    rank had just found them (the upper bracket).  Also checks the sharding
    on the device: per round, the minimum over shards and the sum of their
    combination counts equal the unsharded run's."""
    lp = [0] + [t[1] for t in st.trace[:-1]]  # L_prev of round g = L after round g - 1
    full = [(t[2], r.combinations) for t, r in zip(st.trace, st.rounds)]

    def run(s, nsh):
        flush.zero_()
        sync()
        ctx.timer_start()
        res = ctx.rounds(1, lp, u0, s, nsh)
        return ctx.timer_stop(), res

    def folded(results):
        """min over shards / sum of counts per round == the unsharded run's?"""
        mins, sums = None, None
        for res in results:
            mn = [min(r[0]) for r in res]
            cb = [sum(r[1]) for r in res]
            mins = mn if mins is None else [min(a, b) for a, b in zip(mins, mn)]
            sums = cb if sums is None else [a + b for a, b in zip(sums, cb)]
        # U after round g is the running minimum of the rounds' minima
        run_min, ok = u0, True
        for g, (u_full, c_full) in enumerate(full):
            run_min = min(run_min, mins[g])
            ok = ok and run_min == u_full and sums[g] == c_full
        return ok

    def sweep(nsh, check=None):
        times, results = [], []
        for s in range(nsh):
            ms, res = min((run(s, nsh) for _ in range(reps)), key=lambda x: x[0])
            times.append(ms)
            results.append(res)
        return {"shard_ms": [round(t, 4) for t in times], "slowest_ms": max(times),
                "device_speedup": t1 / max(times),
                "matches_unsharded": folded(results) if check is None else check}

    out = {"rounds": len(lp), "note": "per-shard device time on one GPU, shards run one after "
                                      "another, no exchange; own_bound / shared_bound bracket the "
                                      "effect of the ranks' shared bound"}
    t1 = statistics.median(run(0, 1)[0] for _ in range(3))
    out["unsharded_ms"] = t1
    for nsh in (2, 4, 8):
        out[f"N{nsh}"] = {"own_bound": sweep(nsh)}
    ctx.shared_bound_export()
    ctx.shared_bound_open(None)
    try:
        for nsh in (2, 4, 8):
            ctx.shared_bound_epoch(next(_SHARD_EPOCH))  # a newer tag per sweep
            # untimed: every shard's minima into the mirror, each shard seeing
            # the finds of the ones before it -- the fold of THIS pass is the
            # sharded result (in the timed pass the mirror already holds every
            # minimum, so no shard finds anything below it to report)
            ok = folded([ctx.rounds(1, lp, u0, s, nsh) for s in range(nsh)])
            out[f"N{nsh}"]["shared_bound"] = sweep(nsh, check=ok)
    finally:
        ctx.shared_bound_close()
    return out


def cpu_baseline(G, gs, sample_g: int) -> dict:
    """Oracle (C restatement of enumerate_stack) on all host cores over one
    bounded sample: every g-combination of Gamma_1 at g = sample_g."""
    from oracle import oracle

    threads = oracle.max_threads()
    gm = gs.gammas[0]
    t0 = time.perf_counter()
    mn, combos = oracle.min_weight(list(gm.rows), gm.num_cols, sample_g, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": combos / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"all C(80,{sample_g}) = {combos} combinations of Gamma_1 "
                      f"(min {mn}) in {dt:.2f} s, oracle/bz_oracle.c on {threads} threads"}


def reference_python(rows: list[int], n: int, max_g: int) -> dict:
    """The reference package itself (baseline/_ref, installed from
    /root/reference/pkg; pure Python + numpy) on the same code:
    minimum_distance(G, EngineConfig(strategy="saved", s=3, workers=W))
    (m/engine.py:57-67, :157-220) over rounds g <= max_g, W = 1 and W = all
    host cores.  Its rounds past max_g take hours."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mindist")):
        return {"unavailable": "baseline/_ref is not installed"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from mindist.engine import EngineConfig as RefConfig
    from mindist.engine import minimum_distance as ref_md
    from mindist.gf2 import BitMatrix as RefMatrix

    cores = len(os.sched_getaffinity(0))
    out = {"package": "mindist 0.1.0 (baseline/_ref)", "rounds": f"g<={max_g}"}
    for w in sorted({1, cores}):
        t0 = time.perf_counter()
        rep = ref_md(RefMatrix(list(rows), n),
                     RefConfig(strategy="saved", s=3, workers=w, max_g=max_g))
        dt = time.perf_counter() - t0
        out[f"workers_{w}"] = {"value": rep.counters.combinations / dt, "unit": UNIT,
                               "s": round(dt, 3), "combinations": rep.counters.combinations,
                               "bounds_trace": [list(t) for t in rep.bounds_trace]}
    out["cores"] = cores
    return out


def reference_arm(args):
    """The CPU reference arm: the oracle port of the reference's path
    (oracle/bz_oracle.c, enumerate_stack on all host threads inside the
    Algorithm-1 loop) on the SAME workload as the GPU arm -- every round of
    full BZ to d.  The input is drawn by oracle.draw_code (no product
    package import).  Under torchrun only rank 0 runs; the GPU count only
    labels the line."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle

    k, n, target, seed0 = CODES[args.config]
    seed = seed0 if args.seed is None else args.seed
    rows = oracle.draw_code(k, n, seed, target)
    threads = oracle.max_threads()

    def step():
        return oracle.minimum_distance(rows, n, threads=threads)

    for _ in range(args.warmup):
        step()
    times, combos = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rep = step()
        times.append(time.perf_counter() - t0)
        combos += rep["combinations"]
    total = sum(times)
    value = combos / total
    workload = WORKLOAD if args.config == "cfg5" else f"{args.config} seed {seed}, full BZ to d"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": workload, "k": k, "n": n, "d": rep["distance"],
                   "g_final": rep["g_reached"],
                   "combinations_per_step": rep["combinations"]},
        "wall_time_to_d_s": total / args.steps,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"oracle/bz_oracle.c (enumerate_stack restated in C, "
                                   f"pthreads) full BZ to d of {workload}: "
                                   f"{rep['combinations']} combinations per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_extra:
        line["reference_python"] = reference_python(rows, n, args.ref_python_max_g)
    print(json.dumps(line), flush=True)


def cpu_selftest(args):
    """Hidden CPU mode for tests/test_bench_launch.py: the rank launcher,
    barriers, max-over-ranks timing and the JSON contract on gloo, with a
    fixed host-side step instead of the device rounds."""
    rank, world, _ = dist_env()
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    steps_ms = []
    for i in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        time.sleep(0.002 * (1 + rank))
        if i >= args.warmup:
            steps_ms.append((time.perf_counter() - t0) * 1e3)
    ms = sum(steps_ms)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": world * args.steps / (ms * 1e-3),
                          "unit": "steps/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "selftest": True}), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.cpu_selftest:
        cpu_selftest(args)
        return
    if args.impl == "reference":
        reference_arm(args)
        return
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")

    import torch

    distributed = world > 1
    if distributed:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1603_06757_b200 import EngineConfig, _native, engine, minimum_distance
    from paper_1603_06757_b200.configs import code

    G, gs, _ = code(args.config, args.seed)
    k, n, m = G.num_rows, G.num_cols, gs.matrix_count
    w32 = -(-n // 32)
    cfg = EngineConfig(device=local, distributed=distributed)
    comm = engine._make_comm(cfg)
    backend = engine.make_backend(cfg, comm)
    backend.load(gs, n)
    ctx = backend.ctx

    def barrier():
        if distributed:
            comm.barrier()
        torch.cuda.synchronize(local)

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")

    def step():
        st = engine.start_state(gs, n, k, cfg)
        engine.run_rounds(backend, gs, k, cfg, st)
        return st

    # warm-up
    for _ in range(max(args.warmup, 3)):
        st = step()
    ref_trace = st.trace

    # ---- value: device-resident rounds, CUDA events on the library stream
    launches0 = ctx.launch_count()
    dev_ms, combos_total, g_top_ms, g_top_combos = 0.0, 0, [], 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            ctx.timer_start()
            st = step()
            dev_ms += ctx.timer_stop()
            combos_total += st.counters.combinations
            top = max(st.rounds, key=lambda r: r.combinations)
            g_top_ms.append(top.kernel_ms)
            g_top_combos = top.combinations
            assert st.trace == ref_trace
    launches = ctx.launch_count() - launches0
    clock = clocks.summary()

    # max over ranks of the time; the counters are already whole-job sums
    # (every round's all-gather adds the shards' combination counts)
    dev_ms_max = dev_ms
    if distributed:
        import torch.distributed as dist

        t_max = torch.tensor([dev_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dev_ms_max = float(t_max.item())
    combos_all = float(combos_total)
    value = combos_all / (dev_ms_max * 1e-3)

    # ---- e2e: public API from a host matrix
    e2e_times = []
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        rep = minimum_distance(G, cfg)
        barrier()
        e2e_times.append(time.perf_counter() - t0)
        assert rep.bounds_trace == ref_trace
    e2e_s = statistics.median(e2e_times)
    if distributed:
        import torch.distributed as dist

        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = rep.counters.combinations / e2e_s
    # the device stores only the kept columns (identity-column elision)
    mask = ctx.elided()
    n_eff = max((n - k) if (mask >> j) & 1 else n for j in range(m))
    w_eff = (max(n_eff, 1) + 31) // 32
    wp = 1 if w_eff <= 1 else 2 if w_eff <= 2 else 4 if w_eff <= 4 else 8
    h2d = m * k * wp * 4 + m * (k + 1) * wp * 4  # padded rows + prefix-XOR table
    # per round: a result record {cursor, combos[m], bounds[m+1]} both ways
    # and the round's plan (56-byte groups, 256-byte aligned) host -> device
    # (bz.cu io_layout / run_batch)
    # (the round plans stay resident on the device between runs of the same
    # shape -- bz.cu run_batch -- so a repeated run uploads records only)
    record = (8 + 3 * 8 * m + 4 * (m + 1) + 15) // 16 * 16
    d2h = 0
    for (g, L, U) in rep.bounds_trace:
        h2d += record
        d2h += record

    if rank != 0:
        if distributed:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    # ---- roofline of the dominant launch: the tensor-core launch that runs
    # rounds g >= 5 back to back (K5Batch; the library fuses consecutive
    # rounds of one tensor-core kernel).  Its device time is bracketed by
    # CUDA events on the library stream inside the timed steps (bz_round_ms
    # splits it over its rounds by combination count, so the largest round's
    # combinations / its share is the launch's rate); the other kernels of
    # the library and the largest round alone are timed after the region.
    peaks = ctx.measure_int_peaks(w_eff)
    top_ms = statistics.median(g_top_ms)
    achieved = (g_top_combos / world) / (top_ms * 1e-3)
    fused = [r for r in st.rounds if r.combinations >= 1e7 * 0.999]
    fused_g = (min(r.g for r in fused), max(r.g for r in fused)) if fused else (0, 0)
    q_kernel = w_eff <= 4 and n_eff <= 128
    # MACs per combination: algorithmic = the stored columns of one codeword
    # (its dot product, SURVEY.md 8(d) with identity elision); issued = the
    # K the kernel runs (issued_macs)
    macs_alg = n_eff
    macs_issued = issued_macs(w_eff)
    mac_rate = peaks["mxf4_mac_per_s"]
    peak_alg = mac_rate / macs_alg
    peak_issued = mac_rate / macs_issued
    popc_peak = peaks["popc_per_s"] / w_eff
    g_top = max(st.rounds, key=lambda r: r.combinations).g

    # the round as the run meets it: the L and U the previous round left
    prev = [t for t in st.trace if t[0] == g_top - 1]
    l_prev, u_prev = (prev[0][1], prev[0][2]) if prev else (0, 1 << 30)

    def engine_rate(engine_name):
        ctx.set_engine(engine_name)
        ms = []
        for _ in range(3):
            ctx.round(g_top, l_prev, u_prev, local, world)
            ms.append(ctx.last_kernel_ms())
        ctx.set_engine(cfg.engine)
        return (g_top_combos / world) / (statistics.median(ms) * 1e-3)

    alone_achieved = engine_rate(cfg.engine)
    k5_achieved = engine_rate("mxf4")
    k1_achieved = engine_rate("popc")
    # the same launch without elision (full n-column rows)
    ctx.set_elision(False)
    backend.load(gs, n)
    full_rate = engine_rate(cfg.engine)
    w_full = w32
    full_kernel = "K5q" if (w_full <= 4 and n <= 128) else "K5"
    macs_full_issued = issued_macs(w_full)
    ctx.set_elision(True)
    backend.load(gs, n)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    kname = (f"k4_round_umma<{w_eff},true,4> = K5q, rounds g={fused_g[0]}..{fused_g[1]} in one "
             f"launch (tcgen05.mma kind::mxf4nvf4 block16, two codewords as bytes of one fp32 "
             f"accumulator)"
             if q_kernel else
             f"k4_round_umma<{w_eff},true,1> = K5, rounds g={fused_g[0]}..{fused_g[1]} in one "
             f"launch (tcgen05.mma kind::mxf4)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "e2m1 tensor (fp32 acc) / u32", "data": "synthetic",
        "config": {"workload": WORKLOAD if args.config == "cfg5" else args.config,
                   "k": k, "n": n, "m": m, "d": rep.distance, "g_final": rep.g_reached,
                   "combinations_per_step": int(combos_all / args.steps),
                   "engine": cfg.engine,
                   "identity_elision": bool(mask),
                   "parallelism": f"rank-space shards x{world}",
                   "l2": "flushed (256 MiB memset) before every timed step; working set "
                         "(rows, prefix table, suffix tables) is L2/shared-memory resident"},
        "wall_time_to_d_s": e2e_s,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "wall_s": e2e_s},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clock,
        "roofline": {"bound": "tensor", "achieved": achieved / 1e9, "peak": peak_alg / 1e9,
                     "unit": "Gcombinations/s", "frac": achieved / peak_alg,
                     "frac_issued": achieved / peak_issued,
                     "macs_per_combination": {"algorithmic": macs_alg, "issued": macs_issued},
                     "traffic": traffic,
                     "kernel": kname,
                     "peak_source": f"live microbenchmark: tcgen05.mma kind::mxf4 M128xN240xK64 "
                                    f"{peaks['mxf4_mac_per_clk_sm']:.0f} MACs/clk/SM, "
                                    f"{mac_rate / 1e15:.2f} PMAC/s / {macs_alg} algorithmic "
                                    f"MACs per combination (the stored columns; the kernel "
                                    f"issues {macs_issued})",
                     "popc_roofline": popc_peak / 1e9,
                     "frac_of_popc_roofline": achieved / popc_peak,
                     "identity_elision": {
                         "on": bool(mask), "gamma_mask": mask, "stored_columns": n_eff,
                         "words": w_eff,
                         "note": "rows of Gammas with a unit column per row are stored without "
                                 "those k columns and every weight gets +g (exact)"},
                     "without_elision": {
                         "kernel": full_kernel, "achieved": full_rate / 1e9,
                         "peak": mac_rate / n / 1e9, "frac": full_rate / (mac_rate / n),
                         "frac_issued": full_rate / (mac_rate / macs_full_issued),
                         "macs_per_combination": {"algorithmic": n,
                                                  "issued": macs_full_issued}}},
        "largest_round_alone": {"kernel": f"{'K5q' if q_kernel else 'K5'} round g={g_top} in its own "
                                          f"launch", "achieved": alone_achieved / 1e9,
                                "peak": peak_alg / 1e9, "unit": "Gcombinations/s",
                                "frac": alone_achieved / peak_alg,
                                "frac_issued": alone_achieved / peak_issued},
        "k5_mxf4": {"kernel": f"k4_round_umma<{w_eff},true,1> round g={g_top} "
                              f"(tcgen05.mma kind::mxf4, one codeword per accumulator)",
                    "achieved": k5_achieved / 1e9, "peak": peak_alg / 1e9,
                    "unit": "Gcombinations/s", "frac": k5_achieved / peak_alg},
        "k1_popc": {"kernel": f"k1_round_min<{w_eff},2> round g={g_top} (XOR+POPC)",
                    "achieved": k1_achieved / 1e9, "peak": popc_peak / 1e9,
                    "unit": "Gcombinations/s", "frac": k1_achieved / popc_peak,
                    "peak_source": f"live microbenchmark: {peaks['popc_per_clk_sm']:.1f} POPC/clk/SM"
                                   f" / {w_eff} POPC per combination",
                    "alu_peak": peaks["lop3_per_s"] / (2 * w_eff) / 1e9},
    }
    rounds = [{"g": r.g, "combinations": r.combinations, "kernel_ms": r.kernel_ms}
              for r in st.rounds]
    line["rounds"] = rounds
    if args.config == "cfg5" and not args.no_extra and world == 1:
        line["cfg5_other_seeds"] = other_seeds(args, cfg, local, flush)
        line["section6_C1"] = section6_c1(cfg)
        line["configs_1_3"] = configs_wall(cfg)
        line["cfg4"] = cfg4_side(ctx, peaks)
        backend.load(gs, n)
        line["shards_on_one_gpu"] = shard_times(ctx, st, engine.start_state(gs, n, k, cfg).U, m,
                                                flush, barrier)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(G, gs, args.cpu_sample_g)
    print(json.dumps(line), flush=True)
    if distributed:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

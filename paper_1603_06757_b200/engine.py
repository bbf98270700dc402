"""Brouwer-Zimmermann outer loop with the enumeration on the GPU.

Drop-in for the reference's ``mindist.engine`` (pkg/src/mindist/engine.py):
``minimum_distance(G, config) -> DistanceReport`` keeps its signature and
its semantics -- Gamma family from ``build_gamma_set`` (gf2.py:168-199),
bounds (1, n-k+1) (engine.py:90-94), the per-round lower bound
(m-1)(g+1) + max(0, g+1-k+k_m) with the all-full-rank convention of
``_line7_args`` (engine.py:106-116), the loop ``while g <= k and L < U``
with the ``max_g`` cap, one ``(g, L, U)`` trace entry per round, the
``progress`` callback and ``Interrupted`` carrying a resumable partial
report (engine.py:157-220).

What changes is the inside of a round.  The reference runs one strategy
call per Gamma_j (engine.py:208-211); here the whole round -- every
g-combination of every Gamma_j -- is ONE call into the sm_100a kernel
(``bz_round``), which returns per-Gamma minima that the loop folds into U
in Gamma order exactly as the reference does.  Clipping by the running U is
the only thing the reference passes between the passes of a round
(engine.py:7-9), so a round-level call yields the same U, L and trace.

Multi-GPU: with ``EngineConfig(distributed=True)`` each process (one per
GPU) enumerates its shard of every round and the shards' results are
combined by one collective per round (parallel.py).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from math import comb

import numpy as np

from . import _native
from .enumeration import EnumerationResult, PassCount, family_words
from .errors import InvalidArity, InvalidDimensions, Interrupted, TooLarge
from .gf2 import BitMatrix, GammaSet, build_gamma_set
from .parallel import LocalComm, combine_rounds

STRATEGIES = ("gpu",)

DEFAULT_MAX_G = 16

STATUS_EXACT = "exact"
STATUS_UPPER_BOUND_ONLY = "upper_bound_only"
STATUS_INTERRUPTED = "interrupted"


@dataclass(frozen=True)
class Bounds:
    lower: int
    upper: int


@dataclass
class Counters:
    combinations: int = 0
    row_additions: int = 0
    row_accesses: int = 0

    def add(self, res: EnumerationResult) -> None:
        self.combinations += res.combinations
        self.row_additions += res.row_additions
        self.row_accesses += res.row_accesses


@dataclass
class EngineConfig:
    """Reference fields (engine.py:57-67) plus the GPU placement.

    ``s``, ``unroll``, ``workers`` and ``memory_budget`` configure the
    reference's CPU strategies and are accepted but unused here.
    ``device`` defaults to $LOCAL_RANK (or 0); ``distributed`` shards every
    round over the torch.distributed default group."""

    strategy: str = "gpu"
    s: int = 3
    unroll: int = 2
    workers: int = 1
    memory_budget: int = 256 * 1024 * 1024
    max_g: int = DEFAULT_MAX_G
    start_g: int = 1
    start_upper: int | None = None
    progress: object = None  # callable(g, L, U) after each round
    device: int | None = None
    distributed: bool = False
    # in-round early exit: stop a round once U reaches the previous L (the
    # trace is the same; only that round's `combinations` count drops below
    # the reference's m*C(k,g)).  Off by default, so every pass runs to
    # completion and the counters are schedule-independent, as the
    # reference's are (enumeration.py:21-24).  Batched rounds past
    # termination stop at once either way (their results are discarded).
    early_exit: bool = False
    # consecutive rounds with at most this many combinations in total (per
    # rank) run as one batch (one launch sequence, one synchronisation, one
    # exchange); 0 disables batching
    batch_combinations: int = 2_000_000_000
    # on a single device the batch may run far ahead: each batched round
    # starts on the device from the U its predecessor ended with and exits
    # at once if that U already meets its L (the run had terminated), so a
    # speculative round costs a launch, not its enumeration
    batch_combinations_single: int = 100_000_000_000
    # multi-GPU: share each round's running minimum across ranks through
    # peer memory (kernels stop as soon as any rank meets the bound), which
    # lets the batch run ahead there too
    shared_bound: bool = True
    engine: str = "auto"     # "auto" | "mxf4q" | "mxf4" | ... | "popc" (kernel; same results)
    elide_identity: bool = True  # drop each full-rank Gamma's identity columns (+g; exact)
    # one rank: the loop itself runs natively (bz_advance: the same batch
    # rule and fold, one library call per batch); False keeps it in Python
    native_loop: bool = True


@dataclass
class RoundStat:
    g: int
    combinations: int
    kernel_ms: float
    wall_ms: float


@dataclass
class DistanceReport:
    distance: int
    status: str
    g_reached: int
    n: int
    k: int
    m: int
    k_m: int
    pivot_sets: tuple[tuple[int, ...], ...]
    bounds_trace: list[tuple[int, int, int]] = field(default_factory=list)
    counters: Counters = field(default_factory=Counters)
    store_build_additions: int = 0
    elapsed: float = 0.0
    rounds: list[RoundStat] = field(default_factory=list)

    @property
    def exact(self) -> bool:
        return self.status == STATUS_EXACT


def initial_bounds(n: int, k: int) -> Bounds:
    """(1, n-k+1): trivial lower bound and the Singleton upper bound."""
    if not 0 < k <= n:
        raise InvalidDimensions(f"need 0 < k <= n, got k={k}, n={n}")
    return Bounds(1, n - k + 1)


def lower_bound_update(g: int, m: int, k: int, k_m: int) -> int:
    """Certified lower bound after round g: (m-1)(g+1) + max(0, g+1-k+k_m)."""
    if m < 1:
        raise InvalidDimensions(f"need m >= 1, got {m}")
    if not 0 <= k_m <= k:
        raise InvalidDimensions(f"need 0 <= k_m <= k, got k_m={k_m}, k={k}")
    return (m - 1) * (g + 1) + max(0, g + 1 - k + k_m)


def line7_args(gs: GammaSet, k: int) -> tuple[int, int]:
    """(m, k_m) for lower_bound_update: a deficient remainder counts as the
    m-th matrix with its rank; otherwise the last full matrix plays the
    remainder of rank k (engine.py:106-116)."""
    if gs.remainder_rank > 0:
        return gs.full_rank_count + 1, gs.remainder_rank
    return gs.full_rank_count, k


class GpuRounds:
    """Round backend on one CUDA device (the product path)."""

    def __init__(self, config: EngineConfig, comm):
        dev = config.device
        if dev is None:
            dev = int(os.environ.get("LOCAL_RANK", "0"))
        self.ctx = _native.context(dev)
        self.ctx.set_engine(config.engine)
        if self.ctx.elision != config.elide_identity:
            self.ctx.set_elision(config.elide_identity)
        self.ctx.set_early_exit(config.early_exit)
        self.comm = comm
        # multi-GPU: the shared bound mirror (rank 0's array, mapped into
        # every rank over CUDA IPC), set up once per context and world
        self.shared = False
        if comm.world > 1 and config.shared_bound:
            key = ("shared", comm.world)
            if getattr(self.ctx, "shared_key", None) != key:
                handle = self.ctx.shared_bound_export() if comm.rank == 0 else None
                handle = comm.broadcast_bytes(handle)
                self.ctx.shared_bound_open(None if comm.rank == 0 else handle)
                self.ctx.shared_key = key
                self.ctx.shared_epoch = 0
            self.shared = True

    def begin_run(self) -> None:
        """A new minimum-distance run: a fresh shared-bound tag (every rank
        counts its runs alike)."""
        if self.shared:
            self.ctx.shared_epoch += 1
            self.ctx.shared_bound_epoch(self.ctx.shared_epoch)

    def load(self, gs: GammaSet, n: int) -> None:
        self.ctx.load(family_words(gs.gammas, n), n)

    def run(self, g: int, lower_prev: int, upper: int):
        mins, combos = self.ctx.round(g, lower_prev, upper, self.comm.rank, self.comm.world)
        kernel_ms = self.ctx.last_kernel_ms()
        adds, accs = self.ctx.counters(1)
        m = len(mins)
        mins, sums = self.comm.combine(mins, combos + adds[0] + accs[0])
        return mins, [PassCount(*sums[j::m]) for j in range(m)], kernel_ms

    def run_batch(self, g0: int, lower_prevs: list[int], upper: int):
        """Rounds g0.. in one call, each sharded over the ranks like a single
        round, then one exchange for all of them: [(mins, combos)] per round
        and the batch's kernel ms."""
        res = self.ctx.rounds(g0, lower_prevs, upper, self.comm.rank, self.comm.world)
        ms = self.ctx.round_ms(len(lower_prevs))
        adds, accs = self.ctx.counters(len(lower_prevs))
        if self.comm.world == 1:
            return [(mn, [PassCount(c, a, x) for c, a, x in zip(cb, ad, ac)])
                    for (mn, cb), ad, ac in zip(res, adds, accs)], ms
        res = [(mn, cb + ad + ac) for (mn, cb), ad, ac in zip(res, adds, accs)]
        out = []
        for mn, sums in combine_rounds(self.comm, res):
            m = len(mn)
            out.append((mn, [PassCount(*sums[j::m]) for j in range(m)]))
        return out, ms


def make_backend(config: EngineConfig, comm):
    """Seam for tests (cf. the reference's monkeypatch of enumerate_basic,
    t/test_engine.py:165-208): returns the object that runs the rounds."""
    return GpuRounds(config, comm)


def _make_comm(config: EngineConfig):
    if not config.distributed:
        return LocalComm()
    from .parallel import TorchComm

    return TorchComm()


@dataclass
class LoopState:
    """Mutable state of Algorithm 1 between rounds."""

    L: int
    U: int
    g: int
    g_reached: int
    status: str = STATUS_EXACT
    counters: Counters = field(default_factory=Counters)
    trace: list = field(default_factory=list)
    rounds: list = field(default_factory=list)


def start_state(gs: GammaSet, n: int, k: int, config: EngineConfig) -> LoopState:
    m_arg, km_arg = line7_args(gs, k)
    start = initial_bounds(n, k)
    L, U = start.lower, start.upper
    if config.start_upper is not None:
        U = min(U, config.start_upper)
    g = max(1, config.start_g)
    if g > 1:
        L = lower_bound_update(g - 1, m_arg, k, km_arg)
    return LoopState(L=L, U=U, g=g, g_reached=g - 1)


def lightest_row(gs: GammaSet) -> int:
    """Weight of the lightest row of any Gamma (every row is a codeword, so
    U never exceeds it once round 1 is in); cached on the family."""
    w = getattr(gs, "_lightest_row", None)
    if w is None:
        w = min(int(np.bitwise_count(gm.words64()).sum(axis=1).min()) for gm in gs.gammas)
        object.__setattr__(gs, "_lightest_row", w)  # frozen dataclass: a cache only
    return w


def _run_rounds_native(backend, gs: GammaSet, k: int, config: EngineConfig, st: LoopState,
                       m_arg: int, km_arg: int) -> None:
    """run_rounds on one rank through bz_advance: the batch rule and the
    fold of the Python loop below, one library call per batch (the loop is
    on the timed path of every run)."""
    ctx = backend.ctx
    backend.begin_run()
    budget = (max(config.batch_combinations, config.batch_combinations_single)
              if config.batch_combinations > 0 else 0)
    u_rows = lightest_row(gs)
    state = np.array([st.g, st.L, st.U, st.g_reached, 0], dtype=np.int32)
    progress = config.progress
    trace, rounds, ctr = st.trace, st.rounds, st.counters
    while True:
        t0 = time.perf_counter()
        recs = ctx.advance(m_arg, km_arg, config.max_g, u_rows, budget, state)
        wall = (time.perf_counter() - t0) * 1e3
        # st follows the records (an interrupt between two calls leaves it
        # at the last round folded in, as the Python loop does)
        for g, L, U, _, c, a, x, ms, _ in recs:
            ctr.combinations += c
            ctr.row_additions += a
            ctr.row_accesses += x
            rounds.append(RoundStat(g, c, ms, wall))
            wall = 0.0
            trace.append((g, L, U))
            st.g_reached = g
            st.g, st.L, st.U = g + 1, L, U
            if progress is not None:
                progress(g, L, U)
        status = int(state[4])
        if status == _native.BZ_LOOP_MAX_G:
            st.status = STATUS_UPPER_BOUND_ONLY
        if status != _native.BZ_LOOP_RUNNING:
            break


def run_rounds(backend, gs: GammaSet, k: int, config: EngineConfig, st: LoopState) -> None:
    """The loop of engine.py:204-217 with one device round per g: fold the
    per-Gamma minima into U in Gamma order, then raise L, append (g, L, U),
    report progress.  ``backend`` already holds the family on the device.

    (This loop sits inside every timed run: it keeps to plain locals and
    arithmetic -- the L formula inlined, counters summed once per round.)"""
    m_arg, km_arg = line7_args(gs, k)
    if (config.native_loop and isinstance(backend, GpuRounds) and backend.comm.world == 1
            and not backend.shared):
        return _run_rounds_native(backend, gs, k, config, st, m_arg, km_arg)
    m = gs.matrix_count
    batch_ok = config.batch_combinations > 0 and hasattr(backend, "run_batch")
    if hasattr(backend, "begin_run"):
        backend.begin_run()
    max_g = config.max_g
    progress = config.progress
    g, L, U = st.g, st.L, st.U
    trace, rounds, ctr = st.trace, st.rounds, st.counters

    def lower(gg: int) -> int:  # lower_bound_update (engine.py:97-103)
        return (m_arg - 1) * (gg + 1) + max(0, gg + 1 - k + km_arg)

    queued: list = []  # precomputed (g, mins, combos, kernel_ms) of a batch
    qi = 0
    # A batch need not run past the round where the loop must stop: round g
    # runs only while L(g - 1) < U, and every row of every Gamma is a
    # codeword, so U never exceeds the lightest row once round 1 is in.
    # (Only the batch length depends on this; results do not.)
    u_rows = min(U, lightest_row(gs))
    try:
        while g <= k and L < U:
            if g > max_g:
                st.status = STATUS_UPPER_BOUND_ONLY
                break
            tr = time.perf_counter()
            if qi == len(queued) and batch_ok:
                # the next rounds whose total size fits the batch budget (per
                # rank: a batch is sharded like a round)
                world = getattr(getattr(backend, "comm", None), "world", 1)
                ahead = world == 1 or getattr(backend, "shared", False)
                budget = (max(config.batch_combinations * world, config.batch_combinations_single)
                          if ahead else config.batch_combinations * world)
                count, total = 0, 0
                top = min(k, max_g)
                u_cap = min(U, u_rows)
                while g + count <= top and (count == 0 or lower(g + count - 1) < u_cap):
                    c = m * comb(k, g + count)
                    if total + c > budget:
                        break
                    total += c
                    count += 1
                if count >= 2:
                    lps = [L] + [lower(g + i - 1) for i in range(1, count)]
                    res, batch_ms = backend.run_batch(g, lps, U)
                    per_round = isinstance(batch_ms, list)
                    queued = []
                    qi = 0
                    for i, (mn, cb) in enumerate(res):
                        ms = (batch_ms[i] if per_round else
                              batch_ms * ((m * comb(k, g + i)) / total if total else 0.0))
                        queued.append((g + i, mn, cb, ms))
            if qi < len(queued) and queued[qi][0] == g:
                _, mins, combos, kernel_ms = queued[qi]
                qi += 1
            else:
                queued, qi = [], 0
                mins, combos, kernel_ms = backend.run(g, L, U)
            rc = ra = rx = 0
            for mn, cnt in zip(mins, combos):
                if mn < U:
                    U = mn
                if isinstance(cnt, PassCount):
                    rc += cnt.combinations
                    ra += cnt.additions
                    rx += cnt.accesses
                else:
                    rc += cnt
                    ra += cnt
                    rx += cnt
            ctr.combinations += rc
            ctr.row_additions += ra
            ctr.row_accesses += rx
            rounds.append(RoundStat(g, rc, kernel_ms, (time.perf_counter() - tr) * 1e3))
            L = lower(g)
            trace.append((g, L, U))
            st.g_reached = g
            st.L, st.U = L, U
            if progress is not None:
                progress(g, L, U)
            g += 1
            st.g = g
    finally:
        st.g, st.L, st.U = g, L, U


def minimum_distance(G: BitMatrix, config: EngineConfig | None = None) -> DistanceReport:
    """Exact minimum weight of the code generated by G (Algorithm 1).

    Raises RankDeficient for rank-deficient input.  With ``max_g`` cutting
    the loop short the distance is only an upper bound (status says so).
    On KeyboardInterrupt, Interrupted carries the partial report; rerun
    with start_g = g_reached + 1 and start_upper = distance to continue."""
    config = config or EngineConfig()
    if config.strategy not in STRATEGIES:
        raise InvalidArity(f"unknown strategy {config.strategy!r} (this build: {STRATEGIES})")
    t0 = time.perf_counter()
    gs = build_gamma_set(G)
    k, n = G.num_rows, G.num_cols
    st = start_state(gs, n, k, config)

    def report(status: str) -> DistanceReport:
        return DistanceReport(
            distance=st.U, status=status, g_reached=st.g_reached, n=n, k=k,
            m=gs.matrix_count, k_m=gs.remainder_rank, pivot_sets=gs.pivot_sets,
            bounds_trace=st.trace, counters=st.counters, store_build_additions=0,
            elapsed=time.perf_counter() - t0, rounds=st.rounds)

    try:
        if st.g <= k and st.L < st.U and st.g <= config.max_g:
            backend = make_backend(config, _make_comm(config))
            lock = getattr(getattr(backend, "ctx", None), "lock", None)
            if lock is None:
                backend.load(gs, n)
                run_rounds(backend, gs, k, config, st)
            else:
                # the device context is per process: hold it across the load
                # and every round, so concurrent calls on distinct matrices
                # never run on each other's family
                with lock:
                    backend.ctx.set_engine(config.engine)
                    backend.ctx.set_early_exit(config.early_exit)
                    if backend.ctx.elision != config.elide_identity:
                        backend.ctx.set_elision(config.elide_identity)
                    backend.load(gs, n)
                    run_rounds(backend, gs, k, config, st)
        elif st.g <= k and st.L < st.U:
            st.status = STATUS_UPPER_BOUND_ONLY
    except KeyboardInterrupt:
        raise Interrupted(report(STATUS_INTERRUPTED)) from None
    return report(st.status)


# ---------------------------------------------------------------------------
# report text: key=value lines plus one "g=.. L=.. U=.." line per completed
# round -- the reference's checkpoint format (engine.py:245-285).


def brute_force_distance(G: BitMatrix, max_k: int = 28, device: int | None = None) -> int:
    """Minimum weight over all 2^k - 1 nonzero codewords (engine.py:223-237),
    on the GPU (bz_brute_force: Gray-code order, one row XOR per message).
    Same cap semantics as the reference (TooLarge above max_k); the device
    kernel lifts the practical limit to k = 48."""
    k = G.num_rows
    if k > max_k:
        raise TooLarge(f"k={k} exceeds brute-force cap {max_k}")
    dev = device if device is not None else int(os.environ.get("LOCAL_RANK", "0"))
    ctx = _native.context(dev)
    words = np.ascontiguousarray(G.with_word_width(64).to_numpy(), dtype=np.uint64)
    with ctx.lock:
        d, _ = ctx.brute_force(words, G.num_cols, max_k)
    return d


def format_report(r: DistanceReport) -> str:
    rate = r.counters.combinations / r.elapsed if r.elapsed > 0 else 0.0
    lines = [f"status={r.status}", f"n={r.n}", f"k={r.k}", f"distance={r.distance}",
             f"g_reached={r.g_reached}", f"m={r.m}", f"k_m={r.k_m}",
             f"combinations={r.counters.combinations}",
             f"row_additions={r.counters.row_additions}",
             f"row_accesses={r.counters.row_accesses}",
             f"store_build_additions={r.store_build_additions}",
             f"elapsed_s={r.elapsed:.3f}", f"combos_per_sec={rate:.0f}"]
    lines += [f"g={g} L={L} U={U}" for g, L, U in r.bounds_trace]
    return "\n".join(lines) + "\n"


_INT_KEYS = ("n", "k", "distance", "g_reached", "m", "k_m", "combinations",
             "row_additions", "row_accesses", "store_build_additions")


def parse_report(text: str) -> dict:
    out: dict = {"bounds_trace": []}
    for raw in text.splitlines():
        line = raw.strip()
        if not line:
            continue
        if line.startswith("g=") and " L=" in line:
            kv = dict(p.split("=", 1) for p in line.split())
            out["bounds_trace"].append((int(kv["g"]), int(kv["L"]), int(kv["U"])))
        elif "=" in line:
            key, value = line.split("=", 1)
            out[key] = value
    for key in _INT_KEYS:
        if key in out:
            out[key] = int(out[key])
    return out

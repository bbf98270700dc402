"""CPU oracle for the Brouwer-Zimmermann enumeration path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py (its cpu_baseline leg and ``--impl reference``) import this module,
and only as the checker or as the timed CPU baseline.  The product package
``paper_1603_06757_b200`` never imports it and has no CPU fallback.

What it restates (paths relative to the reference's pkg/src/mindist/):

* ``min_weight`` / ``histogram`` -- ``enumerate_stack`` (enumeration.py:128-178)
  in C (bz_oracle.c), multithreaded; ``brute_distance`` -- ``brute_force_distance``
  (engine.py:223-237).
* ``gamma_family`` -- ``reduce_on_columns`` + ``build_gamma_set``
  (gf2.py:133-199): greedy Gauss-Jordan on the still-unused columns with
  leftmost pivots, each pass starting from the previous reduced matrix.
* ``minimum_distance`` -- the Algorithm-1 loop of ``minimum_distance``
  (engine.py:157-220) with ``initial_bounds`` (:90-94),
  ``lower_bound_update`` (:97-103) and ``_line7_args`` (:106-116).
* ``enumerate_chunks`` -- pure-Python walk over the device work plan
  (bz_plan, include/bz.h) used to check that shards partition the rank space;
  ``expected_counters`` -- the row additions / accesses the device counts
  for that plan (bz_counters), restating the reference's counter semantics
  (enumeration.py:19-24, :254-302).

Pinned by tests/test_oracle.py against tests/golden/goldens.json and
tests/golden/cfg5_seed7.json, which tests/golden/make_golden.py produced
by running the reference package itself, and against the reference's own
known answers (t/test_enumeration.py:65-76, t/test_engine.py:88-104).
"""

from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from math import comb

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libbzoracle.so")

_lib = None


def build() -> str:
    """Compile bz_oracle.c (idempotent)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.bzo_min_stack.argtypes = [u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, i32p, u64p]
        L.bzo_hist_stack.argtypes = [u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, u64p, ctypes.c_int]
        L.bzo_brute.argtypes = [u64p, ctypes.c_int, ctypes.c_int, i32p]
        L.bzo_max_threads.argtypes = []
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().bzo_max_threads())


# ---------------------------------------------------------------------------
# row images


def words64(rows: list[int], n: int) -> np.ndarray:
    """(k, ceil(n/64)) uint64 image, bit j = column j (gf2.py:74-79)."""
    w64 = -(-n // 64)
    out = np.zeros((len(rows), w64), dtype=np.uint64)
    mask = (1 << 64) - 1
    for i, r in enumerate(rows):
        for w in range(w64):
            out[i, w] = (r >> (64 * w)) & mask
    return out


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def min_weight(rows: list[int], n: int, g: int, threads: int = 0) -> tuple[int, int]:
    """(unclipped minimum weight, combinations) over all g-combinations."""
    img = np.ascontiguousarray(words64(rows, n))
    out_min = np.zeros(1, dtype=np.int32)
    out_c = np.zeros(1, dtype=np.uint64)
    rc = lib().bzo_min_stack(_ptr(img, ctypes.c_uint64), len(rows), img.shape[1], g,
                             threads, _ptr(out_min, ctypes.c_int32),
                             _ptr(out_c, ctypes.c_uint64))
    if rc:
        raise ValueError(f"bzo_min_stack failed ({rc}) for k={len(rows)} g={g}")
    return int(out_min[0]), int(out_c[0])


def histogram(rows: list[int], n: int, g: int, threads: int = 0) -> np.ndarray:
    img = np.ascontiguousarray(words64(rows, n))
    hist = np.zeros(n + 1, dtype=np.uint64)
    rc = lib().bzo_hist_stack(_ptr(img, ctypes.c_uint64), len(rows), img.shape[1], g,
                              threads, _ptr(hist, ctypes.c_uint64), n + 1)
    if rc:
        raise ValueError(f"bzo_hist_stack failed ({rc})")
    return hist


def brute_distance(rows: list[int], n: int) -> int:
    img = np.ascontiguousarray(words64(rows, n))
    out = np.zeros(1, dtype=np.int32)
    rc = lib().bzo_brute(_ptr(img, ctypes.c_uint64), len(rows), img.shape[1],
                         _ptr(out, ctypes.c_int32))
    if rc:
        raise ValueError(f"bzo_brute failed ({rc})")
    return int(out[0])


# ---------------------------------------------------------------------------
# Gamma family (gf2.py:133-199), restated on Python ints


def reduce_columns(rows: list[int], n: int, cols) -> tuple[list[int], list[int]]:
    work = list(rows)
    k = len(work)
    pivots: list[int] = []
    top = 0
    for col in cols:
        bit = 1 << col
        hit = next((r for r in range(top, k) if (work[r] >> col) & 1), None)
        if hit is None:
            continue
        work[top], work[hit] = work[hit], work[top]
        pv = work[top]
        for r in range(k):
            if r != top and work[r] & bit:
                work[r] ^= pv
        pivots.append(col)
        top += 1
        if top == k:
            break
    return work, pivots


def gamma_family(rows: list[int], n: int):
    """(gammas, pivot_sets, full_rank_count, remainder_rank)."""
    k = len(rows)
    gammas, pivsets = [], []
    used: set[int] = set()
    cur = list(rows)
    rem = 0
    while len(used) < n:
        red, piv = reduce_columns(cur, n, [c for c in range(n) if c not in used])
        rank = len(piv)
        if not gammas and rank < k:
            raise ValueError(f"rank {rank} < {k}")
        gammas.append(red)
        pivsets.append(tuple(piv))
        if rank == k:
            used.update(piv)
            cur = red
            continue
        if rank == 0:
            gammas.pop()
            pivsets.pop()
        else:
            rem = rank
        break
    full = len(gammas) - (1 if rem else 0)
    return gammas, pivsets, full, rem


def draw_code(k: int, n: int, seed: int, target: tuple[int, int]) -> list[int]:
    """Rows of SURVEY.md Appendix A's seeded draw, restated here so that
    bench.py's CPU arm builds its input without the product package:
    ``random.Random(seed)``, one ``getrandbits(n)`` per row, the whole matrix
    redrawn (same RNG stream) until the information-set family has
    ``target`` = (full-rank count, remainder rank).  Equal to
    ``paper_1603_06757_b200.configs.draw_code`` (tests/test_oracle.py)."""
    import random

    rng = random.Random(seed)
    while True:
        rows = [rng.getrandbits(n) for _ in range(k)]
        try:
            _, _, full, rem = gamma_family(rows, n)
        except ValueError:  # rank deficient
            continue
        if (full, rem) == tuple(target):
            return rows


def minimum_distance(rows: list[int], n: int, threads: int = 0, max_g: int = 16,
                     start_g: int = 1, start_upper: int | None = None,
                     round_fn=None) -> dict:
    """Algorithm 1 (engine.py:157-220) on the C enumerator.

    ``round_fn(gammas, g, U) -> list[(min, combos)]`` may replace the
    per-round enumeration (used by the multi-rank tests)."""
    k = len(rows)
    gammas, pivsets, full, rem = gamma_family(rows, n)
    m_arg, km_arg = (full + 1, rem) if rem > 0 else (full, k)

    def lbu(g):
        return (m_arg - 1) * (g + 1) + max(0, g + 1 - k + km_arg)

    L, U = 1, n - k + 1
    if start_upper is not None:
        U = min(U, start_upper)
    g = max(1, start_g)
    if g > 1:
        L = lbu(g - 1)
    trace, combos, g_reached, status = [], 0, g - 1, "exact"
    while g <= k and L < U:
        if g > max_g:
            status = "upper_bound_only"
            break
        if round_fn is not None:
            res = round_fn(gammas, g, U)
        else:
            res = [min_weight(gm, n, g, threads) for gm in gammas]
        for mn, c in res:
            U = min(U, mn)
            combos += c
        L = lbu(g)
        trace.append((g, L, U))
        g_reached = g
        g += 1
    return dict(distance=U, status=status, g_reached=g_reached, m=len(gammas),
                k_m=rem, pivot_sets=[list(p) for p in pivsets], bounds_trace=trace,
                combinations=combos)


# ---------------------------------------------------------------------------
# walking the device work plan (small sizes, pure Python)


def colex_unrank(r: int, q: int, ell: int) -> list[int]:
    """q-subset of [0, ell) with colex rank r (sum_i C(c_i, i))."""
    out = []
    c = ell - 1
    for i in range(q, 0, -1):
        while comb(c, i) > r:
            c -= 1
        r -= comb(c, i)
        out.append(c)
        c -= 1
    return sorted(out)


def enumerate_chunks(gammas: list[list[int]], k: int, g: int, groups, nchunks: int,
                     shard: int, nshards: int, hist_bins: int | None = None):
    """Visit every combination of the chunks owned by `shard` exactly as the
    device kernel does (chunk c -> shard c % nshards; lane-major prefix
    ranges of ppl colex ranks of (g-1-depth)-subsets of [0, ell), plus ell;
    then every depth-subset of the suffix rows [suffix_floor, k)).  Returns
    (per-gamma minima, per-gamma combos, list of visited combos)."""
    m = len(gammas)
    mins = [None] * m
    cnt = [0] * m
    seen = []
    starts = [gr[0] for gr in groups]
    for chunk in range(shard, nchunks, nshards):
        gi = max(i for i, s in enumerate(starts) if s <= chunk)
        begin, nprefix, gamma, ell, ppl, _, depth, lanes, spc, nsb, sfloor, sl = groups[gi]
        merged = depth >= 3 and sl == 0  # K5 family: (g - depth)-subsets of [0, ell + 1)
        if not merged:
            lanes //= sl  # K1: prefix blocks per warp (suffix lanes share a block)
        local = chunk - begin
        pb, sb = divmod(local, nsb)
        rows = gammas[gamma]
        sufs = suffix_order(ell, k, depth, sfloor)
        if depth >= 3:
            sufs = sufs[sb * spc:(sb + 1) * spc]
        for lane in range(lanes):
            first = (pb * lanes + lane) * ppl
            for p in range(first, min(first + ppl, nprefix)):
                if g == 1:
                    prefix = []
                elif merged:
                    prefix = colex_unrank(p, g - depth, ell + 1)
                else:
                    prefix = colex_unrank(p, g - 1 - depth, ell) + [ell]
                acc = 0
                for i in prefix:
                    acc ^= rows[i]
                for suf in sufs:
                    w = acc
                    for e in suf:
                        w ^= rows[e]
                    w = w.bit_count()
                    mins[gamma] = w if mins[gamma] is None else min(mins[gamma], w)
                    cnt[gamma] += 1
                    seen.append((gamma, tuple(prefix + list(suf))))
    return mins, cnt, seen


def _walk_cost(first: int, cnt: int, q: int, ell: int, merged: bool = False) -> int:
    """Row additions of one prefix walker over colex ranks [first,
    first+cnt): the init folds R[ell] and the q rows of the first subset (q
    additions), each colex successor adds 2 prefix-XOR rows, 3 when the low
    run of the subset's bits is longer than one (bz_kernels.cuh Walker).  A
    merged group's prefixes are the (q + 1)-subsets of [0, ell + 1): the same
    q additions for the first one."""
    if cnt <= 0:
        return 0
    cost = max(q, 0)
    if q <= 0 and not merged:
        return cost
    x = 0
    for b in (colex_unrank(first, q + 1, ell + 1) if merged else colex_unrank(first, q, ell)):
        x |= 1 << b
    for _ in range(cnt - 1):
        s = (x & -x).bit_length() - 1
        run = 0
        while (x >> (s + run)) & 1:
            run += 1
        cost += 3 if run >= 2 else 2
        u = x & -x
        v = x + u
        x = v | (((v ^ x) // u) >> 2)
    return cost


def expected_counters(m: int, k: int, g: int, groups, nchunks: int, shard: int = 0,
                      nshards: int = 1):
    """Per-Gamma (row_additions, row_accesses) the device reports
    (bz_counters, include/bz.h) for the chunks of `shard`, from the work
    plan alone: K1 groups (32 lanes, two walkers per lane over the halves of
    its prefix range) and K5/K5q groups (128 lanes, one walker each, every
    stored suffix row of the chunk streamed once per prefix step).  Restates
    the counting of the reference's strategies (enumeration.py:19-24,
    :254-302) for the device's prefix-sum + stored-row decomposition."""
    adds = [0] * m
    accs = [0] * m
    starts = [gr[0] for gr in groups]
    for chunk in range(shard, nchunks, nshards):
        gi = max(i for i, st in enumerate(starts) if st <= chunk)
        begin, nprefix, gamma, ell, ppl, _, depth, lanes, spc, nsb, sfloor, sl = groups[gi]
        q = g - 1 - depth
        local = chunk - begin
        if depth < 3:
            # K1: one warp, 32 / sl prefix blocks (lane-major ranges, walkers
            # A / B on the halves) x sl suffix lanes taking every sl-th
            # first suffix row
            e0 = ell + 1
            per_prefix = comb(k - e0, depth) + (max(0, k - 1 - e0) if depth == 2 else 0)
            maxca = 0
            for lane in range(32):
                blk, s0 = divmod(lane, sl)
                first = (local * (32 // sl) + blk) * ppl
                cnt = max(0, min(ppl, nprefix - first))
                ca = (cnt + 1) >> 1
                cb = cnt - ca
                if lane == 0:
                    maxca = ca
                w = _walk_cost(first, ca, q, ell) + _walk_cost(first + ca, cb, q, ell)
                ninit = (cnt > 0) + (cb > 0)
                if depth == 1:
                    lane_pp = len(range(e0 + s0, k, sl))
                else:
                    firsts = range(e0 + s0, k - 1, sl)
                    lane_pp = sum(k - 1 - e1 for e1 in firsts) + len(firsts)
                if s0:  # the block's walkers are counted on its first lane
                    w = ninit = 0
                adds[gamma] += w + cnt * lane_pp
                accs[gamma] += w + ninit
            accs[gamma] += maxca * per_prefix
        else:
            # K5 / K5q: one CTA, 128 producer rows, tiles of the suffix block
            pb, sb = divmod(local, nsb)
            slice_rows = comb(k - sfloor, depth)
            cols = min(spc, slice_rows - sb * spc)
            bfirst = pb * 128 * ppl
            maxcnt = min(ppl, nprefix - bfirst)
            for r in range(128):
                first = bfirst + r * ppl
                cnt = max(0, min(ppl, nprefix - first))
                w = _walk_cost(first, cnt, q, ell, merged=(sl == 0))
                adds[gamma] += w + cnt * cols
                accs[gamma] += w + (cnt > 0)
            accs[gamma] += maxcnt * cols
    return adds, accs


def suffix_order(ell: int, k: int, depth: int, floor: int | None = None):
    """Suffixes of rows >= floor (default ell + 1) in device order: lex for
    depth 1-2; for depth >= 3 the table order (smallest element descending,
    then the other depth-1 elements lex)."""
    lo = ell + 1 if floor is None else floor
    if depth < 3:
        return list(itertools.combinations(range(lo, k), depth))
    out = []
    for a in range(k - depth, lo - 1, -1):
        out += [(a,) + rest for rest in itertools.combinations(range(a + 1, k), depth - 1)]
    return out


def all_combinations(m: int, k: int, g: int):
    return [(j, c) for j in range(m) for c in itertools.combinations(range(k), g)]

"""Per-(Gamma, g) enumeration on the GPU.

Drop-in for the reference's strategy functions (pkg/src/mindist/
enumeration.py:76-444): ``enumerate_gpu(gamma, g, ubound)`` returns the same
``EnumerationResult`` record (enumeration.py:43-50) with ``min_weight``
clipped to ``ubound`` (enumeration.py:60-64) and ``InvalidArity`` for g
outside 1..k (enumeration.py:67-69).  The work runs in the sm_100a kernel
K1 behind the C ABI (include/bz.h); there is no CPU path.

Counters: ``combinations`` is exact (C(k, g) per pass).  ``row_additions``
and ``row_accesses`` are counted on the device (bz_counters, include/bz.h)
with the reference's meaning (enumeration.py:19-24): one addition per
codeword (its prefix sum combined with its last stored row -- a XOR in K1,
the tensor-core dot product in K5/K5q), K1's partial sums, and the prefix
walkers' updates; accesses are the rows a warp (K1) or CTA (K5/K5q, up to
128 prefixes per stored row load) brings into its working set.  The paper's
point -- many additions per row access -- is their ratio.
"""

from __future__ import annotations

from collections import namedtuple
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvalidArity
from .gf2 import BitMatrix


@dataclass
class EnumerationResult:
    min_weight: int
    combinations: int
    row_additions: int
    row_accesses: int


# one pass's counts as the backends report them (an int = combinations only)
PassCount = namedtuple("PassCount", "combinations additions accesses")


def split_count(v) -> tuple[int, int, int]:
    """(combinations, row_additions, row_accesses) of a backend's count."""
    if isinstance(v, PassCount):
        return int(v.combinations), int(v.additions), int(v.accesses)
    return int(v), int(v), int(v)


def family_words(gammas, n: int) -> np.ndarray:
    """(m, k, ceil(n/64)) uint64 image of a family (BitMatrix.to_numpy at
    word width 64, gf2.py:74-79) -- the layout bz_load_gammas expects."""
    mats = [gm.words64() for gm in gammas]
    return np.ascontiguousarray(np.stack(mats, axis=0), dtype=np.uint64)


def _load_single(gamma: BitMatrix, device: int) -> _native.Context:
    ctx = _native.context(device)
    key = ("single", gamma.num_cols, gamma.rows)
    if ctx.loaded_key != key:
        ctx.load(family_words([gamma], gamma.num_cols), gamma.num_cols, key=key)
    return ctx


def _check(g: int, k: int) -> None:
    if not 1 <= g <= k:
        raise InvalidArity(f"g={g} not in 1..{k}")


def enumerate_gpu(gamma: BitMatrix, g: int, ubound: int | None = None,
                  device: int = 0) -> EnumerationResult:
    """Minimum weight over all XORs of exactly g rows of gamma."""
    _check(g, gamma.num_rows)
    ctx = _native.context(device)
    with ctx.lock:
        _load_single(gamma, device)
        mn, combos = ctx.enumerate(0, g)
        adds, accs = ctx.counters(1)
    if ubound is not None:
        mn = min(mn, ubound)
    return EnumerationResult(int(mn), combos, adds[0][0], accs[0][0])


def weight_histogram_gpu(gamma: BitMatrix, g: int, device: int = 0):
    """(histogram over weights 0..n, min weight, combinations) of one pass."""
    _check(g, gamma.num_rows)
    ctx = _native.context(device)
    with ctx.lock:
        _load_single(gamma, device)
        return ctx.histogram(0, g)


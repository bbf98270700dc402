"""Per-(Gamma, g) enumeration on the GPU.

Drop-in for the reference's strategy functions (pkg/src/mindist/
enumeration.py:76-444): ``enumerate_gpu(gamma, g, ubound)`` returns the same
``EnumerationResult`` record (enumeration.py:43-50) with ``min_weight``
clipped to ``ubound`` (enumeration.py:60-64) and ``InvalidArity`` for g
outside 1..k (enumeration.py:67-69).  The work runs in the sm_100a kernel
K1 behind the C ABI (include/bz.h); there is no CPU path.

Counters: ``combinations`` is exact (C(k, g) per pass).  In the GPU
algorithm every codeword costs exactly one row addition (prefix XOR ^ row
e) and one row access (the broadcast read of row e), so ``row_additions`` and
``row_accesses`` both equal ``combinations``; the prefix-maintenance XORs
(three prefix-table rows per prefix step) are not counted.
"""

from __future__ import annotations

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
    if ubound is not None:
        mn = min(mn, ubound)
    return EnumerationResult(int(mn), combos, combos, combos)


def weight_histogram_gpu(gamma: BitMatrix, g: int, device: int = 0):
    """(histogram over weights 0..n, min weight, combinations) of one pass."""
    _check(g, gamma.num_rows)
    ctx = _native.context(device)
    with ctx.lock:
        _load_single(gamma, device)
        return ctx.histogram(0, g)


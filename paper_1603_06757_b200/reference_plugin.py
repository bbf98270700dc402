"""The reference-side binding: a ``"gpu"`` strategy for the reference package
``mindist`` itself, bound to libbz.so through ctypes only.

This is the stub INTEGRATION.md section B shows a ``mindist`` maintainer
adding, made installable into an unmodified copy of the package (the
reference's strategy seam is the ``STRATEGIES`` tuple, ``m/engine.py:29``,
and ``_Runner.run``, ``m/engine.py:136-150``):

    import mindist.engine
    from paper_1603_06757_b200 import reference_plugin
    reference_plugin.install(mindist.engine)
    mindist.engine.minimum_distance(G, mindist.engine.EngineConfig(strategy="gpu"))

``install`` appends ``"gpu"`` to ``STRATEGIES`` and wraps ``_Runner.run`` so
that strategy ``"gpu"`` runs each (Gamma_j, g) pass as one ``bz_enumerate``
call -- the same per-pass contract as ``enumerate_basic/stack/saved``
(``m/enumeration.py:76,128,305``): the full pass (no early exit, the
reference's counters are schedule-independent), ``min_weight`` clipped to
``ubound`` (``m/enumeration.py:60-64``), ``InvalidArity`` for g outside 1..k
(``m/enumeration.py:67-69``).  The running-U loop, bounds, trace, max_g,
resume and Interrupted stay the reference's own code.

Nothing here imports the rest of this package: the module needs only
numpy, ctypes and the library file, as a reference-side stub would.  The
reference's own exception classes are raised (looked up on the installed
engine module's ``errors``).
"""

from __future__ import annotations

import ctypes
import os
import sys
import threading
from math import comb

import numpy as np

DEFAULT_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbz.so")

_vp = ctypes.c_void_p
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)

_BZ_ERR_INVALID_ARITY = 1
_BZ_ERR_INVALID_DIMENSIONS = 2
_BZ_ERR_TOO_LARGE = 3


def _bind(path: str):
    L = ctypes.CDLL(path)
    L.bz_create.argtypes = [ctypes.c_int, ctypes.POINTER(_vp)]
    L.bz_destroy.argtypes = [_vp]
    L.bz_destroy.restype = None
    L.bz_last_error.argtypes = [_vp]
    L.bz_last_error.restype = ctypes.c_char_p
    L.bz_load_gammas.argtypes = [_vp, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.bz_enumerate.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               _i32p, _u64p]
    L.bz_launch_count.argtypes = [_vp, _u64p]
    L.bz_counters.argtypes = [_vp, ctypes.c_int, _u64p, _u64p]
    return L


class GpuPasses:
    """One device context per reference ``_Runner`` Gamma index (the device
    analogue of ``_Runner.store_for``, ``m/engine.py:128-134``: built lazily
    per Gamma, kept across rounds)."""

    def __init__(self, lib, errors, device: int = 0):
        self.lib = lib
        self.errors = errors
        self.device = device
        self.ctxs: dict[int, tuple[_vp, object]] = {}
        self.lock = threading.Lock()

    def _fail(self, rc: int, ctx, what: str):
        raw = self.lib.bz_last_error(ctx) if ctx is not None else b""
        msg = f"{what}: {raw.decode() if raw else ''}"
        e = self.errors
        if rc == _BZ_ERR_INVALID_ARITY:
            raise e.InvalidArity(msg)
        if rc == _BZ_ERR_INVALID_DIMENSIONS:
            raise e.InvalidDimensions(msg)
        if rc == _BZ_ERR_TOO_LARGE:
            raise e.TooLarge(msg)
        raise e.MindistError(msg)

    def _context(self, idx: int, gamma):
        hit = self.ctxs.get(idx)
        if hit is not None and hit[1] is gamma:
            return hit[0]
        ctx = hit[0] if hit is not None else None
        if ctx is None:
            ctx = _vp()
            rc = self.lib.bz_create(self.device, ctypes.byref(ctx))
            if rc:
                self._fail(rc, ctx, "bz_create")
        words = np.ascontiguousarray(gamma.with_word_width(64).to_numpy(), dtype=np.uint64)
        k = gamma.num_rows
        rc = self.lib.bz_load_gammas(ctx, words.ctypes.data_as(_u64p), 1, k, gamma.num_cols)
        if rc:
            self._fail(rc, ctx, "bz_load_gammas")
        self.ctxs[idx] = (ctx, gamma)
        return ctx

    def run(self, idx: int, gamma, g: int, ubound):
        """One (Gamma, g) pass -> the reference's EnumerationResult."""
        k = gamma.num_rows
        if not 1 <= g <= k:
            raise self.errors.InvalidArity(f"g={g} not in 1..{k}")
        with self.lock:
            ctx = self._context(idx, gamma)
            mn = np.zeros(1, np.int32)
            combos = np.zeros(1, np.uint64)
            rc = self.lib.bz_enumerate(ctx, 0, g, 0, 1, mn.ctypes.data_as(_i32p),
                                       combos.ctypes.data_as(_u64p))
            if rc:
                self._fail(rc, ctx, "bz_enumerate")
            adds = np.zeros(1, np.uint64)
            accs = np.zeros(1, np.uint64)
            rc = self.lib.bz_counters(ctx, 1, adds.ctypes.data_as(_u64p), accs.ctypes.data_as(_u64p))
            if rc:
                self._fail(rc, ctx, "bz_counters")
        best = int(mn[0])
        if ubound is not None:
            best = min(best, ubound)
        c = int(combos[0])
        assert c == comb(k, g), (c, k, g)
        # the device's row additions / row accesses for this pass
        # (bz_counters) -- strategy-specific, as the reference's are
        return self.enumeration_result(best, c, int(adds[0]), int(accs[0]))

    def close(self):
        for ctx, _ in self.ctxs.values():
            self.lib.bz_destroy(ctx)
        self.ctxs.clear()


def install(engine, lib_path: str | None = None, device: int = 0):
    """Add strategy "gpu" to an imported ``mindist.engine`` module.

    Idempotent.  Returns the ``GpuPasses`` object runners of this engine
    share (its ``lib`` is the loaded libbz.so handle)."""
    if getattr(engine, "_bz_gpu_passes", None) is not None:
        return engine._bz_gpu_passes
    pkg = sys.modules[engine.__name__.rsplit(".", 1)[0]]
    errors = pkg.errors if hasattr(pkg, "errors") else sys.modules[pkg.__name__ + ".errors"]
    enumeration = sys.modules[pkg.__name__ + ".enumeration"]
    lib = _bind(lib_path or os.environ.get("BZ_LIB") or DEFAULT_LIB)
    passes = GpuPasses(lib, errors, device)
    passes.enumeration_result = enumeration.EnumerationResult

    engine.STRATEGIES = tuple(engine.STRATEGIES) + ("gpu",)
    real_run = engine._Runner.run

    def run(self, idx, gamma, g, ubound):
        if self.config.strategy == "gpu":
            return passes.run(idx, gamma, g, ubound)
        return real_run(self, idx, gamma, g, ubound)

    engine._Runner.run = run
    engine._bz_gpu_passes = passes
    return passes

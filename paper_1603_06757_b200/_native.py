"""ctypes binding of the C ABI in include/bz.h (libbz.so, built in-tree).

The library is the product: there is no CPU fallback.  If ``libbz.so`` is
missing, or no sm_100 GPU is visible, every compute entry point raises
``NoDevice`` -- loudly, never silently degrading.  ``bz_plan`` and the
version/device-count queries need no GPU.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import (DeviceError, InvalidArity, InvalidDimensions, MindistError,
                     NoDevice, TooLarge)

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BZ_LIB") or os.path.join(PKG_DIR, "libbz.so")
ABI_VERSION = 16

BZ_OK = 0
BZ_LOOP_RUNNING, BZ_LOOP_DONE, BZ_LOOP_MAX_G = 0, 1, 2
# bz_round_record (include/bz.h)
ROUND_RECORD = np.dtype([("g", np.int32), ("L", np.int32), ("U", np.int32), ("pad", np.int32),
                         ("combinations", np.uint64), ("row_additions", np.uint64),
                         ("row_accesses", np.uint64), ("kernel_ms", np.float32),
                         ("pad2", np.int32)])
_CODES = {
    1: InvalidArity,
    2: InvalidDimensions,
    3: TooLarge,
    4: DeviceError,
    5: NoDevice,
    6: MindistError,
    7: ValueError,
}

# every symbol include/bz.h declares (checked by tests/test_abi.py)
SYMBOLS = ("bz_abi_version", "bz_device_count", "bz_create", "bz_destroy",
           "bz_last_error", "bz_set_engine", "bz_set_elision", "bz_set_early_exit", "bz_elided",
           "bz_reduce_on_columns", "bz_brute_force", "bz_load_gammas",
           "bz_round", "bz_rounds", "bz_advance", "bz_counters",
           "bz_enumerate",
           "bz_histogram", "bz_plan", "bz_timer_start", "bz_timer_stop",
           "bz_last_kernel_ms", "bz_round_ms", "bz_gamma_family",
           "bz_shared_bound_export", "bz_shared_bound_open", "bz_shared_bound_epoch",
           "bz_shared_bound_read",
           "bz_shared_bound_close", "bz_launch_count", "bz_measure_int_peaks",
           "bz_k5q_selftest")

_lib = None

c_int, c_float, c_double = ctypes.c_int, ctypes.c_float, ctypes.c_double
u64p = ctypes.POINTER(ctypes.c_uint64)
i64p = ctypes.POINTER(ctypes.c_int64)
i32p = ctypes.POINTER(ctypes.c_int32)
vp = ctypes.c_void_p


def lib():
    """Load libbz.so (raises NoDevice if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NoDevice(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                       "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.bz_abi_version.restype = c_int
    L.bz_device_count.restype = c_int
    L.bz_create.argtypes = [c_int, ctypes.POINTER(vp)]
    L.bz_destroy.argtypes = [vp]
    L.bz_destroy.restype = None
    L.bz_last_error.argtypes = [vp]
    L.bz_last_error.restype = ctypes.c_char_p
    L.bz_set_engine.argtypes = [vp, c_int]
    L.bz_set_elision.argtypes = [vp, c_int]
    L.bz_set_early_exit.argtypes = [vp, c_int]
    L.bz_k5q_selftest.argtypes = [i32p]
    L.bz_brute_force.argtypes = [vp, u64p, c_int, c_int, c_int, i32p, u64p]
    L.bz_reduce_on_columns.argtypes = [u64p, c_int, c_int, i32p, c_int, i32p, ctypes.POINTER(c_int)]
    L.bz_elided.argtypes = [vp, u64p]
    L.bz_load_gammas.argtypes = [vp, u64p, c_int, c_int, c_int]
    L.bz_round.argtypes = [vp, c_int, c_int, c_int, c_int, c_int, i32p, u64p]
    L.bz_rounds.argtypes = [vp, c_int, c_int, i32p, c_int, c_int, c_int, i32p, u64p]
    L.bz_advance.argtypes = [vp, c_int, c_int, c_int, c_int, ctypes.c_int64, i32p, vp, c_int,
                             ctypes.POINTER(c_int)]
    L.bz_enumerate.argtypes = [vp, c_int, c_int, c_int, c_int, i32p, u64p]
    L.bz_counters.argtypes = [vp, c_int, u64p, u64p]
    L.bz_histogram.argtypes = [vp, c_int, c_int, c_int, c_int, u64p, i32p, u64p]
    L.bz_plan.argtypes = [c_int, c_int, c_int, c_int, c_int, i64p, c_int, i32p, u64p]
    L.bz_timer_start.argtypes = [vp]
    L.bz_timer_stop.argtypes = [vp, ctypes.POINTER(c_float)]
    L.bz_last_kernel_ms.argtypes = [vp, ctypes.POINTER(c_float)]
    L.bz_round_ms.argtypes = [vp, ctypes.POINTER(c_float), c_int]
    L.bz_shared_bound_export.argtypes = [vp, ctypes.c_char_p]
    L.bz_shared_bound_open.argtypes = [vp, ctypes.c_char_p]
    L.bz_shared_bound_epoch.argtypes = [vp, ctypes.c_uint32]
    L.bz_shared_bound_close.argtypes = [vp]
    L.bz_shared_bound_read.argtypes = [vp, c_int, i32p]
    L.bz_gamma_family.argtypes = [u64p, c_int, c_int, c_int, u64p, i32p, i32p,
                                  ctypes.POINTER(c_int)]
    L.bz_launch_count.argtypes = [vp, u64p]
    L.bz_measure_int_peaks.argtypes = [vp, c_int, ctypes.POINTER(c_double)]
    if L.bz_abi_version() != ABI_VERSION:
        raise NoDevice(f"libbz ABI {L.bz_abi_version()} != {ABI_VERSION}: rebuild")
    _lib = L
    return L


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def check(rc: int, ctx=None, what: str = "") -> None:
    if rc == BZ_OK:
        return
    msg = ""
    if ctx is not None:
        raw = lib().bz_last_error(ctx)
        msg = raw.decode() if raw else ""
    exc = _CODES.get(rc, DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)


def k5q_selftest() -> tuple[int, tuple[int, int] | None]:
    """Host-only check of the K5q offset encoding (bz_k5q_selftest):
    (failures, first failing (prefix weight, bound) or None)."""
    bad = np.zeros(2, dtype=np.int32)
    n = int(lib().bz_k5q_selftest(_ptr(bad, ctypes.c_int32)))
    return n, (int(bad[0]), int(bad[1])) if n else None


def device_count() -> int:
    return int(lib().bz_device_count())


ENGINES = {"auto": 0, "popc": 1, "imma": 2, "umma": 3, "mxf4": 4, "mxf4p": 5, "mxf4t": 6, "mxf4q": 7,
           "mxf4w": 8, "mxf4f": 9}


def plan(m: int, k: int, g: int, engine: str = "auto", nshards: int = 1):
    """The device work plan for one round (host-only; see bz_plan)."""
    L = lib()
    e = ENGINES[engine]
    ng = np.zeros(1, dtype=np.int32)
    nc = np.zeros(1, dtype=np.uint64)
    check(L.bz_plan(m, k, g, e, nshards, None, 0, _ptr(ng, ctypes.c_int32),
                    _ptr(nc, ctypes.c_uint64)), what="bz_plan")
    out = np.zeros((int(ng[0]), 12), dtype=np.int64)
    check(L.bz_plan(m, k, g, e, nshards, _ptr(out, ctypes.c_int64), int(ng[0]),
                    _ptr(ng, ctypes.c_int32), _ptr(nc, ctypes.c_uint64)), what="bz_plan")
    return [tuple(int(v) for v in row) for row in out], int(nc[0])


class Context:
    """One CUDA device.  Owns the device copy of the loaded Gamma family."""

    def __init__(self, device: int = 0):
        L = lib()
        h = vp()
        rc = L.bz_create(int(device), ctypes.byref(h))
        self._h = h
        if rc != BZ_OK:
            try:
                check(rc, h, f"bz_create(device={device})")
            finally:
                L.bz_destroy(h)
                self._h = None
        self.device = device
        self.engine = "auto"
        self.elision = True
        self.early_exit = False
        # a context is not thread-safe (include/bz.h): callers hold this
        # across a whole load + rounds sequence (minimum_distance,
        # enumerate_gpu, ...), so concurrent calls on distinct matrices
        # never interleave each other's loads
        self.lock = threading.RLock()
        self.loaded_key = None
        self.m = self.k = self.n = 0

    def close(self) -> None:
        if self._h is not None:
            lib().bz_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        if self._h is None:
            raise MindistError("context is closed")
        return self._h

    def set_engine(self, engine: str) -> None:
        """'auto' (= 'mxf4': tcgen05 kind::mxf4 K5 for g >= 4), 'umma'
        (tcgen05 kind::i8 K4), 'imma' (legacy-IMMA K3) or 'popc' (K1 only)."""
        if engine not in ENGINES:
            raise ValueError(f"unknown engine {engine!r}")
        check(lib().bz_set_engine(self.handle, ENGINES[engine]), self.handle, "bz_set_engine")
        self.engine = engine

    def shared_bound_export(self) -> bytes:
        """Allocate this context's shared-bound mirror; its 64-byte CUDA IPC
        handle (see bz_shared_bound_export)."""
        buf = ctypes.create_string_buffer(64)
        check(lib().bz_shared_bound_export(self.handle, buf), self.handle,
              "bz_shared_bound_export")
        return buf.raw

    def shared_bound_open(self, handle: bytes | None) -> None:
        """Use the mirror of `handle` (None: this context's own)."""
        if handle is not None and len(handle) != 64:
            raise ValueError("IPC handle must be 64 bytes")
        check(lib().bz_shared_bound_open(self.handle, handle), self.handle,
              "bz_shared_bound_open")

    def shared_bound_epoch(self, epoch: int) -> None:
        check(lib().bz_shared_bound_epoch(self.handle, epoch & 0xffffffff), self.handle,
              "bz_shared_bound_epoch")

    def shared_bound_read(self, g: int) -> int:
        out = np.zeros(1, dtype=np.int32)
        check(lib().bz_shared_bound_read(self.handle, g, _ptr(out, ctypes.c_int32)), self.handle,
              "bz_shared_bound_read")
        return int(out[0])

    def shared_bound_close(self) -> None:
        check(lib().bz_shared_bound_close(self.handle), self.handle, "bz_shared_bound_close")

    def set_elision(self, on: bool) -> None:
        """Identity-column elision for the next load (see bz_set_elision);
        results are identical either way."""
        check(lib().bz_set_elision(self.handle, 1 if on else 0), self.handle, "bz_set_elision")
        self.elision = bool(on)
        self.loaded_key = None

    def set_early_exit(self, on: bool) -> None:
        """In-round early exit at lower_prev (see bz_set_early_exit)."""
        if bool(on) != self.early_exit:
            check(lib().bz_set_early_exit(self.handle, 1 if on else 0), self.handle,
                  "bz_set_early_exit")
            self.early_exit = bool(on)

    def elided(self) -> int:
        """Bit mask of the loaded Gammas stored without identity columns."""
        v = np.zeros(1, dtype=np.uint64)
        check(lib().bz_elided(self.handle, _ptr(v, ctypes.c_uint64)), self.handle, "bz_elided")
        return int(v[0])

    def brute_force(self, words: np.ndarray, n: int, max_k: int):
        """(distance, codewords) over all 2^k - 1 messages (bz_brute_force)."""
        words = np.ascontiguousarray(words, dtype=np.uint64)
        d = np.zeros(1, dtype=np.int32)
        c = np.zeros(1, dtype=np.uint64)
        check(lib().bz_brute_force(self.handle, _ptr(words, ctypes.c_uint64), words.shape[0],
                                   n, max_k, _ptr(d, ctypes.c_int32),
                                   _ptr(c, ctypes.c_uint64)),
              self.handle, "bz_brute_force")
        return int(d[0]), int(c[0])

    def load(self, words: np.ndarray, n: int, key=None) -> None:
        """words: (m, k, ceil(n/64)) uint64 row image of the family.  `key`
        identifies the family for callers that cache what is loaded."""
        self.loaded_key = None
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if words.ndim != 3:
            raise InvalidDimensions("expected an (m, k, w64) array")
        m, k, _ = words.shape
        check(lib().bz_load_gammas(self.handle, _ptr(words, ctypes.c_uint64), m, k, n),
              self.handle, "bz_load_gammas")
        self.m, self.k, self.n = m, k, n
        self.loaded_key = key

    def _buf(self, name: str, dtype, size: int):
        """A reusable host buffer and its ctypes pointer (ctypes pointer
        objects cost microseconds each; the batched rounds sit on the timed
        path of every run)."""
        bufs = self.__dict__.setdefault("_bufs", {})
        hit = bufs.get(name)
        if hit is None or hit[0].size < size:
            arr = np.zeros(max(size, 1), dtype=dtype)
            hit = (arr, arr.ctypes.data_as(ctypes.POINTER(np.ctypeslib.as_ctypes_type(dtype))))
            bufs[name] = hit
        return hit

    def round(self, g: int, lower_prev: int, upper: int, shard: int = 0,
              nshards: int = 1):
        m = max(self.m, 1)
        mins, pmin = self._buf("mins", np.int32, m)
        combos, pcb = self._buf("combos", np.uint64, m)
        check(lib().bz_round(self.handle, g, lower_prev, upper, shard, nshards, pmin, pcb),
              self.handle, f"bz_round(g={g})")
        return mins[:self.m].tolist(), combos[:self.m].tolist()

    def rounds(self, g0: int, lower_prev: list[int], upper: int, shard: int = 0,
               nshards: int = 1):
        """Rounds g0 .. g0+len(lower_prev)-1 in one call (see bz_rounds);
        returns [(mins, combos)] per round."""
        count = len(lower_prev)
        m = max(self.m, 1)
        lp, plp = self._buf("lp", np.int32, count)
        lp[:count] = lower_prev
        mins, pmin = self._buf("mins", np.int32, count * m)
        combos, pcb = self._buf("combos", np.uint64, count * m)
        check(lib().bz_rounds(self.handle, g0, count, plp, upper, shard, nshards, pmin, pcb),
              self.handle, f"bz_rounds(g0={g0}, count={count})")
        mn = mins[:count * m].reshape(count, m).tolist()
        cb = combos[:count * m].reshape(count, m).tolist()
        return list(zip(mn, cb))

    def advance(self, m_arg: int, km_arg: int, max_g: int, u_rows: int, budget: int,
                state):
        """One step of the Algorithm-1 loop (bz_advance).  ``state`` is an
        int32 array [g, L, U, g_reached, status], updated in place; returns
        the records of the rounds folded in as ROUND_RECORD tuples (g, L, U,
        pad, combinations, row_additions, row_accesses, kernel_ms, pad)."""
        k = max(self.k, 1)
        recs = self.__dict__.get("_recs")
        if recs is None or len(recs) < k:
            recs = np.zeros(k, dtype=ROUND_RECORD)
            self._recs = recs
            self._recs_p = ctypes.c_void_p(recs.ctypes.data)
            self._nrec = c_int()
            self._nrec_p = ctypes.byref(self._nrec)
        check(lib().bz_advance(self.handle, m_arg, km_arg, min(max_g, 1 << 30), u_rows, budget,
                               state.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                               self._recs_p, len(recs), self._nrec_p),
              self.handle, f"bz_advance(g={int(state[0])})")
        return recs[:self._nrec.value].tolist()

    def counters(self, count: int = 1):
        """Row additions and row accesses (count x m, round-major) of the
        last round / rounds / enumerate call (bz_counters)."""
        m = max(self.m, 1)
        adds, pad = self._buf("adds", np.uint64, count * m)
        accs, pac = self._buf("accs", np.uint64, count * m)
        check(lib().bz_counters(self.handle, count, pad, pac), self.handle, "bz_counters")
        return (adds[:count * m].reshape(count, m).tolist(),
                accs[:count * m].reshape(count, m).tolist())

    def round_ms(self, count: int) -> list[float]:
        """Per-round device ms of the last round / rounds call."""
        out, pout = self._buf("round_ms", np.float32, count)
        check(lib().bz_round_ms(self.handle, pout, count), self.handle, "bz_round_ms")
        return out[:count].tolist()

    def enumerate(self, gamma: int, g: int, shard: int = 0, nshards: int = 1):
        mn = np.zeros(1, dtype=np.int32)
        c = np.zeros(1, dtype=np.uint64)
        check(lib().bz_enumerate(self.handle, gamma, g, shard, nshards,
                                 _ptr(mn, ctypes.c_int32), _ptr(c, ctypes.c_uint64)),
              self.handle, f"bz_enumerate(g={g})")
        return int(mn[0]), int(c[0])

    def histogram(self, gamma: int, g: int, shard: int = 0, nshards: int = 1):
        hist = np.zeros(self.n + 1, dtype=np.uint64)
        mn = np.zeros(1, dtype=np.int32)
        c = np.zeros(1, dtype=np.uint64)
        check(lib().bz_histogram(self.handle, gamma, g, shard, nshards,
                                 _ptr(hist, ctypes.c_uint64), _ptr(mn, ctypes.c_int32),
                                 _ptr(c, ctypes.c_uint64)),
              self.handle, f"bz_histogram(g={g})")
        return hist, int(mn[0]), int(c[0])

    def timer_start(self) -> None:
        check(lib().bz_timer_start(self.handle), self.handle, "bz_timer_start")

    def timer_stop(self) -> float:
        ms = c_float()
        check(lib().bz_timer_stop(self.handle, ctypes.byref(ms)), self.handle, "bz_timer_stop")
        return float(ms.value)

    def last_kernel_ms(self) -> float:
        ms = c_float()
        check(lib().bz_last_kernel_ms(self.handle, ctypes.byref(ms)), self.handle)
        return float(ms.value)

    def launch_count(self) -> int:
        v = np.zeros(1, dtype=np.uint64)
        check(lib().bz_launch_count(self.handle, _ptr(v, ctypes.c_uint64)), self.handle)
        return int(v[0])

    def measure_int_peaks(self, w_words: int) -> dict:
        out = (c_double * 14)()
        check(lib().bz_measure_int_peaks(self.handle, w_words, out), self.handle,
              "bz_measure_int_peaks")
        keys = ("popc_per_s", "lop3_per_s", "sm_mhz", "sm_count", "popc_per_clk_sm",
                "lop3_per_clk_sm", "codeword_per_s", "codeword_per_clk_sm", "imma_mac_per_s",
                "imma_mac_per_clk_sm", "umma_mac_per_s", "umma_mac_per_clk_sm",
                "mxf4_mac_per_s", "mxf4_mac_per_clk_sm")
        return dict(zip(keys, (float(v) for v in out)))


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    """Process-wide context per device (created on first use)."""
    ctx = _contexts.get(device)
    if ctx is None or ctx._h is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx

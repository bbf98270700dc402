"""ABI-independent A/B of library builds (raw ctypes: bz_create /
bz_load_gammas / bz_round / bz_rounds / bz_last_kernel_ms, unchanged since
ABI 10): config 5's g = 8 round alone and the whole batch g = 1..8, each
library in turn, interleaved.

    python tools/raw_ab.py lib1.so lib2.so ...
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_06757_b200.configs import code  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

G, gs, _ = code("cfg5", 7)
words = np.ascontiguousarray(family_words(gs.gammas, 160), dtype=np.uint64)
vp, i32p, u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint64)
libs = []
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    L.bz_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    L.bz_load_gammas.argtypes = [vp, u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.bz_round.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           i32p, u64p]
    L.bz_rounds.argtypes = [vp, ctypes.c_int, ctypes.c_int, i32p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_int, i32p, u64p]
    L.bz_last_kernel_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
    h = vp()
    assert L.bz_create(0, ctypes.byref(h)) == 0
    assert L.bz_load_gammas(h, words.ctypes.data_as(u64p), 2, 80, 160) == 0
    libs.append((path, L, h))
mins = np.zeros(16, np.int32)
cb = np.zeros(16, np.uint64)
lp = np.array([0] + [2 * (g + 1) for g in range(1, 8)], dtype=np.int32)
ms = ctypes.c_float()
res = {p: {"g8": [], "batch": []} for p, _, _ in libs}
for rep in range(int(os.environ.get("REPS", "6"))):
    for path, L, h in libs:
        assert L.bz_round(h, 8, 0, 18, 0, 1, mins.ctypes.data_as(i32p), cb.ctypes.data_as(u64p)) == 0
        L.bz_last_kernel_ms(h, ctypes.byref(ms))
        res[path]["g8"].append(ms.value)
        assert L.bz_rounds(h, 1, 8, lp.ctypes.data_as(i32p), 81, 0, 1, mins.ctypes.data_as(i32p),
                           cb.ctypes.data_as(u64p)) == 0
        L.bz_last_kernel_ms(h, ctypes.byref(ms))
        res[path]["batch"].append(ms.value)
for path, r in res.items():
    g8 = sorted(r["g8"][1:])
    b = sorted(r["batch"][1:])
    print(f"{path:45s} g8 alone {g8[len(g8) // 2]:.4f} ms   rounds 1..8 {b[len(b) // 2]:.4f} ms")

"""Summarise a K4/K5 per-chunk timeline (BZ_K4_DEBUG & 32, BZ_K4_CTRACE):
clocks per tile and per prefix step by ell band, and the spread of SM
finish times.

    python tools/ctrace_stats.py ctrace.bin [m k g engine]
"""

from __future__ import annotations

import bisect
import os
import sys
from math import comb

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1603_06757_b200 import _native  # noqa: E402


def main():
    path = sys.argv[1]
    m, k, g = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (2, 80, 8)
    engine = sys.argv[5] if len(sys.argv) > 5 else "mxf4"
    N = 240 if engine in ("mxf4", "auto") else 256
    ct = np.fromfile(path, dtype=np.int64).reshape(1024, 64, 4)
    groups, _ = _native.plan(m, k, g, engine)
    begins = [int(gr[0]) for gr in groups]

    def info(c):
        gi = bisect.bisect_right(begins, c) - 1
        b, npf, gam, ell, ppl, combs, depth, lanes, spc, nsb, sfloor, _ = (int(x) for x in groups[gi])
        local = c - b
        pb, tb = divmod(local, nsb)
        steps = min(ppl, npf - pb * lanes * ppl)
        ntiles = -(-comb(k - sfloor, depth) // N)
        tpc = -(-spc // N)
        tiles = min(ntiles, tb * tpc + tpc) - tb * tpc
        return ell, steps, steps * tiles

    rows, ends = [], []
    for b in range(1024):
        if ct[b, 0, 0] < 0:
            continue
        last = 0
        for q in range(64):
            c, ts, te, gt = (int(x) for x in ct[b, q])
            if c < 0:
                break
            ell, steps, tiles = info(c)
            rows.append((ell, steps, tiles, te - ts))
            last = max(last, gt)
        ends.append(last)
    r = np.array(rows, dtype=np.float64)
    print(f"chunks {len(r)}  clk/tile {r[:, 3].sum() / r[:, 2].sum():.0f}")
    for lo, hi in [(0, 40), (40, 50), (50, 60), (60, 66), (66, 72), (72, k)]:
        s = (r[:, 0] >= lo) & (r[:, 0] < hi)
        if s.any():
            print(f"ell [{lo},{hi}): chunks {int(s.sum())} tiles {int(r[s, 2].sum())} "
                  f"steps {int(r[s, 1].sum())} clk/tile {r[s, 3].sum() / r[s, 2].sum():.0f} "
                  f"clk/step {r[s, 3].sum() / r[s, 1].sum():.0f}")
    e = np.array(ends)
    print(f"SM finish spread {(e.max() - e.min()) / 1e3:.1f} us "
          f"(mean lag behind the last {(e.max() - e).mean() / 1e3:.1f} us)")


if __name__ == "__main__":
    main()

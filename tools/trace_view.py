"""Print a K4/K5 tile timeline (BZ_K4_DEBUG & 8, BZ_K4_TRACE_OUT): per tile,
the clock of each traced event relative to the first loader event, and the
gaps between consecutive events of the MMA issuer and of epilogue warp 0.

    python tools/trace_view.py bz_trace.bin [first] [count]
"""

from __future__ import annotations

import sys

import numpy as np

SLOTS = {0: "ld_go", 15: "ld_tma", 5: "mma_pre", 6: "mma_bfull", 1: "mma_acc0",
         12: "mma_p0_done", 13: "mma_acc1", 4: "mma_end", 8: "e0_top", 9: "e0_full",
         2: "e0_go", 10: "e0_ldw", 11: "e0_arr", 3: "e0_done", 7: "eL_go", 14: "eL_arr"}
ORDER = [0, 15, 5, 6, 1, 12, 13, 4, 8, 9, 2, 10, 11, 3, 7, 14]


def main():
    h = np.fromfile(sys.argv[1], dtype=np.int64).reshape(16, 256)
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    count = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    base = h[0][h[0] > 0].min() if (h[0] > 0).any() else 0
    print("tile " + " ".join(f"{SLOTS[s]:>11}" for s in ORDER))
    for t in range(first, first + count):
        print(f"{t:4d} " + " ".join(f"{(h[s][t] - base) if h[s][t] else 0:11d}" for s in ORDER))
    # mean per-tile durations between events (steady state)
    def d(a, b):
        x = h[b][first:first + count] - h[a][first:first + count]
        return float(np.median(x))
    print("median gaps: bfull wait %.0f | acc0 wait+fence %.0f | part0 issue %.0f | "
          "acc1 wait %.0f | part1 issue %.0f" % (d(5, 6), d(6, 1), d(1, 12), d(12, 13), d(13, 4)))
    print("epi0: full wait %.0f | fence %.0f | ld %.0f | arrive %.0f | reduce %.0f" %
          (d(8, 9), d(9, 2), d(2, 10), d(10, 11), d(11, 3)))
    per = np.diff(h[4][first:first + count])
    print("tile period (mma_end): median %.0f clk" % float(np.median(per)))


if __name__ == "__main__":
    main()

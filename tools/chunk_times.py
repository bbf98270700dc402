"""Per-chunk timeline summary of one K5 launch (BZ_K4_DEBUG & 32 ->
BZ_K4_CTRACE): chunks per block, chunk durations, block spans.

    BZ_K4_DEBUG=32 BZ_K4_CTRACE=ct.bin python tools/profile_round.py cfg5 G
    python tools/chunk_times.py ct.bin
"""
import sys

import numpy as np

ct = np.fromfile(sys.argv[1], dtype=np.int64).reshape(1024, 64, 4)
life = ct[:, 63, :3].copy()
ct[:, 63, 0] = -1
valid = ct[:, :, 0] >= 0
nblk = int(valid.any(axis=1).sum())
per = valid.sum(axis=1)[:nblk]
dur = (ct[:, :, 2] - ct[:, :, 1])[valid]
t_done = ct[:, :, 3][valid]
print(f"blocks {nblk}, chunks/block min {per.min()} median {np.median(per):.0f} max {per.max()}")
print(f"chunk duration (clk): median {np.median(dur):.0f} p10 {np.percentile(dur, 10):.0f} "
      f"p90 {np.percentile(dur, 90):.0f} max {dur.max()}")
span = []
for b in range(nblk):
    v = valid[b]
    if v.any():
        span.append(ct[b, v, 2].max() - ct[b, v, 1].min())
print(f"block span (dequeue first -> done last, clk): median {np.median(span):.0f} max {max(span)}")
print(f"done spread across blocks (ns): {t_done.max() - t_done.min()}")

lv = life[:nblk]
if (lv > 0).all():
    t0 = lv[:, 0].min()
    first_done = np.array([ct[b, valid[b], 3].min() for b in range(nblk) if valid[b].any()]) - t0
    print(f"block entry skew {lv[:, 0].max() - t0} ns; prologue median "
          f"{np.median(lv[:, 1] - lv[:, 0]):.0f} ns; first chunk done median "
          f"{np.median(first_done):.0f} ns; last chunk done {t_done.max() - t0} ns; "
          f"block exit max {lv[:, 2].max() - t0} ns")

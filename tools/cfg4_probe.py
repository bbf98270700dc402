"""Config 4 on the device: the histogram (K1h) and the minimum (K5q / K5),
kernel time of each (median of 7)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import microbench_gamma  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

ctx = _native.context(0)
ctx.load(family_words([microbench_gamma(1)], 192), 192)


def t(fn, n=7):
    ms = []
    for i in range(n + 1):
        r = fn()
        if i:
            ms.append(ctx.last_kernel_ms())
    return sorted(ms)[n // 2] * 1e3, r


us, (hist, mn, c) = t(lambda: ctx.histogram(0, 6))
print(f"histogram {us:.1f} us  min {mn} combos {c} sum {int(sum(hist))}")
us, r = t(lambda: ctx.enumerate(0, 6))
print(f"minimum   {us:.1f} us  {r}")

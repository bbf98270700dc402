"""One round of a BASELINE config on the default engine with the per-tile
timeline on (needs a library built with -DBZ_K4_TRACE=1, e.g. BZ_LIB=...):

    BZ_K4_DEBUG=8 BZ_K4_TRACE_OUT=tr.bin python tools/trace_round.py cfg5 5 [upper]
    python tools/trace_view.py tr.bin 16 32
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_06757_b200 import _native  # noqa: E402
from paper_1603_06757_b200.configs import code, microbench_gamma  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402

name, g = sys.argv[1], int(sys.argv[2])
upper = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 20
ctx = _native.context(0)
if name == "cfg4":
    ctx.load(family_words([microbench_gamma(1)], 192), 192)
else:
    G, gs, _ = code(name)
    ctx.load(family_words(gs.gammas, G.num_cols), G.num_cols)
dbg = os.environ.pop("BZ_K4_DEBUG", None)
ctx.round(g, 0, upper)  # warm: tables, plan
if dbg:
    os.environ["BZ_K4_DEBUG"] = dbg
print(ctx.round(g, 0, upper), f"{ctx.last_kernel_ms() * 1e3:.1f} us")

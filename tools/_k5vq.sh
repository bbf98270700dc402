cd $GRAFT_REPO_ROOT
python - <<'PY'
import sys
sys.path.insert(0, ".")
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.configs import code, microbench_gamma
from paper_1603_06757_b200.enumeration import family_words
ctx = _native.context(0)
def t(fn, n=6):
    ms = []
    for i in range(n):
        fn()
        if i: ms.append(ctx.last_kernel_ms())
    return round(sorted(ms)[len(ms) // 2] * 1e3, 1)
ctx.load(family_words([microbench_gamma(1)], 192), 192)
for e in ("mxf4", "mxf4q"):
    ctx.set_engine(e); print("cfg4", e, t(lambda: ctx.enumerate(0, 6)))
G, gs, _ = code("cfg5", 7)
ctx.load(family_words(gs.gammas, 160), 160)
for g, U in ((5, 22), (6, 20), (7, 20)):
    for e in ("mxf4", "mxf4q"):
        ctx.set_engine(e)
        print("cfg5", g, e, "loose", t(lambda: ctx.round(g, 0, 1 << 20)), "tight", t(lambda: ctx.round(g, 0, U)))
PY

# Timing ablations of the config-5 g = 8 tensor-core round (results are NOT
# valid under BZ_K4_DEBUG): 0 none, 1 no epilogue TMEM reads, 2 no TMA tile
# loads, 16 no producer A rows, 4 no MMAs, and combinations.
cd ${GRAFT_REPO_ROOT:-.}
for d in ${DBGS:-0 1 2 16 3 17 19 4}; do
  BZ_K4_DEBUG=$d python - "$d" <<'PY'
import sys
sys.path.insert(0, ".")
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.configs import code
from paper_1603_06757_b200.enumeration import family_words
G, gs, _ = code("cfg5", 7)
ctx = _native.context(0)
import os
ctx.set_engine(os.environ.get("ENGINE", "auto"))
ctx.load(family_words(gs.gammas, 160), 160)
ms = []
for i in range(4):
    ctx.round(8, -1, 18)
    if i: ms.append(ctx.last_kernel_ms())
print(f"{os.environ.get('ENGINE', 'auto')} debug {sys.argv[1]:>3}: g=8 {sorted(ms)[1]:.3f} ms")
PY
done

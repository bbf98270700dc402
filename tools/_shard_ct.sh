cd ${GRAFT_REPO_ROOT:-.}
for N in 1 8; do
python - $N <<'PY'
import os, sys
sys.path.insert(0, ".")
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.configs import code
from paper_1603_06757_b200.enumeration import family_words
N = int(sys.argv[1])
G, gs, _ = code("cfg5", 7)
ctx = _native.context(0)
ctx.load(family_words(gs.gammas, 160), 160)
ctx.round(8, 16, 18, 0, N)
print("N", N, "normal kernel ms", ctx.last_kernel_ms())
os.environ["BZ_K4_DEBUG"] = "32"
os.environ["BZ_K4_CTRACE"] = f"gpurun_out/ct_{N}.bin"
ctx.round(8, 16, 18, 0, N)
print("N", N, "ctrace kernel ms", ctx.last_kernel_ms())
PY
python tools/chunk_times.py gpurun_out/ct_$N.bin
done

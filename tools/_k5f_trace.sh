# per-tile timelines of config 5's g = 8 round, K5q and K5f (trace build)
cd ${GRAFT_REPO_ROOT:-.}
export BZ_LIB=$PWD/tools/libbz_trace.so
for e in mxf4q mxf4f; do
  python - $e <<'PY'
import os, sys
sys.path.insert(0, ".")
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.configs import code
from paper_1603_06757_b200.enumeration import family_words
eng = sys.argv[1]
G, gs, _ = code("cfg5", 7)
ctx = _native.context(0)
ctx.set_engine(eng)
ctx.load(family_words(gs.gammas, 160), 160)
ctx.round(8, 0, 18)
os.environ["BZ_K4_DEBUG"] = "8"
os.environ["BZ_K4_TRACE_FROM"] = "3000"
os.environ["BZ_K4_TRACE_OUT"] = f"gpurun_out/tr_{eng}.bin"
print(eng, ctx.round(8, 0, 18), ctx.last_kernel_ms())
PY
  python tools/trace_view.py gpurun_out/tr_$e.bin 100 24
done

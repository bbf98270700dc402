# A/B of library builds on one box: bench step time, per-round kernel times
# and the config-4 / standalone g=5 launches, each build twice, interleaved.
#   bash tools/ab_libs.sh lib1.so lib2.so ...
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do
for lib in "$@"; do
BZ_LIB=$lib python bench.py --no-extra --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null
BZ_LIB=$lib python - "$lib" <<'PY'
import json, sys
sys.path.insert(0, ".")
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.configs import code, microbench_gamma
from paper_1603_06757_b200.enumeration import family_words
ctx = _native.context(0)
def t(fn, n=5):
    ms = []
    for i in range(n + 1):
        fn()
        if i: ms.append(ctx.last_kernel_ms())
    return round(sorted(ms)[n // 2] * 1e3, 1)
ctx.load(family_words([microbench_gamma(1)], 192), 192)
c4 = t(lambda: ctx.enumerate(0, 6))
G, gs, _ = code("cfg5", 7)
ctx.load(family_words(gs.gammas, 160), 160)
g5 = t(lambda: ctx.round(5, 0, 1 << 20))
print(f"{sys.argv[1]:40s} step {d['ms_per_step']:.4f} ms  e2e {d['e2e']['wall_s']*1e3:.3f} ms  rounds "
      f"{[(r['g'], round(r['kernel_ms'] * 1e3, 1)) for r in d['rounds'][4:]]}  cfg4 {c4} us  g5-loose {g5} us", flush=True)
PY
done; done

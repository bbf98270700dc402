"""A/B of library builds x engines on config 5 (g = 8 alone, rounds 1..8):
    python tools/_ab_engines.py lib1.so lib2.so ...   (ENGINES=mxf4q,mxf4f)"""
import os, subprocess, sys
libs = sys.argv[1:]
engines = os.environ.get("ENGINES", "mxf4q,mxf4f").split(",")
code = r'''
import os, sys
sys.path.insert(0, ".")
from paper_1603_06757_b200 import _native
from paper_1603_06757_b200.configs import code
from paper_1603_06757_b200.enumeration import family_words
G, gs, _ = code("cfg5", 7)
ctx = _native.context(0)
ctx.set_engine(sys.argv[1])
ctx.load(family_words(gs.gammas, 160), 160)
ms = []
for i in range(8):
    r = ctx.round(8, -1, 18)
    if i: ms.append(ctx.last_kernel_ms())
print(f"{os.environ['BZ_LIB']:40s} {sys.argv[1]:6s} g=8 {sorted(ms)[3]:.4f} ms (min {min(ms):.4f}) {r[0]}")
'''
for rep in range(2):
    for lib in libs:
        for e in engines:
            env = dict(os.environ, BZ_LIB=os.path.abspath(lib))
            subprocess.run([sys.executable, "-c", code, e], env=env, check=False)

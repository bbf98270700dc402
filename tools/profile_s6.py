"""One round of a section-6 code for ncu: python tools/profile_s6.py NAME G"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1603_06757_b200 import BitMatrix, _native  # noqa: E402
from paper_1603_06757_b200.enumeration import family_words  # noqa: E402
from paper_1603_06757_b200.gf2 import build_gamma_set  # noqa: E402
name, g = sys.argv[1], int(sys.argv[2])
fx = [c for c in json.load(open(os.path.join(ROOT, "tests/golden/section6_codes.json")))["codes"]
      if c["name"] == name][0]
G = BitMatrix([int(r, 16) for r in fx["rows"]], fx["n"])
gs = build_gamma_set(G)
ctx = _native.context(0)
for a in sys.argv[3:]:
    if a.startswith("--engine="):
        ctx.set_engine(a.split("=", 1)[1])
ctx.load(family_words(gs.gammas, G.num_cols), G.num_cols)
res = ctx.round(g, 0, fx["paper_d"] + 1)
print(name, g, res, ctx.last_kernel_ms(), "ms")

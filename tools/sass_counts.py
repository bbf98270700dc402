"""Per-kernel SASS instruction counts of libbz.so (static, from
cuobjdump -sass): the tcgen05 family (UTC*MMA = tcgen05.mma, UTCBAR =
tcgen05.commit, LDTM / STTM = tcgen05.ld / st), the TMA bulk copy (UBLKCP),
the mbarrier family (SYNCS.*) and the integer pipes of the XOR+POPC kernels
(POPC, LOP3).  Writes a JSON summary.

    python tools/sass_counts.py [libbz.so] [out.json]
"""
import json
import re
import subprocess
import sys
from collections import Counter, defaultdict

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1603_06757_b200/libbz.so"
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/r2_sass_counts.json"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
keep = re.compile(r"^(UTC\w*MMA|UTCBAR|LDTM|STTM|UBLKCP|SYNCS|POPC|LOP3|ELECT|UTCATOMSWS)")
counts = defaultdict(Counter)
name = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]+)", line)
    if name and m and keep.match(m.group(1)):
        counts[name][m.group(1)] += 1
demangled = {}
if counts:
    dm = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout
    demangled = dict(zip(counts, dm.splitlines()))
res = {"library": lib, "source": "cuobjdump -sass (static instruction counts)",
       "kernels": {demangled.get(k, k): dict(sorted(v.items())) for k, v in sorted(counts.items())}}
with open(out, "w") as fh:
    json.dump(res, fh, indent=1)
for k, v in res["kernels"].items():
    if "k4_round_umma" in k or "k1_" in k:
        print(k, {x: c for x, c in v.items() if not x.startswith("SYNCS")})

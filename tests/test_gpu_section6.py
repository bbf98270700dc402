"""The paper's section-6 codes to their exact minimum distances on the GPU.

C1 = [234,51] and C2 = [234,52] (matrix-product codes of the paper's
polynomials), their extensions and punctures (tests/golden/
section6_codes.json, built by the reference package) -- the paper's new
codes, whose distances it reports after runs of 1.3e5 to 2.3e5 s on one
core (section 6 tables).  Every run here must end exact, at the
paper's distance, with a consistent trace (L >= U only at the end).
"""

from __future__ import annotations

import pytest

from conftest import hexrows
from paper_1603_06757_b200 import BitMatrix, EngineConfig, minimum_distance

pytestmark = pytest.mark.gpu


def test_section6_distances(section6):
    for fx in section6["codes"]:
        G = BitMatrix(hexrows(fx["rows"]), fx["n"])
        rep = minimum_distance(G, EngineConfig())
        assert rep.status == "exact", fx["name"]
        assert rep.distance == fx["paper_d"], (fx["name"], rep.distance)
        g, L, U = rep.bounds_trace[-1]
        assert L >= U == rep.distance
        assert all(l < u for (_, l, u) in rep.bounds_trace[:-1])
        assert [t[0] for t in rep.bounds_trace] == list(range(1, g + 1))

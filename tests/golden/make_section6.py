"""The paper's section-6 codes, built by the REFERENCE package.

Test infrastructure only (build container): imports the reference's
``mindist.constructions`` and the section-6 polynomial exponent lists of
its acceptance test (pkg/tests/test_acceptance.py), builds C1 = [234,51]
and C2 = [234,52] with the matrix-product construction and their extended
/ punctured relatives exactly as that test does, and writes the generator
rows (hex, bit j = column j) with the distances the paper reports for
them (section 6 tables) to tests/golden/section6_codes.json.

    python tests/golden/make_section6.py
"""

from __future__ import annotations

import json
import os
import sys
import warnings

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from mindist.constructions import (  # noqa: E402  (reference package)
    cyclic_code_generator, extend_code, matrix_product_code, poly_divmod,
    poly_from_exponents, poly_mod_ring, puncture_code, ring_modulus)
import test_acceptance as acc  # noqa: E402  (the reference's own test module)

HERE = os.path.dirname(os.path.abspath(__file__))

# distances the paper reports for these codes (section 6 tables)
PAPER_D = {"C1": 63, "C2": 62, "C3": 64, "C4": 64, "C5": 62, "C5b": 61, "C5c": 61}


def main():
    m = 117
    f1 = poly_from_exponents(acc.F1_EXPS)
    f2_c1, _ = poly_divmod(ring_modulus(m), poly_from_exponents([1, 0]))
    f2_c2, _ = poly_divmod(ring_modulus(m), poly_from_exponents([2, 1, 0]))
    p1 = poly_mod_ring(poly_from_exponents(acc.P1_EXPS), m)
    p2 = poly_mod_ring(poly_from_exponents(acc.P2_EXPS), m)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        c1 = matrix_product_code(cyclic_code_generator(f1, m),
                                 cyclic_code_generator(f2_c1, m), p1, m)
    c2 = matrix_product_code(cyclic_code_generator(f1, m),
                             cyclic_code_generator(f2_c2, m), p2, m)
    c3 = extend_code(c1)
    codes = {"C1": c1, "C2": c2, "C3": c3, "C4": extend_code(c3),
             "C5": puncture_code(c1, {233}), "C5b": puncture_code(c1, {233, 232}),
             "C5c": puncture_code(c2, {233})}
    out = {"m": m, "f1_exps": acc.F1_EXPS, "p1_exps": acc.P1_EXPS, "p2_exps": acc.P2_EXPS,
           "codes": [{"name": name, "n": G.num_cols, "k": G.num_rows,
                      "rows": [format(r, "x") for r in G.rows], "paper_d": PAPER_D[name]}
                     for name, G in codes.items()]}
    with open(os.path.join(HERE, "section6_codes.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for c in out["codes"]:
        print(c["name"], c["n"], c["k"], c["paper_d"])


if __name__ == "__main__":
    main()

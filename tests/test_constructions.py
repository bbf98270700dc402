"""Section-6 constructions (paper_1603_06757_b200.constructions) against the
reference's: the same polynomial arithmetic identities its acceptance test
checks and bit-identical generator matrices for C1..C5c
(tests/golden/section6_codes.json, made by make_section6.py from the
reference package)."""

from __future__ import annotations

import warnings

import pytest

from conftest import hexrows
from paper_1603_06757_b200.constructions import (
    NotADivisor, NotAUnit, cyclic_code_generator, extend_code, is_subcode, is_unit,
    matrix_product_code, poly_degree, poly_divmod, poly_from_exponents, poly_gcd,
    poly_mod_ring, poly_mul, poly_mul_mod, puncture_code, ring_modulus)


def build(section6):
    m = section6["m"]
    f1 = poly_from_exponents(section6["f1_exps"])
    f2_c1, _ = poly_divmod(ring_modulus(m), poly_from_exponents([1, 0]))
    f2_c2, _ = poly_divmod(ring_modulus(m), poly_from_exponents([2, 1, 0]))
    p1 = poly_mod_ring(poly_from_exponents(section6["p1_exps"]), m)
    p2 = poly_mod_ring(poly_from_exponents(section6["p2_exps"]), m)
    with pytest.warns(UserWarning, match="not nested"):
        c1 = matrix_product_code(cyclic_code_generator(f1, m),
                                 cyclic_code_generator(f2_c1, m), p1, m)
    with warnings.catch_warnings():
        warnings.simplefilter("error")  # the nested pair must not warn
        c2 = matrix_product_code(cyclic_code_generator(f1, m),
                                 cyclic_code_generator(f2_c2, m), p2, m)
    c3 = extend_code(c1)
    return {"C1": c1, "C2": c2, "C3": c3, "C4": extend_code(c3),
            "C5": puncture_code(c1, {233}), "C5b": puncture_code(c1, {233, 232}),
            "C5c": puncture_code(c2, {233})}


def test_polynomial_identities(section6):
    m = section6["m"]
    f1 = poly_from_exponents(section6["f1_exps"])
    assert poly_degree(f1) == 67
    q, r = poly_divmod(ring_modulus(m), f1)
    assert r == 0 and poly_mul(q, f1) == ring_modulus(m)
    for e in ("p1_exps", "p2_exps"):
        p = poly_mod_ring(poly_from_exponents(section6[e]), m)
        assert is_unit(p, m) and poly_degree(p) < m
    assert poly_gcd(0b110, 0b11) == 0b11
    assert poly_mul_mod(1 << (m - 1), 0b10, m) == 1  # x^(m-1) * x = x^m = 1
    assert not is_unit(0b11, m)                      # x + 1 divides x^m - 1


def test_section6_matrices_match_reference(section6):
    codes = build(section6)
    for fx in section6["codes"]:
        G = codes[fx["name"]]
        assert (G.num_cols, G.num_rows) == (fx["n"], fx["k"]), fx["name"]
        assert list(G.rows) == hexrows(fx["rows"]), fx["name"]


def test_construction_errors():
    m = 7
    with pytest.raises(NotADivisor):
        cyclic_code_generator(0b111, m)          # x^2+x+1 does not divide x^7-1
    g = cyclic_code_generator(0b1011, m)         # the [7,4] Hamming code
    assert (g.num_rows, g.num_cols) == (4, 7)
    with pytest.raises(NotAUnit):
        matrix_product_code(g, g, 0b11, m)
    assert is_subcode(g, g)

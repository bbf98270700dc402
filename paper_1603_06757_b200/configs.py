"""Seeded synthetic inputs of BASELINE.json's five configurations.

Generator (shared by the oracle goldens and the GPU
runs): ``random.Random(seed)``, one ``getrandbits(n)`` per row (bit j =
column j, i.i.d. Bernoulli(1/2) entries), redraw the whole matrix -- the
same RNG stream continuing -- until ``build_gamma_set`` yields the target
(full-rank count, remainder rank).  Config 4 is the reference's own
``random_systematic_matrix(64, 192, seed)`` = [I_64 | A] (gf2.py:202-215).
The paper's own matrices are not available; these seeded
draws with the configs' shapes stand in for them.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

from .errors import RankDeficient
from .gf2 import BitMatrix, build_gamma_set, random_systematic_matrix


@dataclass(frozen=True)
class CodeConfig:
    name: str
    k: int
    n: int
    target: tuple[int, int]  # (full_rank_count, remainder_rank)
    seeds: tuple[int, ...]
    desc: str


CONFIGS = {
    "cfg1": CodeConfig("cfg1", 24, 48, (2, 0), (1, 2), "random [48,24], 2 full sets"),
    "cfg2": CodeConfig("cfg2", 48, 96, (2, 0), (1, 2), "random [96,48], 2 full sets"),
    "cfg3": CodeConfig("cfg3", 40, 100, (2, 20), (1, 2),
                       "random [100,40], 2 full sets + rank-20 remainder"),
    "cfg5": CodeConfig("cfg5", 80, 160, (2, 0), (7,), "random [160,80], 2 full sets"),
}


def draw_code(k: int, n: int, seed: int, target: tuple[int, int]):
    """(G, GammaSet, draws) for the first draw hitting `target`."""
    rng = random.Random(seed)
    draws = 0
    while True:
        draws += 1
        G = BitMatrix([rng.getrandbits(n) for _ in range(k)], n)
        try:
            gs = build_gamma_set(G)
        except RankDeficient:
            continue
        if (gs.full_rank_count, gs.remainder_rank) == target:
            return G, gs, draws


def code(name: str, seed: int | None = None):
    c = CONFIGS[name]
    return draw_code(c.k, c.n, c.seeds[0] if seed is None else seed, c.target)


def microbench_gamma(seed: int = 1) -> BitMatrix:
    """Config 4: systematic 64x192 Gamma = [I_64 | A]."""
    return random_systematic_matrix(64, 192, seed)

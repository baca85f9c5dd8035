"""Seeded random streams (SURVEY.md §8(d) "Seed and stream legend").

``np.random.default_rng([seed, stream])`` with one stream id per kind of random
input, so that the oracle and the CUDA path see bit-identical inputs without
either side reimplementing a generator.
"""
import numpy as np

SIGMA = 0   # 256 jump-coefficient cells, 10**U, U ~ U[-3, 3]       (BASELINE C2)
XFAC = 1    # X factors of low-rank updates, N(0,1), column-major    (C0, C1)
YFAC = 2    # Y factors                                              (C0, C1)
BLOCKS = 3  # C1 block choices over admissible leaves                (C1)
RHS = 4     # PCG right-hand side b ~ N(0,1)                         (C2, C3)
POWER = 5   # power-iteration start vector                           (C2, C3)
PROBES = 6  # 16 probe vectors for operator parity                   (north_star)


def stream(kind: int, seed: int = 0) -> np.random.Generator:
    """Independent generator for one kind of random input."""
    return np.random.default_rng([int(seed), int(kind)])


def probes(n: int, count: int = 16, seed: int = 0) -> np.ndarray:
    """``count`` probe vectors of length n, shape (count, n), N(0,1)."""
    return stream(PROBES, seed).standard_normal((count, n))

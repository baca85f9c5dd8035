"""Seeded low-rank update streams (BASELINE C0/C1).

Only random numbers and block choices -- no arithmetic of the method.  Both the oracle and the
CUDA path consume exactly these arrays.
"""
import numpy as np

from .rng import stream, XFAC, YFAC, BLOCKS


def c1_stream(adm_targets, count: int, ku: int, seed: int = 0):
    """R16: `count` updates, block uniform over the admissible leaves (stream 3), fresh X_i, Y_i
    ~ N(0,1) drawn in sequence from streams 1 and 2.

    adm_targets: list of (t0, s0, |t0|, |s0|) for the admissible leaves in block-tree DFS order.
    Returns a list of (t0, s0, X, Y) with X: |t0| x ku, Y: |s0| x ku (float64, C-ordered)."""
    gb, gx, gy = stream(BLOCKS, seed), stream(XFAC, seed), stream(YFAC, seed)
    idx = gb.integers(0, len(adm_targets), size=count)
    out = []
    for i in idx:
        t0, s0, mt, ms = adm_targets[int(i)]
        X = gx.standard_normal((ku, mt)).T  # column-major draw
        Y = gy.standard_normal((ku, ms)).T
        out.append((int(t0), int(s0), np.ascontiguousarray(X), np.ascontiguousarray(Y)))
    return out


def c0_global_factors(n: int, k: int = 8, seed: int = 0):
    """R15: one global X, Y in R^{n x k} ~ N(0,1) (ORIGINAL order), applied with alpha = 1/n."""
    X = stream(XFAC, seed).standard_normal((k, n)).T
    Y = stream(YFAC, seed).standard_normal((k, n)).T
    return np.ascontiguousarray(X), np.ascontiguousarray(Y)


def mixed_stream(blocks, count: int, kmax: int, seed: int = 0):
    """Random updates on arbitrary block-tree nodes (edge cases: subdivided, admissible and
    inadmissible targets, ranks 1..kmax).  blocks: list of (t0, s0, |t0|, |s0|)."""
    g = np.random.default_rng([seed, 100])
    out = []
    for _ in range(count):
        t0, s0, mt, ms = blocks[int(g.integers(len(blocks)))]
        k = int(g.integers(1, kmax + 1))
        out.append((int(t0), int(s0), g.standard_normal((mt, k)), g.standard_normal((ms, k))))
    return out

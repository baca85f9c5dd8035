"""Seeded synthetic input generators shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the paper's method (no trees, no bases, no
updates, no factorizations).  It only produces the model problems of PAPER.md §7
(P1 FEM on the unit square; BASELINE.json configs C0-C4) and the
random numbers the experiments draw (SURVEY.md §8(d) seed/stream legend).
"""
from .rng import stream, SIGMA, XFAC, YFAC, BLOCKS, RHS, POWER, PROBES  # noqa: F401
from .fem import (  # noqa: F401
    grid_points_2d,
    grid_points_3d,
    fem2d_csr,
    fem3d_kuhn_csr,
    jump_sigma_cells,
    config,
)

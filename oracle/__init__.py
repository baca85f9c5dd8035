"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU (numpy, float64) implementation of what the
paper's H^2 hot path computes (PAPER.md = arXiv 1402.5056; P:n = PAPER.md line n).
It exists to prove the CUDA path right.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_1402_5056_b200``) never imports, calls or links anything
here, and this package shares no code with it (inputs come from ``inputs/``).

Modules
  structure  cluster tree / block tree / row(t), pred(t)
  h2         H^2 representation, from_sparse, densify, matvec
  update     local low-rank update (O1, the paper's algorithm)
  dense      O2: dense brute-force definitions that pin O1
  arith      product, substitution, LR/Cholesky, PCG

Library primitives used as single steps: numpy.linalg.qr (thin QR), numpy.linalg.svd,
numpy.linalg.cholesky, scipy.linalg.solve_triangular, matrix products.

Parity pins (what holds the oracle to something other than itself) live in
tests/test_oracle_*.py; every function whose result is not pinned says so.
"""

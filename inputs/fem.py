"""Synthetic FEM model problems shaped like PAPER.md §7 and BASELINE.json C0-C4.

2D: P1 Galerkin FEM of -div(sigma grad u) = f on the unit square, zero Dirichlet
BC, N x N interior nodes, h = 1/(N+1), every mesh square split by its SW-NE
diagonal.  On a right triangle with legs along the axes the
P1 element stiffness is h-independent:

    K = sigma_T/2 * [[2,-1,-1],[-1,1,0],[-1,0,1]]   (vertex order: right angle, x-leg, y-leg)

so axis edges get -(sigma_T1 + sigma_T2)/2, hypotenuse couplings vanish and the
constant-coefficient matrix is the 5-point stencil (4, -1).

3D: P1 on the 6-tetrahedron Kuhn subdivision of the cube grid gives the 7-point
stencil h*(6, -1); generated directly as that stencil.

Node (i, j) (1-based grid indices, i along x) has ORIGINAL index (j-1)*N + (i-1);
its point coordinates are the integer grid indices, so every geometric predicate
of the cluster/block tree is exact.
"""
import numpy as np
import scipy.sparse as sp

from .rng import stream, SIGMA


def grid_points_2d(N: int) -> np.ndarray:
    """(n, 2) float64 integer-valued grid coordinates in original order."""
    j, i = np.meshgrid(np.arange(1, N + 1), np.arange(1, N + 1), indexing="ij")
    return np.stack([i.ravel(), j.ravel()], axis=1).astype(np.float64)


def grid_points_3d(N: int) -> np.ndarray:
    k, j, i = np.meshgrid(np.arange(1, N + 1), np.arange(1, N + 1), np.arange(1, N + 1), indexing="ij")
    return np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.float64)


def jump_sigma_cells(seed: int = 0, cells: int = 16) -> np.ndarray:
    """BASELINE C2: sigma piecewise constant on a cells x cells checkerboard, 10**U, U~U[-3,3].

    Returned as (cells, cells) array indexed [cy, cx] (cell index 16*cy + cx)."""
    return (10.0 ** stream(SIGMA, seed).uniform(-3.0, 3.0, cells * cells)).reshape(cells, cells)


def fem2d_csr(N: int, sigma_cells: np.ndarray | None = None):
    """Assemble the 2D P1 stiffness matrix; returns scipy CSR (float64, sorted indices).

    sigma_cells=None gives sigma = 1 (the plain Laplacian of C0/C1)."""
    M = N + 1  # squares per axis
    # lower-left corners (a, b) of every mesh square, a, b in 0..N
    b, a = np.meshgrid(np.arange(M), np.arange(M), indexing="ij")
    a = a.ravel()
    b = b.ravel()
    if sigma_cells is None:
        s_low = np.ones(a.shape)
        s_up = np.ones(a.shape)
    else:
        C = sigma_cells.shape[0]
        # centroids: T_low = {(a,b),(a+1,b),(a+1,b+1)} -> ((3a+2)h/3, (3b+1)h/3)
        #            T_up  = {(a,b),(a,b+1),(a+1,b+1)} -> ((3a+1)h/3, (3b+2)h/3)
        # cell = floor(C * x_c) computed exactly in integers (never on an edge, R18)
        cx_lo = (C * (3 * a + 2)) // (3 * M)
        cy_lo = (C * (3 * b + 1)) // (3 * M)
        cx_up = (C * (3 * a + 1)) // (3 * M)
        cy_up = (C * (3 * b + 2)) // (3 * M)
        s_low = sigma_cells[cy_lo, cx_lo]
        s_up = sigma_cells[cy_up, cx_up]

    def node(ii, jj):
        inside = (ii >= 1) & (ii <= N) & (jj >= 1) & (jj <= N)
        return np.where(inside, (jj - 1) * N + (ii - 1), -1)

    rows, cols, vals = [], [], []
    # T_low: right angle at (a+1, b); x-leg vertex (a, b); y-leg vertex (a+1, b+1)
    # T_up : right angle at (a, b+1); x-leg vertex (a+1, b+1); y-leg vertex (a, b)
    Kloc = 0.5 * np.array([[2.0, -1.0, -1.0], [-1.0, 1.0, 0.0], [-1.0, 0.0, 1.0]])
    for verts, sig in (
        (((a + 1, b), (a, b), (a + 1, b + 1)), s_low),
        (((a, b + 1), (a + 1, b + 1), (a, b)), s_up),
    ):
        ids = [node(np.asarray(v[0]), np.asarray(v[1])) for v in verts]
        for p in range(3):
            for q in range(3):
                if Kloc[p, q] == 0.0:
                    continue
                m = (ids[p] >= 0) & (ids[q] >= 0)
                rows.append(ids[p][m])
                cols.append(ids[q][m])
                vals.append(Kloc[p, q] * sig[m])
    n = N * N
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()
    A.sum_duplicates()
    A.eliminate_zeros()
    A.sort_indices()
    return A


def fem3d_kuhn_csr(N: int):
    """3D P1 Laplacian on Kuhn-subdivided cubes == 7-point stencil h*(6,-1), h=1/(N+1)."""
    h = 1.0 / (N + 1)
    n = N ** 3
    idx = np.arange(n)
    i = idx % N
    j = (idx // N) % N
    k = idx // (N * N)
    rows = [idx]
    cols = [idx]
    vals = [np.full(n, 6.0 * h)]
    for di, dj, dk in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        ii, jj, kk = i + di, j + dj, k + dk
        m = (ii >= 0) & (ii < N) & (jj >= 0) & (jj < N) & (kk >= 0) & (kk < N)
        rows.append(idx[m])
        cols.append((kk * N * N + jj * N + ii)[m])
        vals.append(np.full(int(m.sum()), -h))
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()
    A.sort_indices()
    return A


# BASELINE.json configs (0-based), SURVEY.md §8(d) table.
_CONFIGS = {
    "C0": dict(dim=2, N=32, leaf=32, eta=2.0, eps=1e-4, jump=False),
    "C1": dict(dim=2, N=128, leaf=32, eta=2.0, eps=None, max_rank=16, jump=False),
    "C2": dict(dim=2, N=512, leaf=32, eta=2.0, eps=1e-4, jump=True),
    "C3": dict(dim=3, N=64, leaf=64, eta=2.0, eps=1e-4, jump=False),
    "C4": dict(dim=2, N=1024, leaf=32, eta=2.0, eps=1e-4, jump=True),
}


def config(name: str, seed: int = 0, N: int | None = None) -> dict:
    """Points + CSR + parameters of a BASELINE config (N may be overridden for scaled-down variants)."""
    c = dict(_CONFIGS[name])
    if N is not None:
        c["N"] = N
    if c["dim"] == 2:
        pts = grid_points_2d(c["N"])
        A = fem2d_csr(c["N"], jump_sigma_cells(seed) if c["jump"] else None)
    else:
        pts = grid_points_3d(c["N"])
        A = fem3d_kuhn_csr(c["N"])
    c.update(name=name, n=pts.shape[0], points=pts, A=A, seed=seed)
    return c

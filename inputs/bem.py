"""Synthetic BEM model problem shaped like PAPER.md's second experiment (Table 2):
the Galerkin matrix of the single layer potential operator on a circle, piecewise constant basis
functions on a regular mesh of n arcs.  Workload generation only: the kernel, its
Galerkin entries and degenerate-kernel (interpolation) factors of far-field blocks.  None of the
method's arithmetic (trees, bases, updates, factorizations) lives here; the oracle and the CUDA
path both consume exactly these arrays.

Reading own-12 (the paper says only "single layer potential operator on the two-dimensional unit
circle using a regular mesh and piecewise constant basis functions"):
  * curve: the circle of radius r = 1/2 -- on the circle of radius 1 the operator annihilates the
    constants (logarithmic capacity 1: the Galerkin matrix is exactly singular, no Cholesky
    factorization exists), so "unit" is read as the diameter;
  * x(theta) = r (cos theta, sin theta), arcs [i h, (i+1) h), h = 2 pi / n, basis = indicators,
        G_ij = -(1/2pi) int_{arc i} int_{arc j} log|x - y| ds_x ds_y,   ds = r dtheta;
  * |x(theta) - y(phi)| = 2 r |sin((theta - phi)/2)| and log(2|sin(psi/2)|) = -sum_{m>=1} cos(m psi)/m,
    so G is the symmetric circulant matrix with first row
        g(d) = r^2 [ -h^2 log(r) / (2pi) + (2/pi) sum_{m>=1} sin^2(m h / 2) cos(m d h) / m^3 ],
    evaluated EXACTLY (to rounding) by folding m mod n: sin^2(m h/2) = sin^2(pi p/n) for m = p + q n,
    sum_q (p + q n)^-3 = zeta(3, p/n) / n^3 (Hurwitz zeta), and one real FFT over p.
Point of arc i (for the cluster tree): its midpoint, scaled to integer-free doubles.

Far-field factors: for a block (t, s) of arcs with separated angle ranges, interpolation of the
kernel in theta over t's angle interval at m Chebyshev nodes theta_v gives
    G|_{t x s} ~ X Y^T,  X[i, v] = int_{arc i} L_v(theta) dtheta (exact Gauss-Legendre),
    Y[j, v] = -(r^2 / 2pi) int_{arc j} [log r + log(2|sin((theta_v - phi)/2)|)] dphi (Gauss-Legendre;
    the integrand is analytic because the ranges are separated).
"""
import numpy as np
import scipy.sparse as sp
from scipy.special import zeta

R = 0.5


def circle_points(n: int) -> np.ndarray:
    """(n, 2) midpoints of the n arcs, original order = arc index."""
    th = (np.arange(n) + 0.5) * (2.0 * np.pi / n)
    return np.stack([R * np.cos(th), R * np.sin(th)], axis=1)


def first_row(n: int) -> np.ndarray:
    """g(d), d = 0..n-1: first row of the circulant Galerkin matrix (see the module docstring)."""
    h = 2.0 * np.pi / n
    p = np.arange(1, n)
    a = np.zeros(n)
    a[1:] = np.sin(np.pi * p / n) ** 2 * zeta(3.0, p / n) / float(n) ** 3  # folded coefficients, p = 1..n-1
    # sum_p a_p cos(2 pi p d / n) = Re FFT(a)[d]
    series = np.real(np.fft.fft(a))
    return R * R * (-h * h * np.log(R) / (2.0 * np.pi) + (2.0 / np.pi) * series)


def dense_matrix(n: int) -> np.ndarray:
    """The full Galerkin matrix (pins and small cases only)."""
    g = first_row(n)
    idx = (np.arange(n)[None, :] - np.arange(n)[:, None]) % n
    return g[idx]


def nearfield_csr(n: int, pairs) -> sp.csr_matrix:
    """Sparse matrix (original order) holding the exact Galerkin entries of the given index blocks.
    pairs: iterable of (rows, cols) integer arrays (original indices) -- the inadmissible leaves."""
    g = first_row(n)
    ri, ci, vv = [], [], []
    for rows, cols in pairs:
        rr, cc = np.meshgrid(rows, cols, indexing="ij")
        ri.append(rr.ravel())
        ci.append(cc.ravel())
        vv.append(g[(cc.ravel() - rr.ravel()) % n])
    A = sp.csr_matrix((np.concatenate(vv), (np.concatenate(ri), np.concatenate(ci))), shape=(n, n))
    A.sort_indices()
    return A


def _angle_interval(n: int, idx: np.ndarray):
    """Smallest angle interval [a, b] covering the arcs idx (handles the wrap at 2 pi)."""
    h = 2.0 * np.pi / n
    srt = np.sort(np.asarray(idx))
    gaps = np.diff(np.concatenate([srt, [srt[0] + n]]))
    j = int(np.argmax(gaps))  # the largest gap between consecutive arcs: the interval starts after it
    start = srt[(j + 1) % len(srt)]
    length = n - gaps[j] + 1
    return start * h, (start + length) * h


def far_factors(n: int, rows: np.ndarray, cols: np.ndarray, m: int = 12, gauss: int = 8):
    """Interpolation factors X (|rows| x m), Y (|cols| x m) with G[rows][:, cols] ~ X Y^T."""
    h = 2.0 * np.pi / n
    a, b = _angle_interval(n, rows)
    v = np.arange(m)
    nodes = 0.5 * (a + b) + 0.5 * (b - a) * np.cos((2 * v + 1) * np.pi / (2 * m))  # Chebyshev nodes
    gx, gw = np.polynomial.legendre.leggauss(gauss)
    # X[i, v] = int_{arc i} L_v(theta) dtheta; arcs unwrapped into [a, b]
    th0 = (np.asarray(rows) * h - a) % (2.0 * np.pi) + a
    tq = th0[:, None] + 0.5 * h * (gx[None, :] + 1.0)  # (|rows|, gauss)
    L = np.ones((len(rows), gauss, m))
    for vv in range(m):
        for u in range(m):
            if u != vv:
                L[:, :, vv] *= (tq - nodes[u]) / (nodes[vv] - nodes[u])
    X = 0.5 * h * np.einsum("igv,g->iv", L, gw)
    # Y[j, v] = -(R^2/2pi) int_{arc j} [log R + log(2 |sin((theta_v - phi)/2)|)] dphi
    pq = np.asarray(cols)[:, None] * h + 0.5 * h * (gx[None, :] + 1.0)  # (|cols|, gauss)
    K = np.log(R) + np.log(2.0 * np.abs(np.sin(0.5 * (nodes[None, None, :] - pq[:, :, None]))))
    Y = -(R * R / (2.0 * np.pi)) * 0.5 * h * np.einsum("jgv,g->jv", K, gw)
    return np.ascontiguousarray(X), np.ascontiguousarray(Y)


def pieces(n: int, perm, lo, hi, bt_t, bt_s, bt_kind, lower: bool = False, m: int = 12):
    """The workload in the shape the method consumes it, for a given cluster/block structure
    (arrays as exported by either side; they are bit-identical): the sparse matrix of the exact
    entries of the inadmissible leaves (kind 2) and, per admissible leaf (kind 1) in block order,
    (t, s, X, Y) with X, Y in TREE order of t / s.  lower: only blocks with lo[t] >= lo[s]."""
    near, far = [], []
    for t, s, k in zip(bt_t, bt_s, bt_kind):
        t, s = int(t), int(s)
        if lower and lo[t] < lo[s]:
            continue
        rows, cols = perm[lo[t]:hi[t]], perm[lo[s]:hi[s]]
        if k == 2:
            near.append((rows, cols))
        elif k == 1:
            X, Y = far_factors(n, rows, cols, m=m)
            far.append((t, s, X, Y))
    return nearfield_csr(n, near), far

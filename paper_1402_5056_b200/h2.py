"""ctypes binding of include/h2.h (argument marshalling only).

Host arrays are numpy; device arrays are torch CUDA tensors (data_ptr() is passed through);
streams are torch.cuda streams.  Dense matrices are column-major, as in the C ABI.
"""
import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, os.environ.get("H2_LIB_NAME", "libh2b200.so"))  # override: sanitizer builds (tools)

# every symbol include/h2.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = [
    "h2_cluster_tree", "h2_cluster_tree_dd", "h2_tree_ddpair", "h2_tree_export", "h2_tree_destroy",
    "h2_block_tree", "h2_btree_export", "h2_btree_destroy",
    "h2_from_sparse", "h2_lowrank_update", "h2_matvec", "h2_addmul", "h2_lr_factor", "h2_solve",
    "h2_ranks", "h2_storage_report", "h2_export", "h2_check_device_flags",
    "h2_profile_enable", "h2_profile_read", "h2_profile_debug", "h2_profile_ops", "h2_stats", "h2_pcg", "h2_launch_count",
    "h2_mat_destroy", "h2_last_error", "h2_batch_begin", "h2_batch_end", "h2_inverse", "h2_import",
]

if not os.path.exists(_LIBPATH):
    raise ImportError(f"libh2b200.so not built ({_LIBPATH}); run `python paper_1402_5056_b200/build.py` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(_LIBPATH)


def library_path() -> str:
    return _LIBPATH


_p = C.c_void_p
_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double
_sig = {
    "h2_cluster_tree": [_p, _i64, _i32, _i32, C.POINTER(_p)],
    "h2_cluster_tree_dd": [_p, _i64, _i32, _i32, _p, _p, C.POINTER(_p)],
    "h2_tree_ddpair": [_p, _p],
    "h2_tree_export": [_p, _p, _p, _p, _p, _p, _p, _p],
    "h2_tree_destroy": [_p],
    "h2_block_tree": [_p, _p, _f64, C.POINTER(_p)],
    "h2_btree_export": [_p, _p, _p, _p, _p, _p],
    "h2_btree_destroy": [_p],
    "h2_from_sparse": [_p, _i64, _p, _p, _p, C.c_int, _i32, _i32, _p, C.POINTER(_p)],
    "h2_lowrank_update": [_p, _i32, _i32, _i32, _f64, _p, _i64, _p, _i64, _p, _p],
    "h2_matvec": [_p, _i32, _f64, _p, _f64, _p, _p],
    "h2_addmul": [_p, _f64, _p, _p, _p, _p],
    "h2_lr_factor": [_p, C.c_int, _p, _p],
    "h2_solve": [_p, _p, _i32, _i64, _p],
    "h2_ranks": [_p, _p, _p],
    "h2_storage_report": [_p, _p],
    "h2_export": [_p, _p, _p, _p, _p, _p, _p, _p],
    "h2_check_device_flags": [_p, _p],
    "h2_profile_enable": [_i32],
    "h2_stats": [_p, _p],
    "h2_profile_debug": [_p],
    "h2_profile_ops": [_p, _p, _i32, _p],
    "h2_pcg": [_p, _p, _p, _p, _f64, _i32, _p, _p, _p],
    "h2_launch_count": [_p],
    "h2_profile_read": [_p, _p, _p, _p, _p, _p],
    "h2_mat_destroy": [_p],
    "h2_last_error": [],
    "h2_batch_begin": [_p],
    "h2_batch_end": [],
    "h2_inverse": [_p, _p, _p],
    "h2_import": [_p, _p, _p, _p, _p, _p, _p, _p, _p, C.c_int, _i32, _i32, _p, C.POINTER(_p)],
}
for _name, _args in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = None if _name.endswith("_destroy") else (C.c_char_p if _name == "h2_last_error" else C.c_int)

STATUS = {0: "H2_OK", 1: "H2_ERR_ARG", 2: "H2_ERR_SHAPE", 3: "H2_ERR_STRUCTURE", 4: "H2_ERR_NONFINITE",
          5: "H2_ERR_BREAKDOWN", 6: "H2_ERR_NOMEM", 7: "H2_ERR_CUDA", 8: "H2_ERR_UNSUPPORTED",
          9: "H2_ERR_NOCONV"}


class H2Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def _check(code):
    if code != 0:
        raise H2Error(code, _lib.h2_last_error().decode())


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(_p)
    return _p(a.data_ptr())  # torch tensor


def _stream(stream):
    if stream is None:
        import torch
        return _p(torch.cuda.current_stream().cuda_stream)
    return _p(getattr(stream, "cuda_stream", stream))


@dataclass
class Trunc:
    """h2_trunc (reading SURVEY R5; blockwise: P:874-879, reading own-10)."""
    rel_tol: float = 1e-4
    abs_tol: float = 0.0
    max_rank: int = 0
    blockwise: bool = False


class _CTrunc(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("abs_tol", C.c_double), ("max_rank", C.c_int32),
                ("blockwise", C.c_int32)]


def _ctrunc(tr):
    tr = tr or Trunc()
    return _CTrunc(float(tr.rel_tol), float(tr.abs_tol), int(tr.max_rank), int(bool(tr.blockwise)))


class Tree:
    """h2_tree handle plus its exported arrays (perm, lo, hi, son0, son1, level)."""

    def __init__(self, handle, n):
        self.h = _p(handle)
        self.n = n
        nc = _i32()
        _check(_lib.h2_tree_export(self.h, None, None, None, None, None, None, C.byref(nc)))
        self.nclusters = nc.value
        self.perm = np.empty(n, dtype=np.int64)
        self.lo, self.hi, self.son0, self.son1, self.level = (np.empty(self.nclusters, dtype=np.int32) for _ in range(5))
        _check(_lib.h2_tree_export(self.h, _ptr(self.perm), _ptr(self.lo), _ptr(self.hi), _ptr(self.son0),
                                   _ptr(self.son1), _ptr(self.level), C.byref(nc)))
        self.ddpair = np.zeros(self.nclusters, dtype=np.int8)
        _check(_lib.h2_tree_ddpair(self.h, _ptr(self.ddpair)))

    def size(self, t):
        return int(self.hi[t] - self.lo[t])

    def __del__(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.h2_tree_destroy(self.h)
            self.h = None


class BlockTree:
    def __init__(self, handle, rows: Tree, cols: Tree):
        self.h = _p(handle)
        self.rows, self.cols = rows, cols  # keep the trees alive
        nb, csp = _i64(), _i32()
        _check(_lib.h2_btree_export(self.h, None, None, None, C.byref(nb), C.byref(csp)))
        self.nblocks, self.csp = nb.value, csp.value
        self.t = np.empty(self.nblocks, dtype=np.int32)
        self.s = np.empty(self.nblocks, dtype=np.int32)
        self.kind = np.empty(self.nblocks, dtype=np.int8)
        _check(_lib.h2_btree_export(self.h, _ptr(self.t), _ptr(self.s), _ptr(self.kind), C.byref(nb), None))

    def __del__(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.h2_btree_destroy(self.h)
            self.h = None


class Mat:
    def __init__(self, handle, bt: BlockTree, storage, rank_cap, update_cap):
        self.h = _p(handle)
        self.bt = bt
        self.storage, self.rank_cap, self.update_cap = storage, rank_cap, update_cap
        self.n = bt.rows.n

    def __del__(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.h2_mat_destroy(self.h)
            self.h = None


def h2_cluster_tree(points: np.ndarray, leaf_size: int) -> Tree:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    h = _p()
    _check(_lib.h2_cluster_tree(_ptr(pts), pts.shape[0], pts.shape[1], int(leaf_size), C.byref(h)))
    return Tree(h.value, pts.shape[0])


def h2_cluster_tree_dd(points: np.ndarray, leaf_size: int, A) -> Tree:
    """Domain-decomposition cluster tree (NEXT-3); A: scipy.sparse matrix whose
    pattern is the coupling graph (ORIGINAL order)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    A = A.tocsr()
    rowptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    col = np.ascontiguousarray(A.indices, dtype=np.int32)
    h = _p()
    _check(_lib.h2_cluster_tree_dd(_ptr(pts), pts.shape[0], pts.shape[1], int(leaf_size), _ptr(rowptr), _ptr(col),
                                   C.byref(h)))
    return Tree(h.value, pts.shape[0])


def h2_block_tree(rows: Tree, cols: Tree, eta: float) -> BlockTree:
    h = _p()
    _check(_lib.h2_block_tree(rows.h, cols.h, float(eta), C.byref(h)))
    return BlockTree(h.value, rows, cols)


def h2_from_sparse(bt: BlockTree, A, lower: bool = False, rank_cap: int = 32, update_cap: int = 32,
                   stream=None) -> Mat:
    """A: scipy.sparse matrix (ORIGINAL order)."""
    A = A.tocsr()
    rowptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    col = np.ascontiguousarray(A.indices, dtype=np.int32)
    val = np.ascontiguousarray(A.data, dtype=np.float64)
    h = _p()
    _check(_lib.h2_from_sparse(bt.h, A.shape[0], _ptr(rowptr), _ptr(col), _ptr(val), 1 if lower else 0,
                               int(rank_cap), int(update_cap), _stream(stream), C.byref(h)))
    return Mat(h.value, bt, lower, rank_cap, update_cap)


def _colmajor(X):
    """(m, k) torch CUDA tensor -> (pointer-owning tensor, ld) in column-major layout."""
    if X.dim() == 1:
        X = X[:, None]
    m = X.shape[0]
    if X.stride(0) == 1 and (X.shape[1] <= 1 or X.stride(1) >= m):
        return X, max(X.stride(1) if X.shape[1] > 1 else m, 1)
    Xc = X.t().contiguous().t()
    return Xc, m


def h2_lowrank_update(Z: Mat, t0: int, s0: int, X, Y, alpha: float = 1.0, trunc: Trunc | None = None,
                      stream=None):
    """Z|_{t0 x s0} += alpha X Y^T.  X (|t0| x k), Y (|s0| x k): torch float64 CUDA tensors, rows in
    tree order within t0/s0."""
    Xc, ldx = _colmajor(X)
    Yc, ldy = _colmajor(Y)
    k = Xc.shape[1]
    if Yc.shape[1] != k:
        raise H2Error(2, "X and Y have different numbers of columns")
    tr = _ctrunc(trunc)
    _check(_lib.h2_lowrank_update(Z.h, int(t0), int(s0), int(k), float(alpha), _ptr(Xc), int(ldx), _ptr(Yc),
                                  int(ldy), C.byref(tr), _stream(stream)))
    if _batch_keep is not None:  # deferred execution: the recorded pointers must stay valid
        _batch_keep.append((X, Y, Xc, Yc))
    return Xc, Yc  # caller keeps them alive until the stream passes the call


_batch_keep = None  # factor copies made by the binding while a batch is open (kept until h2_batch_end)


def h2_batch_begin(stream=None):
    """Record the following h2_lowrank_update calls (same stream) into one device op list.  The
    column-major copies the binding makes of non-column-major factors are kept alive until
    h2_batch_end (their memory can then only be reused by later work on the same stream)."""
    global _batch_keep
    _check(_lib.h2_batch_begin(_stream(stream)))
    _batch_keep = []


def h2_batch_end():
    global _batch_keep
    try:
        _check(_lib.h2_batch_end())
    finally:
        _batch_keep = None


def h2_matvec(Z: Mat, x, y=None, alpha: float = 1.0, beta: float = 0.0, transpose: bool = False, stream=None):
    """y <- alpha op(Z) x + beta y, x/y torch float64 CUDA vectors in ORIGINAL order."""
    if y is None:
        import torch
        y = torch.zeros_like(x)
    _check(_lib.h2_matvec(Z.h, 1 if transpose else 0, float(alpha), _ptr(x), float(beta), _ptr(y), _stream(stream)))
    return y


def h2_addmul(Z: Mat, alpha, X: Mat, Y: Mat, trunc=None, stream=None):
    tr = _ctrunc(trunc)
    _check(_lib.h2_addmul(Z.h, float(alpha), X.h, Y.h, C.byref(tr), _stream(stream)))


def h2_inverse(A: Mat, trunc=None, stream=None):
    """A <- A^{-1} in place (Remark 1: block Gauss elimination, six products per level)."""
    tr = _ctrunc(trunc)
    _check(_lib.h2_inverse(A.h, C.byref(tr), _stream(stream)))


def h2_lr_factor(A: Mat, cholesky: bool = True, trunc=None, stream=None):
    tr = _ctrunc(trunc)
    _check(_lib.h2_lr_factor(A.h, 1 if cholesky else 0, C.byref(tr), _stream(stream)))


def h2_solve(F: Mat, x, nrhs: int = 1, ldx: int | None = None, stream=None):
    """x <- F^{-1} x in place (x: torch float64 CUDA, n x nrhs column-major, ORIGINAL order)."""
    _check(_lib.h2_solve(F.h, _ptr(x), int(nrhs), int(ldx or F.n), _stream(stream)))
    return x


def h2_stats(Z: Mat):
    out = np.zeros(4, dtype=np.int64)
    _check(_lib.h2_stats(Z.h, _ptr(out)))
    return dict(updates=int(out[0]), dense_adds=int(out[1]), temporaries=int(out[2]), updates_nonzero=int(out[3]))


def h2_ranks(Z: Mat):
    nr, nc = Z.bt.rows.nclusters, Z.bt.cols.nclusters
    kr = np.empty(nr, dtype=np.int32)
    kc = np.empty(nc, dtype=np.int32)
    _check(_lib.h2_ranks(Z.h, _ptr(kr), _ptr(kc)))
    return kr, kc


def h2_storage_report(Z: Mat):
    out = np.zeros(4, dtype=np.int64)
    _check(_lib.h2_storage_report(Z.h, _ptr(out)))
    return out


def h2_check_device_flags(Z: Mat) -> int:
    f = np.zeros(1, dtype=np.int32)
    _check(_lib.h2_check_device_flags(Z.h, _ptr(f)))
    return int(f[0])


def h2_export(Z: Mat):
    """Whole representation on the host: dict V, E, W, F (per cluster), S, N (per stored block) in
    the tight layouts of include/h2.h, plus ranks."""
    sizes = np.zeros(6, dtype=np.int64)
    _check(_lib.h2_export(Z.h, None, None, None, None, None, None, _ptr(sizes)))
    bufs = [np.empty(int(s), dtype=np.float64) for s in sizes]
    _check(_lib.h2_export(Z.h, *[_ptr(b) for b in bufs], _ptr(sizes)))
    kr, kc = h2_ranks(Z)
    return dict(zip(["V", "E", "W", "F", "S", "N"], bufs), k=kr, l=kc)


def h2_import(bt: BlockTree, rep: dict, lower: bool = False, rank_cap: int = 32, update_cap: int = 32,
              stream=None) -> Mat:
    """The inverse of h2_export: rep = dict(k, l, V, E, W, F, S, N) in h2_export's layouts."""
    kr = np.ascontiguousarray(rep["k"], dtype=np.int32)
    kc = np.ascontiguousarray(rep["l"], dtype=np.int32)
    arrs = [np.ascontiguousarray(rep[x], dtype=np.float64) for x in ("V", "E", "W", "F", "S", "N")]
    h = _p()
    _check(_lib.h2_import(bt.h, _ptr(kr), _ptr(kc), *[_ptr(a) if a.size else None for a in arrs],
                          1 if lower else 0, int(rank_cap), int(update_cap), _stream(stream), C.byref(h)))
    return Mat(h.value, bt, lower, rank_cap, update_cap)


def h2_profile_enable(on: bool = True):
    _check(_lib.h2_profile_enable(1 if on else 0))


def h2_profile_read():
    """{kernel name: dict(launches, ms, flops, bytes)} for every kernel kind launched."""
    cnt = _i32()
    _check(_lib.h2_profile_read(None, None, None, None, None, C.byref(cnt)))
    n = cnt.value
    names = C.create_string_buffer(32 * n)
    la = np.zeros(n, dtype=np.int64)
    ms, fl, by = (np.zeros(n) for _ in range(3))
    _check(_lib.h2_profile_read(names, _ptr(la), _ptr(ms), _ptr(fl), _ptr(by), C.byref(cnt)))
    out = {}
    for i in range(n):
        name = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
        if la[i]:
            out[name] = dict(launches=int(la[i]), ms=float(ms[i]), flops=float(fl[i]), bytes=float(by[i]))
    return out


def h2_profile_debug():
    out = np.zeros(16)
    _check(_lib.h2_profile_debug(_ptr(out)))
    return out


OP_NAMES = ["upd_ext_leaf", "upd_ext_level", "upd_w_path", "upd_w_level", "upd_svd_leaf", "upd_svd_level",
            "upd_couple", "upd_install", "upd_rcache", "expand", "gemm", "gemm_part", "gemm_sum", "hm_fwd_leaf",
            "hm_fwd_level", "hm_couple", "hm_bwd_level", "hm_leaf", "potrf", "getrf", "trsm", "tsqr", "temp",
            "copy_cols", "set_int", "add_int", "rank_if", "stack", "choose", "identity", "transpose", "gather",
            "scatter", "zero", "dd", "nztile", "tinv", "c2core", "skipz"]


def h2_profile_ops():
    """Per executor op code: {name: (count, ms)} (profiling must be enabled)."""
    ns = np.zeros(64)
    cnt = np.zeros(64)
    _check(_lib.h2_profile_ops(_ptr(ns), _ptr(cnt), 64, None))
    return {OP_NAMES[i] if i < len(OP_NAMES) else str(i): (int(cnt[i]), round(ns[i] / 1e6, 1))
            for i in range(64) if cnt[i] > 0}


def h2_pcg(A: Mat, F: Mat, b, x=None, tol: float = 1e-8, maxit: int = 500, stream=None):
    """Preconditioned CG on the device: returns (x, iterations, relative residual)."""
    if x is None:
        import torch
        x = torch.empty_like(b)
    it = _i32()
    rr = _f64()
    _check(_lib.h2_pcg(A.h, F.h, _ptr(b), _ptr(x), float(tol), int(maxit), C.byref(it), C.byref(rr), _stream(stream)))
    return x, it.value, rr.value


def h2_launch_count() -> int:
    v = _i64()
    _check(_lib.h2_launch_count(C.byref(v)))
    return v.value

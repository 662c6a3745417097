"""CPU oracle for the SpMxV hot path (arXiv 1203.2739) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  It shares
no code with the CUDA path in ``paper_1203_2739_b200/`` and never imports it.

Every routine is a thin ctypes shim over ``oracle.c`` (plain C, fp64,
``-O3 -ffp-contract=off``); each C function cites the PAPER.md passage it
follows (P:Lnn = /root/reference/PAPER.md line nn).  Parity status of each
function is listed in DESIGN.md "Oracle pins"; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

TOL = 1e-12   # north_star: |y - y_ref| <= 1e-12 * sum_j |a_ij x_j| per entry


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O3 -ffp-contract=off, OpenMP for row-parallel timing)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        vp, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.oracle_validate_csr.argtypes = [i64, i64, i64, vp, vp]
        L.oracle_validate_perm.argtypes = [i64, vp]
        L.oracle_permute.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_permute.restype = None
        L.oracle_permute_x.argtypes = [i64, vp, vp, vp]
        L.oracle_permute_x.restype = None
        L.oracle_unpermute_y.argtypes = [i64, vp, vp, vp]
        L.oracle_unpermute_y.restype = None
        L.oracle_spmv.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32]
        L.oracle_spmv.restype = None
        L.oracle_spmv_rows.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_spmv_rows.restype = None
        L.oracle_split.argtypes = [i64, vp, vp, vp, vp, i32, vp, vp]
        L.oracle_maxabs.argtypes = [i64, vp]
        L.oracle_maxabs.restype = f64
        L.oracle_scale.argtypes = [i64, vp, f64, vp]
        L.oracle_scale.restype = None
        L.oracle_check.argtypes = [i64, vp, vp, vp, f64, ctypes.POINTER(f64), ctypes.POINTER(i64)]
        L.oracle_check.restype = i64
        L.oracle_sb_lambda.argtypes = [i64, i64, vp, vp, vp, vp]
        L.oracle_sb_lambda.restype = i64
        L.oracle_split_lambda.argtypes = [i64, i64, vp, vp, vp, i32, ctypes.POINTER(i64),
                                          ctypes.POINTER(i64)]
        L.oracle_split_lambda.restype = None
        L.oracle_sbfs.argtypes = [i64, i64, vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.oracle_sbfs.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def validate_csr(m, n, row_ptr, col) -> int:
    """0 ok, 1 bad row_ptr, 2 column out of range, 3 duplicate (i, j)."""
    row_ptr = _c(row_ptr, np.int64)
    col = _c(col, np.int32)
    return int(_load().oracle_validate_csr(m, n, int(row_ptr[-1]) if m >= 0 else 0, _p(row_ptr), _p(col)))


def validate_perm(perm) -> int:
    perm = _c(perm, np.int32)
    return int(_load().oracle_validate_perm(len(perm), _p(perm)))


def permute(m, n, row_ptr, col, val, row_perm, col_perm, parts=None):
    """A^ = P_r A P_c in old->new array form.  Returns
    (row_ptr, col, val, parts) of the canonical permuted CSR."""
    row_ptr, col, val = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    rp = _c(np.arange(m) if row_perm is None else row_perm, np.int32)
    cp = _c(np.arange(n) if col_perm is None else col_perm, np.int32)
    nnz = int(row_ptr[-1])
    o_rp = np.empty(m + 1, np.int64)
    o_c = np.empty(nnz, np.int32)
    o_v = np.empty(nnz, np.float64)
    o_p = None
    if parts is not None:
        parts = _c(parts, np.int32)
        o_p = np.empty(nnz, np.int32)
    _load().oracle_permute(m, n, _p(row_ptr), _p(col), _p(val), _p(rp), _p(cp), _p(parts),
                           _p(o_rp), _p(o_c), _p(o_v), _p(o_p))
    return o_rp, o_c, o_v, o_p


def permute_x(col_perm, x):
    """x^[col_perm[j]] = x[j]."""
    x = _c(x, np.float64)
    if col_perm is None:
        return x.copy()
    cp = _c(col_perm, np.int32)
    out = np.empty_like(x)
    _load().oracle_permute_x(len(x), _p(cp), _p(x), _p(out))
    return out


def unpermute_y(row_perm, yhat):
    """y[i] = y^[row_perm[i]]."""
    yhat = _c(yhat, np.float64)
    if row_perm is None:
        return yhat.copy()
    rp = _c(row_perm, np.int32)
    out = np.empty_like(yhat)
    _load().oracle_unpermute_y(len(yhat), _p(rp), _p(yhat), _p(out))
    return out


def spmv(row_ptr, col, val, x, nthreads: int = 1):
    """y = A x, serial per-row temporary.  Returns (y, S)."""
    row_ptr, col, val, x = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64), _c(x, np.float64)
    m = len(row_ptr) - 1
    y = np.empty(m, np.float64)
    S = np.empty(m, np.float64)
    _load().oracle_spmv(m, _p(row_ptr), _p(col), _p(val), _p(x), _p(y), _p(S), nthreads)
    return y, S


def spmv_rows(rows, row_ptr, col, val, x):
    """y_i and S_i for the listed rows only (sampled parity at full size)."""
    rows = _c(rows, np.int64)
    row_ptr, col, val, x = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64), _c(x, np.float64)
    y = np.empty(len(rows), np.float64)
    S = np.empty(len(rows), np.float64)
    _load().oracle_spmv_rows(len(rows), _p(rows), _p(row_ptr), _p(col), _p(val), _p(x), _p(y), _p(S))
    return y, S


def split(row_ptr, col, val, parts, K, x):
    """Literal multiple-SpMxV y <- y + A^k x, k ascending."""
    row_ptr, col, val, x = _c(row_ptr, np.int64), _c(col, np.int32), _c(val, np.float64), _c(x, np.float64)
    parts = _c(parts, np.int32)
    m = len(row_ptr) - 1
    y = np.empty(m, np.float64)
    rc = _load().oracle_split(m, _p(row_ptr), _p(col), _p(val), _p(parts), K, _p(x), _p(y))
    if rc:
        raise ValueError("oracle.split: part id outside [0, K)")
    return y


def maxabs(y) -> float:
    y = _c(y, np.float64)
    return float(_load().oracle_maxabs(len(y), _p(y)))


def scale(y, mt):
    """x_{t+1} = y_t / m_t (original space, square A)."""
    y = _c(y, np.float64)
    out = np.empty_like(y)
    _load().oracle_scale(len(y), _p(y), float(mt), _p(out))
    return out


def check(y, yref, S, tol: float = TOL):
    """Per-entry comparator.  Returns (n_bad, worst |d|/S, first_bad)."""
    y, yref, S = _c(y, np.float64), _c(yref, np.float64), _c(S, np.float64)
    w = ctypes.c_double(0.0)
    fb = ctypes.c_int64(-1)
    bad = _load().oracle_check(len(y), _p(y), _p(yref), _p(S), tol, ctypes.byref(w), ctypes.byref(fb))
    return int(bad), float(w.value), int(fb.value)


def sb_lambda(m, n, row_ptr, col, row_block):
    """Eq.(3) lambda(c_j) per column and its sum (Theorem 1's bound)."""
    row_ptr, col, rb = _c(row_ptr, np.int64), _c(col, np.int32), _c(row_block, np.int32)
    lam = np.empty(n, np.int32)
    s = _load().oracle_sb_lambda(m, n, _p(row_ptr), _p(col), _p(rb), _p(lam))
    return int(s), lam


def split_lambda(m, n, row_ptr, col, parts, K):
    """Theorem 3: (sum_i lambda(r_i), sum_j lambda(c_j))."""
    row_ptr, col, parts = _c(row_ptr, np.int64), _c(col, np.int32), _c(parts, np.int32)
    a, b = ctypes.c_int64(0), ctypes.c_int64(0)
    _load().oracle_split_lambda(m, n, _p(row_ptr), _p(col), _p(parts), K, ctypes.byref(a), ctypes.byref(b))
    return int(a.value), int(b.value)


def sbfs(m, n, row_ptr, col, K):
    """sBFS ordering + SB extraction (reading R5).  Returns dict with
    row_perm, col_perm (old -> new), row_block_ptr, col_block_ptr (K+2 each)
    and the plain BFS numbers bfs_row, bfs_col."""
    row_ptr, col = _c(row_ptr, np.int64), _c(col, np.int32)
    out = dict(row_perm=np.empty(m, np.int32), col_perm=np.empty(n, np.int32),
               row_block_ptr=np.empty(K + 2, np.int64), col_block_ptr=np.empty(K + 2, np.int64),
               bfs_row=np.empty(m, np.int32), bfs_col=np.empty(n, np.int32))
    rc = _load().oracle_sbfs(m, n, _p(row_ptr), _p(col), K, _p(out["row_perm"]), _p(out["col_perm"]),
                             _p(out["row_block_ptr"]), _p(out["col_block_ptr"]), _p(out["bfs_row"]),
                             _p(out["bfs_col"]))
    if rc:
        raise ValueError("oracle.sbfs: bad arguments")
    return out

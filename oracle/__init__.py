"""CPU FP64 oracle for the VIF factor + Gaussian NLL (arXiv 2507.05064).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package; the product
package ``paper_2507_05064_b200`` never does, and this package never imports it.

The arithmetic lives in ``oracle.c`` (plain C loops, OpenMP over rows, no BLAS,
no -ffast-math); this module only compiles it with gcc and marshals numpy
arrays through ctypes.  Each C function cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

FAMILIES = {"matern12": 0, "matern32": 1, "matern52": 2, "gaussian": 3}


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-D_GNU_SOURCE",
               "-fno-fast-math", "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


class _Theta(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("d", ctypes.c_int32), ("sigma2", ctypes.c_double),
                ("lengthscale", ctypes.POINTER(ctypes.c_double)), ("nugget", ctypes.c_double),
                ("jitter", ctypes.c_double)]


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int
        _lib.oracle_cov_matrix.argtypes = [P, P, i64, P, i64, P]
        _lib.oracle_check_neighbors.argtypes = [i64, i32, P]
        _lib.oracle_check_neighbors.restype = i64
        _lib.oracle_factor_nll.argtypes = [i64, i32, i32, P, P, P, P, P, P, P, P, P, P]
        _lib.oracle_rows.argtypes = [i64, i32, i32, P, P, P, P, i64, P, P, P, P, P]
        _lib.oracle_partial.argtypes = [i64, i32, i32, P, P, P, P, P, i64, P, P, P, P, P]
        _lib.oracle_finish.argtypes = [i64, i32, P, P, P, P]
        _lib.oracle_num_threads.restype = ctypes.c_int
        _lib.oracle_grad.argtypes = [i64, i32, i32, P, P, P, P, P, P, P, P]
        _lib.oracle_dcov_matrix.argtypes = [P, P, i64, P, i64, P]
        _lib.oracle_dc_neighbors.argtypes = [i64, i32, i32, P, P, P, P, P]
        _lib.oracle_dc_scores.argtypes = [i64, i32, P, P, P, i64, P, P, P]
        _lib.oracle_predict.argtypes = [i64, i32, i32, P, P, P, P, P, i64, P, P, P, P, P, P, P]
    return _lib


@dataclass
class Theta:
    """Covariance parameters theta: family, sigma_1^2, ARD length-scales, nugget sigma^2, jitter."""
    family: str
    sigma2: float
    lengthscale: Sequence[float]
    nugget: float
    jitter: float

    def _c(self):
        ls = np.ascontiguousarray(np.asarray(self.lengthscale, dtype=np.float64))
        th = _Theta(FAMILIES[self.family], len(ls), float(self.sigma2),
                    ls.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(self.nugget), float(self.jitter))
        return th, ls  # keep ls alive


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def cov_matrix(theta: Theta, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    lib = _load()
    A, B = _f64(A), _f64(B)
    th, keep = theta._c()
    out = np.empty((A.shape[0], B.shape[0]))
    lib.oracle_cov_matrix(ctypes.byref(th), _p(A), A.shape[0], _p(B), B.shape[0], _p(out))
    return out


def check_neighbors(nbr: np.ndarray) -> int:
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    n, mv = nbr.shape
    return int(_load().oracle_check_neighbors(n, mv, _p(nbr)))


class OracleError(RuntimeError):
    def __init__(self, status, bad_row):
        super().__init__(f"oracle status {status}, bad_row {bad_row}")
        self.status, self.bad_row = status, bad_row


@dataclass
class Result:
    nll: float
    logdet_D: float
    logdet_M: float
    quad: float
    U: Optional[np.ndarray]
    B: Optional[np.ndarray]
    D: Optional[np.ndarray]


def factor_nll(X, Z, nbr, y, theta: Theta, want_U=False, want_BD=True) -> Result:
    """Oracle T1: whole factor + NLL."""
    lib = _load()
    X, Z, y = _f64(X), _f64(Z).reshape(-1, X.shape[1]), _f64(y)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    n, mv = nbr.shape
    m = Z.shape[0]
    U = np.empty((n, m)) if want_U and m > 0 else None
    B = np.empty((n, mv)) if want_BD else None
    D = np.empty(n) if want_BD else None
    terms = np.zeros(4)
    bad = ctypes.c_int64(-1)
    th, keep = theta._c()
    st = lib.oracle_factor_nll(n, m, mv, _p(X), _p(Z), _p(nbr), _p(y), ctypes.byref(th), _p(U), _p(B), _p(D),
                               _p(terms), ctypes.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return Result(terms[0], terms[1], terms[2], terms[3], U, B, D)


def rows(X, Z, nbr, theta: Theta, rows_idx, want_U=False):
    """Oracle B/D (and u) for sampled rows, each recomputed from scratch."""
    lib = _load()
    X, Z = _f64(X), _f64(Z).reshape(-1, X.shape[1])
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    rows_idx = np.ascontiguousarray(rows_idx, dtype=np.int64)
    n, mv = nbr.shape
    m = Z.shape[0]
    k = rows_idx.shape[0]
    U = np.empty((k, m)) if want_U else None
    B = np.empty((k, mv))
    D = np.empty(k)
    bad = ctypes.c_int64(-1)
    th, keep = theta._c()
    st = lib.oracle_rows(n, m, mv, _p(X), _p(Z), _p(nbr), ctypes.byref(th), k, _p(rows_idx), _p(U), _p(B), _p(D),
                         ctypes.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return U, B, D


def partial(X, Z, nbr, y, theta: Theta, rows_idx):
    """Partial sums (G lower, v, [sum r^2/D, sum log D]) over a subset of rows."""
    lib = _load()
    X, Z, y = _f64(X), _f64(Z).reshape(-1, X.shape[1]), _f64(y)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    rows_idx = np.ascontiguousarray(rows_idx, dtype=np.int64)
    n, mv = nbr.shape
    m = Z.shape[0]
    G = np.zeros((m, m))
    v = np.zeros(m)
    sums = np.zeros(2)
    bad = ctypes.c_int64(-1)
    th, keep = theta._c()
    st = lib.oracle_partial(n, m, mv, _p(X), _p(Z), _p(nbr), _p(y), ctypes.byref(th), rows_idx.shape[0],
                            _p(rows_idx), _p(G), _p(v), _p(sums), ctypes.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return G, v, sums


def finish(n, G, v, sums):
    lib = _load()
    G, v, sums = _f64(G), _f64(v), _f64(sums)
    m = v.shape[0]
    terms = np.zeros(4)
    st = lib.oracle_finish(n, m, _p(G), _p(v), _p(sums), _p(terms))
    if st != 0:
        raise OracleError(st, -1)
    return terms


@dataclass
class GradResult:
    """dNLL/dtheta for theta = (sigma_1^2, lambda_1..lambda_d, sigma^2) and, per parameter, the
    three derivative terms (d sum log D, d logdet M_w, d quad) whose halves sum to it."""
    grad: np.ndarray
    parts: np.ndarray


def grad(X, Z, nbr, y, theta: Theta) -> GradResult:
    """Oracle gradient of the VIF NLL (Appendix A; oracle.c oracle_grad)."""
    lib = _load()
    X, Z, y = _f64(X), _f64(Z).reshape(-1, X.shape[1]), _f64(y)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    n, mv = nbr.shape
    m = Z.shape[0]
    P = X.shape[1] + 2
    g = np.zeros(P)
    parts = np.zeros((P, 3))
    bad = ctypes.c_int64(-1)
    th, keep = theta._c()
    st = lib.oracle_grad(n, m, mv, _p(X), _p(Z), _p(nbr), _p(y), ctypes.byref(th), _p(g), _p(parts),
                         ctypes.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return GradResult(g, parts)


def dcov_matrix(theta: Theta, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """dk(A_i, B_j)/dtheta_p for p = sigma_1^2, lambda_1..lambda_d: shape (d+1, na, nb)."""
    lib = _load()
    A, B = _f64(A), _f64(B)
    th, keep = theta._c()
    out = np.empty((A.shape[1] + 1, A.shape[0], B.shape[0]))
    lib.oracle_dcov_matrix(ctypes.byref(th), _p(A), A.shape[0], _p(B), B.shape[0], _p(out))
    return out


def predict(X, Z, nbr, y, theta: Theta, Xp, nbrp):
    """Oracle predictive means and variances (Prop. 1; App. C.1; reading p1):
    returns (mu, var, D_p, B_p = -A_p)."""
    lib = _load()
    X, Z, y = _f64(X), _f64(Z).reshape(-1, X.shape[1]), _f64(y)
    Xp = _f64(Xp).reshape(-1, X.shape[1])
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    nbrp = np.ascontiguousarray(nbrp, dtype=np.int32)
    n, mv = nbr.shape
    npred = Xp.shape[0]
    m = Z.shape[0]
    mu, var, Dp, Bp = np.zeros(npred), np.zeros(npred), np.zeros(npred), np.zeros((npred, mv))
    bad = ctypes.c_int64(-1)
    th, keep = theta._c()
    st = lib.oracle_predict(n, m, mv, _p(X), _p(Z), _p(nbr), _p(y), ctypes.byref(th), npred, _p(Xp), _p(nbrp),
                            _p(mu), _p(var), _p(Dp), _p(Bp), ctypes.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return mu, var, Dp, Bp


def dc_neighbors(X, Z, theta: Theta, mv: int):
    """Oracle correlation-distance neighbour sets (readings c5-c7): (nbr n x mv, scores)."""
    lib = _load()
    X, Z = _f64(X), _f64(Z).reshape(-1, X.shape[1])
    n, m = X.shape[0], Z.shape[0]
    nbr = np.empty((n, mv), dtype=np.int32)
    sc = np.empty((n, mv))
    th, keep = theta._c()
    st = lib.oracle_dc_neighbors(n, m, mv, _p(X), _p(Z), ctypes.byref(th), _p(nbr), _p(sc))
    if st != 0:
        raise OracleError(st, -1)
    return nbr, sc


def dc_scores(X, Z, theta: Theta, qi, cj):
    """Scores (|corr|, 0 for degenerate candidates, -dist^2 for degenerate queries) of (qi, cj) pairs."""
    lib = _load()
    X, Z = _f64(X), _f64(Z).reshape(-1, X.shape[1])
    qi = np.ascontiguousarray(qi, dtype=np.int64)
    cj = np.ascontiguousarray(cj, dtype=np.int64)
    out = np.empty(qi.shape[0])
    th, keep = theta._c()
    st = lib.oracle_dc_scores(X.shape[0], Z.shape[0], _p(X), _p(Z), ctypes.byref(th), qi.shape[0], _p(qi), _p(cj),
                              _p(out))
    if st != 0:
        raise OracleError(st, -1)
    return out


def num_threads() -> int:
    return int(_load().oracle_num_threads())

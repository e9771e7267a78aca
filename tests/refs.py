"""Independent dense references for the oracle pins (numpy / scipy / scikit-learn only).

Nothing here imports oracle/ or the CUDA package; kernels come from
scikit-learn's Matern / RBF implementations, linear algebra from LAPACK.
"""
import numpy as np
from sklearn.gaussian_process.kernels import Matern, RBF

NU = {"matern12": 0.5, "matern32": 1.5, "matern52": 2.5}


def sk_cov(family, sigma2, lengthscale, A, B=None):
    ls = np.asarray(lengthscale, dtype=np.float64)
    if family == "gaussian":
        k = RBF(length_scale=ls / np.sqrt(2.0))      # exp(-|d/ls|^2)
    else:
        k = Matern(length_scale=ls, nu=NU[family])
    return sigma2 * k(np.atleast_2d(A), None if B is None else np.atleast_2d(B))


def dense_nll(S, y):
    """Gaussian NLL with covariance S by Cholesky."""
    L = np.linalg.cholesky(S)
    a = np.linalg.solve(L, y)
    n = len(y)
    return 0.5 * n * np.log(2 * np.pi) + np.sum(np.log(np.diag(L))) + 0.5 * a @ a


def nystrom(w, X=None):
    """Q = K_nm K_m^{-1} K_mn (un-whitened, LU solve) with the same jitter as theta."""
    X = w.X if X is None else X
    if w.m == 0:
        return np.zeros((X.shape[0], X.shape[0]))
    Km = sk_cov(w.family, w.sigma2, w.lengthscale, w.Z) + w.jitter * np.eye(w.m)
    Knm = sk_cov(w.family, w.sigma2, w.lengthscale, X, w.Z)
    return Knm @ np.linalg.solve(Km, Knm.T)


def B_matrix(nbr, Bvals):
    n, mv = nbr.shape
    B = np.eye(n)
    for i in range(n):
        for k in range(mv):
            j = nbr[i, k]
            if j >= 0:
                B[i, j] = Bvals[i, k]
    return B


def sk_cov_grad(family, sigma2, lengthscale, A):
    """K(A, A) and dK/dtheta for theta = (sigma_1^2, lambda_1..lambda_d) from scikit-learn's
    analytic kernel gradients (eval_gradient=True returns dK/dlog(length_scale_j))."""
    ls = np.asarray(lengthscale, dtype=np.float64)
    A = np.atleast_2d(A)
    if family == "gaussian":
        k = RBF(length_scale=ls / np.sqrt(2.0))
    else:
        k = Matern(length_scale=ls, nu=NU[family])
    K, G = k(A, eval_gradient=True)        # G[..., j] = dK / dlog ls_j (ls_j proportional to lambda_j)
    if G.shape[2] == 1 and len(ls) > 1:     # isotropic fallback never used (ls is an array)
        raise ValueError("expected per-dimension gradients")
    dK = [K] + [sigma2 * G[:, :, j] / ls[j] for j in range(len(ls))]
    return sigma2 * K, np.stack(dK)


def dense_grad(S, dS, y):
    """Gaussian NLL gradient with covariance S: 1/2 tr(S^{-1} dS_p) - 1/2 a^T dS_p a, a = S^{-1} y."""
    Si = np.linalg.inv(S)
    a = Si @ y
    return np.array([0.5 * np.trace(Si @ d) - 0.5 * a @ d @ a for d in dS])

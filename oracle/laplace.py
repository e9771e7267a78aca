"""CPU FP64 oracle for the VIF-Laplace iterative path (Sect. 3-4).

TEST INFRASTRUCTURE ONLY, like the rest of ``oracle/``: tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs may call it; the product package never does.

Bernoulli likelihood with the logit link, latent VIF prior N(0, Sigma_dagger) whose residual
Vecchia factor B, D is built WITHOUT the error variance (the factor of ``oracle.factor_nll``
with nugget 0), the mode by Newton's method (Eq. one_it_newton_mode) with the linear solves
in the form (pcls2), solved by preconditioned CG with the FITC preconditioner
(App. FITC) on the VIF's own inducing points (k = m, reading l2), and the
approximate negative log-marginal likelihood L^VIFLA with its log-determinant from the SLQ
estimate (slq_v2) (App. RT), the tridiagonal matrices taken from the CG
coefficients.  numpy / scipy primitives serve as steps (a sparse triangular solve, a dense
symmetric eigendecomposition); nothing is blocked, fused or reordered beyond the paper's formulas.

Readings: l1 Bernoulli-logit only; l2 FITC on the VIF inducing points (k = m);
l3 CG stops when ||r||_2 <= tol ||rhs||_2 (or after max_it); l4 Newton starts at b = 0, warm-starts
CG at x0 = W b, and stops when the relative change of log p(y|b) - b^T a / 2 drops below tol;
l5 the quadratic term b^T Sigma_dagger^{-1} b of L^VIFLA is evaluated exactly by Woodbury;
l6 the SLQ weight is n / ell as printed in slq_v2 (not ||P^{-1/2} z_i||^2); l7 probe vectors
z_i = D_V^{1/2} eps2_i + U eps1_i (App. FITC) with caller-supplied standard normals.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from . import Theta, factor_nll


# ------------------------------------------------------------------------------------------ likelihood
def sigmoid(b):
    """Logistic function pi = 1 / (1 + exp(-b)) (logit link)."""
    return 1.0 / (1.0 + np.exp(-b))


def loglik(y, b):
    """log p(y | b) = sum_i y_i b_i - log(1 + exp(b_i)) for y_i in {0, 1} (Bernoulli, logit link)."""
    return float(np.sum(y * b - np.logaddexp(0.0, b)))


def grad_loglik(y, b):
    """d log p(y|b) / db = y - pi."""
    return y - sigmoid(b)


def hess_w(b):
    """W_ii = -d^2 log p / db_i^2 = pi_i (1 - pi_i) (Eq. W_diag)."""
    p = sigmoid(b)
    return p * (1.0 - p)


# ------------------------------------------------------------------------------------------ latent prior
@dataclass
class LatentVIF:
    """Sigma_dagger = B^{-1} D B^{-T} + U U^T, U = Sigma_mn^T L_m^{-T} (whitened)."""
    B: sp.csr_matrix   # n x n unit lower triangular, B[i, N(i)] = -A_i
    Bt: sp.csr_matrix  # B^T (upper triangular)
    D: np.ndarray      # n
    U: np.ndarray      # n x m
    sigma2: float
    logdet_M: float    # log det(I + U^T B^T D^{-1} B U) of the factor (nugget 0)
    logdet_D: float

    @property
    def n(self):
        return self.D.shape[0]

    def binv(self, v):
        """B^{-1} v (forward substitution in the Vecchia order)."""
        return spsolve_triangular(self.B, v, lower=True, unit_diagonal=True)

    def btinv(self, v):
        """B^{-T} v (backward substitution)."""
        return spsolve_triangular(self.Bt, v, lower=False, unit_diagonal=True)

    def sigma_dagger(self, v):
        """Sigma_dagger v = B^{-1} D B^{-T} v + U (U^T v)."""
        v = np.asarray(v, dtype=np.float64)
        return self.binv(self.D[:, None] * self.btinv(v) if v.ndim == 2 else self.D * self.btinv(v)) + \
            self.U @ (self.U.T @ v)

    def sigma_dagger_inv(self, v):
        """Sigma_dagger^{-1} v = B^T D^{-1} B v - B^T D^{-1} B U M^{-1} U^T B^T D^{-1} B v."""
        Bv = self.B @ v
        DBv = Bv / self.D
        if self.U.shape[1] == 0:
            return self.Bt @ DBv
        BU = self.B @ self.U
        M = np.eye(self.U.shape[1]) + BU.T @ (BU / self.D[:, None])
        t = np.linalg.solve(M, BU.T @ DBv)
        return self.Bt @ (DBv - (BU @ t) / self.D)


def latent_factor(X, Z, nbr, theta: Theta) -> LatentVIF:
    """B, D, U of the latent process: the VIF factor with the error variance removed."""
    th0 = Theta(theta.family, theta.sigma2, theta.lengthscale, 0.0, theta.jitter)
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, mv = nbr.shape
    r = factor_nll(X, Z, nbr, np.zeros(n), th0, want_U=True, want_BD=True)
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [np.ones(n)]
    for p in range(mv):
        ok = nbr[:, p] >= 0
        rows.append(np.nonzero(ok)[0])
        cols.append(nbr[ok, p].astype(np.int64))
        vals.append(r.B[ok, p])
    B = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    U = r.U if r.U is not None else np.zeros((n, 0))
    return LatentVIF(B=B, Bt=B.T.tocsr(), D=r.D.copy(), U=U, sigma2=float(theta.sigma2), logdet_M=r.logdet_M,
                     logdet_D=r.logdet_D)


# ------------------------------------------------------------------------------------------ FITC
@dataclass
class FITC:
    """P = D_V + Sigma_kn^T Sigma_k^{-1} Sigma_kn, D_V = diag(Sigma - Sigma_kn^T Sigma_k^{-1} Sigma_kn) + W^{-1}
    (App. FITC); with k = m and the whitened U: Sigma_kn^T Sigma_k^{-1} Sigma_kn = U U^T."""
    DV: np.ndarray
    U: np.ndarray
    MV: np.ndarray     # I + U^T D_V^{-1} U  (= L_k^{-1} M_V L_k^{-T}, M_V of P:1069)

    def solve(self, w):
        """P^{-1} w = D_V^{-1} w - D_V^{-1} U M_V^{-1} U^T D_V^{-1} w."""
        w = np.asarray(w, dtype=np.float64)
        dv = self.DV[:, None] if w.ndim == 2 else self.DV
        t = w / dv
        if self.U.shape[1] == 0:
            return t
        return t - (self.U @ np.linalg.solve(self.MV, self.U.T @ t)) / dv

    def logdet(self):
        """log det P = log det D_V - log det Sigma_k + log det M_V = log det D_V + log det(I + U^T D_V^{-1} U)
        (Sylvester)."""
        s = np.sum(np.log(self.DV))
        if self.U.shape[1]:
            s += np.linalg.slogdet(self.MV)[1]
        return float(s)

    def sample(self, eps1, eps2):
        """z = D_V^{1/2} eps2 + Sigma_kn^T Sigma_k^{-1/2} eps1 = D_V^{1/2} eps2 + U eps1."""
        dv = self.DV[:, None] if eps2.ndim == 2 else self.DV
        return np.sqrt(dv) * eps2 + self.U @ eps1


def fitc(lat: LatentVIF, W) -> FITC:
    DV = lat.sigma2 - np.sum(lat.U * lat.U, axis=1) + 1.0 / W
    MV = np.eye(lat.U.shape[1]) + lat.U.T @ (lat.U / DV[:, None])
    return FITC(DV=DV, U=lat.U, MV=MV)


# ------------------------------------------------------------------------------------------ CG / Lanczos
@dataclass
class CGResult:
    x: np.ndarray
    alpha: List[float]
    beta: List[float]
    iters: int
    relres: float


def pcg(apply_A, b, solve_P, tol, max_it, x0=None) -> CGResult:
    """Preconditioned conjugate gradients (Saad 2003, Alg. 9.1), recording alpha_j and beta_j."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - apply_A(x) if x0 is not None else b.copy()
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return CGResult(x, [], [], 0, 0.0)
    z = solve_P(r)
    p = z.copy()
    rz = float(r @ z)
    alpha, beta = [], []
    it = 0
    relres = np.linalg.norm(r) / nb
    while it < max_it and relres > tol:
        q = apply_A(p)
        a = rz / float(p @ q)
        x = x + a * p
        r = r - a * q
        alpha.append(a)
        it += 1
        relres = np.linalg.norm(r) / nb
        if relres <= tol or it == max_it:
            break
        z = solve_P(r)
        rz_new = float(r @ z)
        bt = rz_new / rz
        beta.append(bt)
        p = z + bt * p
        rz = rz_new
    return CGResult(x, alpha, beta, it, float(relres))


def lanczos_tridiag(alpha, beta):
    """Tridiagonal T_k of the Lanczos process from the CG coefficients (Saad 2003, Sect. 6.7.3):
    T_jj = 1/alpha_j + beta_{j-1}/alpha_{j-1},  T_{j,j+1} = sqrt(beta_j)/alpha_j."""
    k = len(alpha)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / alpha[j] + (beta[j - 1] / alpha[j - 1] if j > 0 else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(beta[j]) / alpha[j]
    return T


def e1_log_e1(T):
    """e_1^T log(T) e_1 = sum_k Q_{1k}^2 log(lambda_k) (T = Q diag(lambda) Q^T)."""
    lam, Q = np.linalg.eigh(T)
    return float(np.sum(Q[0, :] ** 2 * np.log(lam)))


# ------------------------------------------------------------------------------------------ mode and NLL
@dataclass
class LaplaceResult:
    b: np.ndarray            # the mode b~
    a: np.ndarray            # Sigma_dagger^{-1} b~ from the last Newton step (v - x)
    neg_loglik: float        # -log p(y | b~)
    quad: float              # b~^T Sigma_dagger^{-1} b~ (exact, reading l5)
    logdet: Optional[float]  # SLQ estimate of log det(Sigma_dagger W + I) (None without probes)
    nll: Optional[float]     # L^VIFLA = -log p + quad/2 + logdet/2
    newton_iters: int
    cg_iters: List[int]
    slq_iters: List[int] = field(default_factory=list)
    logdet_parts: Optional[dict] = None


def newton_mode(lat: LatentVIF, y, tol=1e-10, max_newton=50, cg_tol=1e-10, max_cg=1000):
    """Mode of p(y|b) N(b; 0, Sigma_dagger) by Newton's method:
    b^{t+1} = (W + Sigma_dagger^{-1})^{-1} (W b^t + d log p / db), solved through (pcls2):
    (W^{-1} + Sigma_dagger) x = Sigma_dagger v with v = W b^t + grad, then b^{t+1} = W^{-1} x and
    Sigma_dagger^{-1} b^{t+1} = v - x (readings l3, l4)."""
    n = lat.n
    b = np.zeros(n)
    psi_old = None
    cg_iters = []
    a = np.zeros(n)
    it = 0
    for it in range(1, max_newton + 1):
        W = hess_w(b)
        v = W * b + grad_loglik(y, b)
        rhs = lat.sigma_dagger(v)
        P = fitc(lat, W)
        res = pcg(lambda p: p / W + lat.sigma_dagger(p), rhs, P.solve, cg_tol, max_cg, x0=W * b)
        cg_iters.append(res.iters)
        b = res.x / W
        a = v - res.x
        psi = loglik(y, b) - 0.5 * float(b @ a)
        if psi_old is not None and abs(psi - psi_old) <= tol * abs(psi_old):
            break
        psi_old = psi
    return b, a, it, cg_iters


def slq_logdet(lat: LatentVIF, W, eps1, eps2, tol=1e-10, max_cg=1000):
    """log det(Sigma_dagger W + I) ~= log det W + (n/ell) sum_i e_1^T log(T_i) e_1 + log det P (slq_v2,
    P:333), T_i from PCG on (W^{-1} + Sigma_dagger) x = z_i, z_i ~ N(0, P) (reading l6, l7)."""
    n = lat.n
    ell = eps2.shape[1]
    P = fitc(lat, W)
    Z = P.sample(eps1, eps2)
    terms, iters = [], []
    for i in range(ell):
        res = pcg(lambda p: p / W + lat.sigma_dagger(p), Z[:, i], P.solve, tol, max_cg)
        terms.append(e1_log_e1(lanczos_tridiag(res.alpha, res.beta)))
        iters.append(res.iters)
    ldW = float(np.sum(np.log(W)))
    ldP = P.logdet()
    est = ldW + n / ell * float(np.sum(terms)) + ldP
    return est, iters, dict(logdet_W=ldW, logdet_P=ldP, slq_terms=terms)


def vifla_nll(X, Z, nbr, y, theta: Theta, eps1=None, eps2=None, newton_tol=1e-10, max_newton=50, cg_tol=1e-10,
              max_cg=1000, slq_tol=1e-10, lat: Optional[LatentVIF] = None) -> LaplaceResult:
    """L^VIFLA(y, theta) = -log p(y|b~) + b~^T Sigma_dagger^{-1} b~ / 2 + log det(Sigma_dagger W + I) / 2
    (P:245), W at the mode."""
    y = np.asarray(y, dtype=np.float64)
    if lat is None:
        lat = latent_factor(X, Z, nbr, theta)
    b, a, nit, cgi = newton_mode(lat, y, newton_tol, max_newton, cg_tol, max_cg)
    nl = -loglik(y, b)
    quad = float(b @ lat.sigma_dagger_inv(b))
    logdet = nll = None
    slq_iters, parts = [], None
    if eps2 is not None:
        logdet, slq_iters, parts = slq_logdet(lat, hess_w(b), eps1, eps2, slq_tol, max_cg)
        nll = nl + 0.5 * quad + 0.5 * logdet
    return LaplaceResult(b=b, a=a, neg_loglik=nl, quad=quad, logdet=logdet, nll=nll, newton_iters=nit,
                         cg_iters=cgi, slq_iters=slq_iters, logdet_parts=parts)


def exact_logdet(lat: LatentVIF, W):
    """log det(Sigma_dagger W + I) from a dense Sigma_dagger (small n; pins only)."""
    n = lat.n
    S = lat.sigma_dagger(np.eye(n))
    return float(np.linalg.slogdet(S * W[None, :] + np.eye(n))[1])

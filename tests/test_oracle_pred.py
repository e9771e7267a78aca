"""Pins of the oracle's predictive means (Proposition 1; reading p1: prediction points
condition on m_v training points, B_p = I).

pp1  all training points as neighbours (training factor exact too): mu_p and var_p are the exact GP
     kriging mean and variance of the response (dense Cholesky, scikit-learn kernels);
pp2  the paper's dense formulas P:143-146 (mean and covariance, first expression of Prop. 1) in
     un-whitened notation (Sigma_m^{-1}, Sigma_mn, M of P:117, B, D, B_po, D_p from P:85-97 and
     (vecchia_pred)) for tiny n, several (m, m_v) incl. m = 0 and m_v = 0; the oracle's variance uses
     the equivalent App. C.1 form, so pp2 also pins that equivalence.
"""
import numpy as np
import pytest

import oracle
import vifgen
from refs import sk_cov


def small(n, m, mv, family="matern32", neighbors="dc", seed=1, rho=0.15, nugget=0.1, d=2, ard=None):
    return vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=nugget, seed=seed,
                                device="cpu", neighbors=neighbors, ard=ard, z="kmeans++" if m > 0 else "subset")


@pytest.mark.parametrize("m", [0, 7])
@pytest.mark.parametrize("family", ["matern32", "matern52"])
def test_pp1_all_neighbours_is_exact_kriging(m, family):
    n = 80
    w = small(n, m, n, family=family, neighbors="all", seed=70 + m)
    Xp = np.random.default_rng(3).random((25, 2))
    nbrp = np.tile(np.arange(n, dtype=np.int32), (25, 1))
    mu, var, Dp, Bp = oracle.predict(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), Xp, nbrp)
    K = sk_cov(w.family, w.sigma2, w.lengthscale, w.X) + w.nugget * np.eye(n)
    Kp = sk_cov(w.family, w.sigma2, w.lengthscale, Xp, w.X)
    ref_mu = Kp @ np.linalg.solve(K, w.y)
    ref_var = w.sigma2 + w.nugget - np.einsum("ij,ji->i", Kp, np.linalg.solve(K, Kp.T))
    np.testing.assert_allclose(mu, ref_mu, rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(var, ref_var, rtol=1e-9)
    if m == 0:  # D_p is the residual process' conditional variance: the predictive variance only when m = 0
        np.testing.assert_allclose(Dp, ref_var, rtol=1e-9)
    else:
        assert np.all(Dp <= ref_var * (1 + 1e-12))


def paper_dense_prediction(w, Xp, nbrp):
    """P:143-144 (mu) and the D_p of (vecchia_pred), un-whitened, dense, for tiny n."""
    n, d, m = w.X.shape[0], w.X.shape[1], w.m
    K = sk_cov(w.family, w.sigma2, w.lengthscale, w.X)
    Kpn = sk_cov(w.family, w.sigma2, w.lengthscale, Xp, w.X)
    npred = Xp.shape[0]
    if m > 0:
        Z = w.Z.reshape(-1, d)
        Sm = sk_cov(w.family, w.sigma2, w.lengthscale, Z) + w.jitter * np.eye(m)
        Smn = sk_cov(w.family, w.sigma2, w.lengthscale, Z, w.X)
        Smp = sk_cov(w.family, w.sigma2, w.lengthscale, Z, Xp)
        Smi = np.linalg.inv(Sm)
        Ql, Qpn, Qpp = Smn.T @ Smi @ Smn, Smp.T @ Smi @ Smn, np.einsum("ai,ab,bi->i", Smp, Smi, Smp)
    else:
        Ql, Qpn, Qpp = np.zeros((n, n)), np.zeros((npred, n)), np.zeros(npred)
    St = K - Ql + w.nugget * np.eye(n)              # residual process + nugget (training)
    B, D = np.eye(n), np.zeros(n)
    for i in range(n):
        N = [j for j in w.nbr[i] if j >= 0]
        if N:
            A = np.linalg.solve(St[np.ix_(N, N)], St[N, i])
            B[i, N] = -A
            D[i] = St[i, i] - A @ St[N, i]
        else:
            D[i] = St[i, i]
    Bpo, Dp = np.zeros((npred, n)), np.zeros(npred)
    for t in range(npred):
        N = [j for j in nbrp[t] if j >= 0]
        cpn = Kpn[t, N] - Qpn[t, N]
        cpp = w.sigma2 + w.nugget - Qpp[t]
        if N:
            A = np.linalg.solve(St[np.ix_(N, N)], cpn)
            Bpo[t, N] = -A
            Dp[t] = cpp - A @ cpn
        else:
            Dp[t] = cpp
    P = B.T @ np.diag(1.0 / D) @ B                 # B^T D^{-1} B
    y = w.y
    if m > 0:
        M = Sm + Smn @ P @ Smn.T
        Mi = np.linalg.inv(M)
        t1 = Smp.T @ Smi @ Smn @ P @ y
        t2 = Smp.T @ Smi @ Smn @ P @ Smn.T @ Mi @ Smn @ P @ y
        t3 = Bpo @ Smn.T @ Mi @ Smn @ P @ y        # B_p^{-1} B_po ... with B_p = I
    else:
        t1 = t2 = t3 = 0.0
    mu = -Bpo @ y + t1 - t2 + t3
    # covariance, first expression of Prop. 1 with B_p = I
    Vs = np.linalg.inv(P)                          # (B^T D^{-1} B)^{-1}
    Sd = Ql + Vs                                   # Sigma_dagger (whitened: U U^T + B^{-1} D B^{-T})
    if m > 0:
        Qpn_full = Smp.T @ Smi @ Smn
        Qpp_full = Smp.T @ Smi @ Smp
    else:
        Qpn_full, Qpp_full = np.zeros((npred, n)), np.zeros((npred, npred))
    L = Qpn_full - Bpo @ Vs                        # Cov(y_p, y) = Sigma_mnp^T Sigma_m^-1 Sigma_mn - B_p^{-1} B_po V
    Sp = np.diag(Dp) + Bpo @ Vs @ Bpo.T + Qpp_full - L @ np.linalg.solve(Sd, L.T)
    return mu, Dp, Bpo, np.diag(Sp)


@pytest.mark.parametrize("family,m,mv", [("matern32", 10, 6), ("matern12", 6, 3), ("matern52", 0, 5),
                                          ("gaussian", 12, 0), ("matern32", 15, 1)])
def test_pp2_paper_dense_formula(family, m, mv):
    w = small(120, m, mv, family=family, seed=71, rho=0.2)
    Xp, nbrp = vifgen.make_prediction(w, 30, device="cpu")
    mu, var, Dp, Bp = oracle.predict(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), Xp, nbrp)
    rmu, rD, rBpo, rvar = paper_dense_prediction(w, Xp, nbrp)
    scale = np.abs(w.y).max()
    np.testing.assert_allclose(mu, rmu, rtol=1e-9, atol=1e-10 * scale)
    np.testing.assert_allclose(Dp, rD, rtol=1e-10)
    np.testing.assert_allclose(var, rvar, rtol=1e-9)
    for t in range(Xp.shape[0]):
        N = [j for j in nbrp[t] if j >= 0]
        np.testing.assert_allclose(Bp[t, :len(N)], rBpo[t, N], rtol=1e-9, atol=1e-12)


def test_pp2_ard_3d():
    w = small(100, 9, 5, family="matern52", seed=72, d=3, ard=(0.5, 2.0))
    Xp, nbrp = vifgen.make_prediction(w, 20, device="cpu")
    mu, var, Dp, _ = oracle.predict(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), Xp, nbrp)
    rmu, rD, _, rvar = paper_dense_prediction(w, Xp, nbrp)
    np.testing.assert_allclose(mu, rmu, rtol=1e-9, atol=1e-10 * np.abs(w.y).max())
    np.testing.assert_allclose(Dp, rD, rtol=1e-10)
    np.testing.assert_allclose(var, rvar, rtol=1e-9)


def test_prediction_neighbours_are_training_indices():
    w = small(300, 10, 8, seed=73)
    Xp, nbrp = vifgen.make_prediction(w, 50, device="cpu")
    assert nbrp.shape == (50, 8) and nbrp.min() >= 0 and nbrp.max() < 300
    assert all(len(set(r)) == 8 for r in nbrp)

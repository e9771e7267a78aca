"""Pins of the oracle's NLL gradient (Appendix A).

p13  central finite differences (Richardson-extrapolated) of the oracle's own NLL;
p14  the all-predecessor case is the exact GP: gradient = dense exact-GP gradient with kernel
     derivatives from scikit-learn (independent of oracle.c's or_dcov);
p15  the paper's dense gradient formula with dB, dD from Appendix A in the
     un-whitened notation (Sigma_m^{-1}, Sigma_mn), assembled in numpy for tiny n.
theta order: (sigma_1^2, lambda_1..lambda_d, sigma^2).
"""
import numpy as np
import pytest

import oracle
import vifgen
from refs import dense_grad, sk_cov, sk_cov_grad


def small(n, m, mv, family="matern32", neighbors="dc", seed=1, rho=0.15, nugget=0.1, d=2, ard=None):
    return vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=nugget, seed=seed,
                                device="cpu", neighbors=neighbors, ard=ard, z="kmeans++" if m > 0 else "subset")


def theta_vec(w):
    return np.concatenate([[w.sigma2], np.asarray(w.lengthscale, float), [w.nugget]])


def theta_from(w, v):
    d = w.X.shape[1]
    return oracle.Theta(w.family, float(v[0]), np.array(v[1:1 + d]), float(v[1 + d]), w.jitter)


def nll_at(w, v):
    return oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_from(w, v), want_BD=False).nll


def fd_grad(w, rel=1e-4):
    v0 = theta_vec(w)
    g = np.zeros_like(v0)
    for p in range(len(v0)):
        h = rel * v0[p]

        def central(hh):
            vp, vm = v0.copy(), v0.copy()
            vp[p] += hh
            vm[p] -= hh
            return (nll_at(w, vp) - nll_at(w, vm)) / (2 * hh)
        g[p] = (4 * central(h / 2) - central(h)) / 3      # Richardson: O(h^4)
    return g


def assert_grad_close(g, ref, parts, rtol):
    # per component: relative to the component or to the scale of its terms (the gradient at the
    # data-generating theta can be much smaller than the terms that cancel in it)
    scale = np.maximum(np.abs(ref), 0.5 * np.abs(parts).sum(axis=1))
    np.testing.assert_array_less(np.abs(g - ref), rtol * scale + 1e-300)


@pytest.mark.parametrize("family,m,mv", [("matern32", 12, 6), ("matern12", 0, 5), ("matern52", 20, 0),
                                          ("gaussian", 8, 4)])
def test_p13_gradient_matches_finite_differences(family, m, mv):
    w = small(150, m, mv, family=family, seed=61, rho=0.2)
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    fd = fd_grad(w)
    assert_grad_close(r.grad, fd, r.parts, rtol=2e-7)


def test_p13_ard_gradient_finite_differences():
    w = small(120, 10, 5, family="matern52", seed=62, d=3, ard=(0.5, 2.0))
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    assert_grad_close(r.grad, fd_grad(w), r.parts, rtol=2e-7)


def test_p13_off_theta_gradient():
    """Away from the data-generating theta the gradient is large; check it there too."""
    w = small(140, 10, 6, seed=63)
    v = theta_vec(w) * np.array([1.7, 0.6, 0.6, 2.5])
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, theta_from(w, v))
    g0 = np.zeros_like(v)
    for p in range(len(v)):
        h = 1e-4 * v[p]
        cen = lambda hh: (nll_at(w, v + hh * np.eye(len(v))[p]) - nll_at(w, v - hh * np.eye(len(v))[p])) / (2 * hh)
        g0[p] = (4 * cen(h / 2) - cen(h)) / 3
    assert np.all(np.abs(r.grad) > 1.0)
    np.testing.assert_allclose(r.grad, g0, rtol=1e-7)


@pytest.mark.parametrize("m", [0, 6])
@pytest.mark.parametrize("family", ["matern32", "gaussian"])
def test_p14_exact_case_equals_dense_gp_gradient(m, family):
    n = 90
    w = small(n, m, n - 1, family=family, neighbors="all", seed=64 + m)
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    K, dK = sk_cov_grad(w.family, w.sigma2, w.lengthscale, w.X)
    S = K + w.nugget * np.eye(n)
    dS = np.concatenate([dK, np.eye(n)[None]])
    ref = dense_grad(S, dS, w.y)
    assert_grad_close(r.grad, ref, r.parts, rtol=1e-9)


def paper_dense_gradient(w):
    """P:128-131 with Appendix A, un-whitened, for tiny n: returns dNLL/dtheta."""
    n, d, m = w.X.shape[0], w.X.shape[1], w.m
    XZ = np.vstack([w.X, w.Z.reshape(-1, d)]) if m > 0 else w.X
    Kall, dKall = sk_cov_grad(w.family, w.sigma2, w.lengthscale, XZ)
    P = d + 2
    # parameter derivatives of the blocks; the nugget is the last parameter
    dK = [dKall[p] for p in range(d + 1)] + [np.zeros_like(Kall)]
    Kn, dKn = Kall[:n, :n], [a[:n, :n] for a in dK]
    if m > 0:
        Smn, dSmn = Kall[n:, :n], [a[n:, :n] for a in dK]
        Sm = Kall[n:, n:] + w.jitter * np.eye(m)
        dSm = [a[n:, n:] for a in dK]
        Smi = np.linalg.inv(Sm)
        Sl = Smn.T @ Smi @ Smn
        dSl = [dSmn[p].T @ Smi @ Smn + Smn.T @ Smi @ dSmn[p] - Smn.T @ Smi @ dSm[p] @ Smi @ Smn for p in range(P)]
    else:
        Sl, dSl = np.zeros((n, n)), [np.zeros((n, n))] * P
    # residual (bracket) covariances with the nugget by index identity
    St = Kn - Sl + w.nugget * np.eye(n)
    dSt = [dKn[p] - dSl[p] + (np.eye(n) if p == P - 1 else 0.0) for p in range(P)]
    B, D = np.eye(n), np.zeros(n)
    dB, dD = [np.zeros((n, n)) for _ in range(P)], np.zeros((P, n))
    for i in range(n):
        N = [j for j in w.nbr[i] if j >= 0]
        if N:
            SNi = np.linalg.inv(St[np.ix_(N, N)])
            A = St[i, N] @ SNi
            B[i, N] = -A
            D[i] = St[i, i] - A @ St[N, i]
            for p in range(P):
                dA = (dSt[p][i, N] - A @ dSt[p][np.ix_(N, N)]) @ SNi          # Appendix A
                dB[p][i, N] = -dA
                dD[p, i] = dSt[p][i, i] - dA @ St[N, i] - A @ dSt[p][N, i]
        else:
            D[i] = St[i, i]
            for p in range(P):
                dD[p, i] = dSt[p][i, i]
    Bi = np.linalg.inv(B)
    Ss = Bi @ np.diag(D) @ Bi.T
    Sd = Sl + Ss
    dSd = []
    for p in range(P):
        dSs = Bi @ np.diag(dD[p]) @ Bi.T - Bi @ dB[p] @ Bi @ np.diag(D) @ Bi.T - Bi @ np.diag(D) @ Bi.T @ dB[p].T @ Bi.T
        dSd.append(dSs + dSl[p])
    return dense_grad(Sd, dSd, w.y)


@pytest.mark.parametrize("family,m,mv", [("matern32", 10, 5), ("matern12", 6, 3), ("matern52", 0, 4),
                                          ("gaussian", 12, 0)])
def test_p15_paper_dense_formula(family, m, mv):
    w = small(110, m, mv, family=family, seed=65, rho=0.2)
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    ref = paper_dense_gradient(w)
    assert_grad_close(r.grad, ref, r.parts, rtol=1e-9)


def test_p15_paper_dense_formula_ard():
    w = small(100, 9, 5, family="matern32", seed=66, d=3, ard=(0.5, 2.0))
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    assert_grad_close(r.grad, paper_dense_gradient(w), r.parts, rtol=1e-9)


def test_oracle_dcov_matches_sklearn():
    rng = np.random.default_rng(7)
    A = rng.standard_normal((12, 3))
    ls = np.array([0.7, 1.3, 2.0])
    for fam in ["matern12", "matern32", "matern52", "gaussian"]:
        th = oracle.Theta(fam, 1.4, ls, 0.0, 0.0)
        got = oracle.dcov_matrix(th, A, A)
        K, dK = sk_cov_grad(fam, 1.4, ls, A)
        np.testing.assert_allclose(got, dK, rtol=1e-10, atol=1e-13)

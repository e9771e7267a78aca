"""Pins of the VIF-Laplace oracle (oracle/laplace.py, Sect. 3-4).

la1  Bernoulli-logit log-likelihood, gradient and W against scipy's Bernoulli pmf and central differences;
la2  all predecessors as neighbours: the latent VIF is exact, so Sigma_dagger v = K v with K the
     dense covariance from scikit-learn's kernels (no nugget);
la3  Sigma_dagger^{-1} (Woodbury) inverts Sigma_dagger (triangular solves + low rank);
la4  FITC preconditioner (App. FITC) against a dense P = diag(K - Q) + W^{-1} + Q,
     Q = K_nk K_k^{-1} K_kn built from scikit-learn's kernels: solve, log-determinant, and the sample
     covariance of z = D_V^{1/2} eps2 + U eps1;
la5  the Lanczos tridiagonal matrix from the CG coefficients: after n steps its eigenvalues are
     those of P^{-1/2} A P^{-1/2} and ||P^{-1/2} z||^2 e_1^T log(T) e_1 = z^T P^{-1/2} log(P^{-1/2} A P^{-1/2})
     P^{-1/2} z (symmetric root, dense eigendecompositions);
la6  exact case: the mode and L^LA with the exact log-determinant equal the textbook Laplace
     approximation (Rasmussen & Williams 2006, Alg. 3.1: Newton on f with B = I + W^1/2 K W^1/2);
la7  general case: the mode is stationary, b~ = Sigma_dagger (y - pi(b~)), and the exact quadratic term
     matches a dense solve;
la8  SLQ (slq_v2) is unbiased: the mean over many probes is within 4 standard errors of the dense
     log det(Sigma_dagger W + I).
"""
import numpy as np
import pytest
from scipy import stats

import oracle
from oracle import laplace as la
import vifgen
from refs import sk_cov


def work(n, m, mv, neighbors="dc", family="matern32", seed=1, d=2, rho=0.2):
    return vifgen.make_laplace_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, seed=seed, device="cpu",
                                        neighbors=neighbors, z="kmeans++" if m > 0 else "subset")


def theta(w):
    return oracle.Theta(**w.theta_dict())


def dense_K(w):
    return sk_cov(w.family, w.sigma2, w.lengthscale, w.X)


def test_la1_likelihood():
    rng = np.random.default_rng(0)
    b = rng.normal(0, 2, 50)
    y = (rng.random(50) < 0.4).astype(float)
    ref = np.sum(stats.bernoulli.logpmf(y, 1 / (1 + np.exp(-b))))
    assert la.loglik(y, b) == pytest.approx(ref, rel=1e-12)
    h = 1e-5
    g_fd = np.array([(la.loglik(y, b + h * e) - la.loglik(y, b - h * e)) / (2 * h) for e in np.eye(50)])
    np.testing.assert_allclose(la.grad_loglik(y, b), g_fd, rtol=1e-7, atol=1e-9)
    w_fd = -(la.grad_loglik(y, b + h) - la.grad_loglik(y, b - h)) / (2 * h)
    np.testing.assert_allclose(la.hess_w(b), w_fd, rtol=1e-6, atol=1e-10)


@pytest.mark.parametrize("m", [0, 6])
def test_la2_all_predecessors_is_exact(m):
    n = 60
    w = work(n, m, n, neighbors="all", seed=3 + m)
    lat = la.latent_factor(w.X, w.Z, w.nbr, theta(w))
    V = np.random.default_rng(1).standard_normal((n, 3))
    np.testing.assert_allclose(lat.sigma_dagger(V), dense_K(w) @ V, rtol=1e-8, atol=1e-9)


def test_la3_woodbury_inverse():
    w = work(300, 12, 8, seed=4)
    lat = la.latent_factor(w.X, w.Z, w.nbr, theta(w))
    v = np.random.default_rng(2).standard_normal(300)
    np.testing.assert_allclose(lat.sigma_dagger_inv(lat.sigma_dagger(v)), v, rtol=1e-7, atol=1e-7)


def test_la4_fitc_dense():
    n, m = 90, 9
    w = work(n, m, 6, seed=5)
    lat = la.latent_factor(w.X, w.Z, w.nbr, theta(w))
    W = la.hess_w(np.random.default_rng(3).normal(0, 1.5, n))
    P = la.fitc(lat, W)
    K = dense_K(w)
    Kk = sk_cov(w.family, w.sigma2, w.lengthscale, w.Z) + w.jitter * np.eye(m)
    Knk = sk_cov(w.family, w.sigma2, w.lengthscale, w.X, w.Z)
    Q = Knk @ np.linalg.solve(Kk, Knk.T)
    Pd = np.diag(np.diag(K - Q) + 1 / W) + Q
    v = np.random.default_rng(4).standard_normal((n, 2))
    np.testing.assert_allclose(P.solve(v), np.linalg.solve(Pd, v), rtol=1e-8, atol=1e-10)
    assert P.logdet() == pytest.approx(np.linalg.slogdet(Pd)[1], rel=1e-10)
    # sample covariance of z = D_V^{1/2} eps2 + U eps1 on 5 rows
    eps1, eps2 = vifgen.make_probes(n, m, 200000, seed=9)
    rows = [0, 7, 30, 55, 89]
    Zs = np.sqrt(P.DV[rows])[:, None] * eps2[rows] + lat.U[rows] @ eps1
    C = Zs @ Zs.T / Zs.shape[1]
    se = np.sqrt((Pd[np.ix_(rows, rows)] ** 2 + np.outer(np.diag(Pd)[rows], np.diag(Pd)[rows])) / Zs.shape[1])
    assert np.all(np.abs(C - Pd[np.ix_(rows, rows)]) < 5 * se)


def _sym_pow(S, f):
    lam, V = np.linalg.eigh(S)
    return (V * f(lam)) @ V.T


def test_la5_lanczos_from_cg():
    n = 14
    w = work(n, 3, 4, seed=6)
    lat = la.latent_factor(w.X, w.Z, w.nbr, theta(w))
    W = la.hess_w(np.random.default_rng(5).normal(0, 1, n))
    P = la.fitc(lat, W)
    A = np.diag(1 / W) + lat.sigma_dagger(np.eye(n))
    A = 0.5 * (A + A.T)
    z = np.random.default_rng(6).standard_normal(n)
    res = la.pcg(lambda p: A @ p, z, P.solve, 0.0, n)
    T = la.lanczos_tridiag(res.alpha, res.beta)
    Pd = np.linalg.inv(P.solve(np.eye(n)))
    Pm = _sym_pow(0.5 * (Pd + Pd.T), lambda l: l ** -0.5)
    At = Pm @ A @ Pm
    # (finite-precision CG after n steps: loss of orthogonality leaves ~1e-7 on a clustered spectrum)
    np.testing.assert_allclose(np.linalg.eigvalsh(T), np.linalg.eigvalsh(At), rtol=1e-6)
    lhs = np.sum((Pm @ z) ** 2) * la.e1_log_e1(T)
    rhs = (Pm @ z) @ _sym_pow(At, np.log) @ (Pm @ z)
    assert lhs == pytest.approx(rhs, rel=1e-6)


def _gpml_laplace(K, y, tol=1e-14, max_it=100):
    """Rasmussen & Williams (2006), Algorithm 3.1, for the logistic likelihood."""
    n = len(y)
    f = np.zeros(n)
    obj_old = -np.inf
    for _ in range(max_it):
        pi = 1 / (1 + np.exp(-f))
        Wd = pi * (1 - pi)
        sW = np.sqrt(Wd)
        L = np.linalg.cholesky(np.eye(n) + sW[:, None] * K * sW[None, :])
        bb = Wd * f + (y - pi)
        a = bb - sW * np.linalg.solve(L.T, np.linalg.solve(L, sW * (K @ bb)))
        f = K @ a
        obj = -0.5 * a @ f + np.sum(y * f - np.logaddexp(0, f))
        if abs(obj - obj_old) < tol * abs(obj):
            break
        obj_old = obj
    pi = 1 / (1 + np.exp(-f))
    sW = np.sqrt(pi * (1 - pi))
    L = np.linalg.cholesky(np.eye(n) + sW[:, None] * K * sW[None, :])
    a = np.linalg.solve(K, f)
    logq = -0.5 * a @ f + np.sum(y * f - np.logaddexp(0, f)) - np.sum(np.log(np.diag(L)))
    return f, -logq


@pytest.mark.parametrize("m", [0, 5])
def test_la6_exact_case_is_textbook_laplace(m):
    n = 45
    w = work(n, m, n, neighbors="all", seed=10 + m, rho=0.3)
    lat = la.latent_factor(w.X, w.Z, w.nbr, theta(w))
    r = la.vifla_nll(w.X, w.Z, w.nbr, w.y, theta(w), lat=lat, newton_tol=1e-14, cg_tol=1e-13)
    f, nll_ref = _gpml_laplace(dense_K(w), w.y)
    np.testing.assert_allclose(r.b, f, rtol=1e-6, atol=1e-7)
    nll = r.neg_loglik + 0.5 * r.quad + 0.5 * la.exact_logdet(lat, la.hess_w(r.b))
    assert nll == pytest.approx(nll_ref, rel=1e-8)


def test_la7_mode_stationary_and_quad():
    w = work(400, 15, 10, seed=12)
    lat = la.latent_factor(w.X, w.Z, w.nbr, theta(w))
    r = la.vifla_nll(w.X, w.Z, w.nbr, w.y, theta(w), lat=lat, newton_tol=1e-13, cg_tol=1e-12)
    g = la.grad_loglik(w.y, r.b)
    np.testing.assert_allclose(lat.sigma_dagger(g), r.b, rtol=1e-7, atol=1e-8)
    S = lat.sigma_dagger(np.eye(400))
    assert r.quad == pytest.approx(r.b @ np.linalg.solve(0.5 * (S + S.T), r.b), rel=1e-6)
    np.testing.assert_allclose(r.a, g, rtol=1e-6, atol=1e-8)  # a = Sigma^-1 b~ = grad at the mode


def test_la8_slq_unbiased():
    n, m, ell = 150, 8, 600
    w = work(n, m, 6, seed=13)
    lat = la.latent_factor(w.X, w.Z, w.nbr, theta(w))
    W = la.hess_w(np.random.default_rng(7).normal(0, 1, n))
    eps1, eps2 = vifgen.make_probes(n, m, ell, seed=14)
    est, iters, parts = la.slq_logdet(lat, W, eps1, eps2, tol=1e-10)
    terms = np.asarray(parts["slq_terms"]) * n + parts["logdet_W"] + parts["logdet_P"]
    exact = la.exact_logdet(lat, W)
    assert est == pytest.approx(terms.mean(), rel=1e-12)
    assert abs(est - exact) < 4 * terms.std(ddof=1) / np.sqrt(ell)

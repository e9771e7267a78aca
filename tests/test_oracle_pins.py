"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every reference here is independent of the oracle's code: kernels from scikit-learn,
dense linear algebra from LAPACK (numpy/scipy), closed forms from tests/golden/.
"""
import math
import os

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

import oracle
import vifgen
from refs import B_matrix, dense_nll, nystrom, sk_cov

HERE = os.path.dirname(os.path.abspath(__file__))


def theta_of(w):
    return oracle.Theta(**w.theta_dict())


def small(n, m, mv, family="matern32", neighbors="dc", seed=1, rho=0.15, nugget=0.1, d=2, ard=None, x="uniform"):
    return vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=nugget, seed=seed,
                                device="cpu", neighbors=neighbors, ard=ard, x=x,
                                z="kmeans++" if m > 0 else "subset")


# ---------------- p9: kernel closed forms ----------------
def test_p9_kernel_golden_values():
    path = os.path.join(HERE, "golden", "kernel_closed_forms.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    assert len(rows) >= 5
    for fam, s2, ls, dist, val in rows:
        th = oracle.Theta(fam, float(s2), [float(ls)], 0.0, 0.0)
        k = oracle.cov_matrix(th, np.array([[0.0]]), np.array([[float(dist)]]))[0, 0]
        assert k == pytest.approx(float(val), rel=1e-14, abs=1e-15), (fam, s2, ls, dist)


@pytest.mark.parametrize("family", ["matern12", "matern32", "matern52", "gaussian"])
def test_p9_kernel_matches_sklearn_ard(family):
    rng = np.random.default_rng(3)
    d = 4
    ls = np.exp(rng.uniform(-1, 1, d))
    A, B = rng.standard_normal((7, d)), rng.standard_normal((9, d))
    th = oracle.Theta(family, 1.7, ls, 0.0, 0.0)
    K = oracle.cov_matrix(th, A, B)
    R = sk_cov(family, 1.7, ls, A, B)
    np.testing.assert_allclose(K, R, rtol=1e-12, atol=1e-15)
    # symmetry and k(x,x) = sigma_1^2
    Kaa = oracle.cov_matrix(th, A, A)
    assert np.array_equal(Kaa, Kaa.T)
    np.testing.assert_allclose(np.diag(Kaa), 1.7, rtol=0, atol=0)


# ---------------- p1: exact GP when N(i) = all predecessors ----------------
@pytest.mark.parametrize("m", [0, 5, 30])
def test_p1_exact_gp_when_all_predecessors(m):
    n = 120
    w = small(n, m, n - 1, neighbors="all", seed=10 + m)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w))
    S = sk_cov(w.family, w.sigma2, w.lengthscale, w.X) + w.nugget * np.eye(n)
    ref = dense_nll(S, w.y)
    assert r.nll == pytest.approx(ref, rel=1e-10)


# ---------------- p10: reorder invariance in the exact case ----------------
def test_p10_reorder_invariance_exact_case():
    n = 100
    w = small(n, 8, n - 1, neighbors="all", seed=21)
    r1 = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w))
    perm = np.random.default_rng(5).permutation(n)
    r2 = oracle.factor_nll(w.X[perm], w.Z, w.nbr, w.y[perm], theta_of(w))
    assert r2.nll == pytest.approx(r1.nll, rel=1e-10)


# ---------------- p2: m = 0 is classical Vecchia ----------------
def test_p2_m0_is_classical_vecchia():
    n, mv = 300, 7
    w = small(n, 0, mv, seed=31)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w))
    S = sk_cov(w.family, w.sigma2, w.lengthscale, w.X) + w.nugget * np.eye(n)
    nll = 0.5 * n * math.log(2 * math.pi)
    for i in range(n):
        N = [j for j in w.nbr[i] if j >= 0]
        if N:
            A = np.linalg.solve(S[np.ix_(N, N)], S[N, i])         # LU conditional regression
            D = S[i, i] - A @ S[N, i]
            res = w.y[i] - A @ w.y[N]
        else:
            A, D, res = np.zeros(0), S[i, i], w.y[i]
        np.testing.assert_allclose(-r.B[i, :len(N)], A, rtol=1e-10, atol=1e-12)
        assert r.D[i] == pytest.approx(D, rel=1e-12)
        nll += 0.5 * (math.log(D) + res * res / D)              # product of univariate conditionals
    assert r.nll == pytest.approx(nll, rel=1e-11)
    assert r.logdet_M == 0.0


# ---------------- p3: m_v = 0 is FITC ----------------
def test_p3_mv0_is_fitc():
    n, m = 300, 20
    w = small(n, m, 0, seed=41)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w))
    Q = nystrom(w)
    S = sk_cov(w.family, w.sigma2, w.lengthscale, w.X) + w.nugget * np.eye(n)
    F = Q + np.diag(np.diag(S - Q))
    assert r.nll == pytest.approx(dense_nll(F, w.y), rel=1e-10)


# ---------------- p5: each B row is the exact conditional of the residual process ------
@pytest.mark.parametrize("family", ["matern12", "matern32", "matern52", "gaussian"])
def test_p5_exact_conditionals(family):
    n, m, mv = 400, 15, 8
    w = small(n, m, mv, family=family, seed=51, rho=0.2)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w))
    C = sk_cov(w.family, w.sigma2, w.lengthscale, w.X) + w.nugget * np.eye(n) - nystrom(w)
    for i in range(n):
        N = [j for j in w.nbr[i] if j >= 0]
        if N:
            A = scipy.linalg.lu_solve(scipy.linalg.lu_factor(C[np.ix_(N, N)]), C[N, i])
            D = C[i, i] - A @ C[N, i]
        else:
            A, D = np.zeros(0), C[i, i]
        np.testing.assert_allclose(-r.B[i, :len(N)], A, rtol=1e-9, atol=1e-11)
        assert r.D[i] == pytest.approx(D, rel=1e-10)
        assert np.all(r.B[i, len(N):] == 0.0)


def test_p5_sampled_rows_match_full_oracle():
    w = small(500, 12, 6, seed=52)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w), want_U=True)
    rows = np.array([0, 1, 5, 77, 499, 250])
    U, B, D = oracle.rows(w.X, w.Z, w.nbr, theta_of(w), rows, want_U=True)
    np.testing.assert_allclose(U, r.U[rows], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(B, r.B[rows], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(D, r.D[rows], rtol=1e-13)


# ---------------- p4: Woodbury + Sylvester vs dense assembly of Sigma_dagger ---------
def test_p4_dense_assembly_identity():
    n, m, mv = 400, 10, 5
    w = small(n, m, mv, seed=61)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w), want_U=True)
    B = B_matrix(w.nbr, r.B)
    Binv = scipy.linalg.solve_triangular(B, np.eye(n), lower=True, unit_diagonal=True)
    Sd = r.U @ r.U.T + Binv @ np.diag(r.D) @ Binv.T
    sign, logdet = np.linalg.slogdet(Sd)
    assert sign > 0
    quad = w.y @ np.linalg.solve(Sd, w.y)
    assert r.logdet_D + r.logdet_M == pytest.approx(logdet, rel=1e-10)
    assert r.quad == pytest.approx(quad, rel=1e-9)
    assert r.nll == pytest.approx(dense_nll(Sd, w.y), rel=1e-10)


# ---------------- p12: whitened M_w vs the paper's M (Eq. def_M) ----------------
def test_p12_whitened_equals_paper_form():
    n, m, mv = 300, 12, 6
    w = small(n, m, mv, seed=71)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w))
    B = B_matrix(w.nbr, r.B)
    Sm = sk_cov(w.family, w.sigma2, w.lengthscale, w.Z) + w.jitter * np.eye(m)
    Smn = sk_cov(w.family, w.sigma2, w.lengthscale, w.Z, w.X)
    BtDB = B.T @ np.diag(1.0 / r.D) @ B
    M = Sm + Smn @ BtDB @ Smn.T
    lhs = np.linalg.slogdet(M)[1] - np.linalg.slogdet(Sm)[1]
    assert lhs == pytest.approx(r.logdet_M, rel=1e-9)
    # Woodbury quad with the paper's M
    v = Smn @ BtDB @ w.y
    quad = w.y @ BtDB @ w.y - v @ np.linalg.solve(M, v)
    assert quad == pytest.approx(r.quad, rel=1e-9)


# ---------------- p6: invariants (D_i >= sigma^2) ----------------
def test_p6_invariants_config1():
    w = vifgen.make_config(1, device="cpu")
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, theta_of(w), want_U=True)
    Cii = w.sigma2 + w.nugget - (r.U * r.U).sum(1)
    assert np.all(r.D >= w.nugget * (1 - 1e-12))
    assert np.all(r.D <= Cii * (1 + 1e-12))
    assert r.D[0] == pytest.approx(Cii[0], rel=1e-14)
    assert r.logdet_M >= 0.0
    B = B_matrix(w.nbr, r.B)
    rt = (B @ w.y) / np.sqrt(r.D)
    assert 0.0 <= r.quad <= rt @ rt * (1 + 1e-12)


# ---------------- p7: chi^2 moment of y ~ N(0, Sigma_dagger) ----------------
def test_p7_chi2_moment():
    n, m, mv = 3000, 20, 8
    w = small(n, m, mv, seed=81, rho=0.08)
    th = theta_of(w)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, th, want_U=True)
    rows, cols, vals = [], [], []
    for i in range(n):
        for k in range(mv):
            if w.nbr[i, k] >= 0:
                rows.append(i); cols.append(w.nbr[i, k]); vals.append(r.B[i, k])
    Bs = scipy.sparse.csr_matrix((vals, (rows, cols)), shape=(n, n)) + scipy.sparse.identity(n, format="csr")
    rng = np.random.default_rng(7)
    reps = 12
    q = 0.0
    for _ in range(reps):
        yy = r.U @ rng.standard_normal(m) + scipy.sparse.linalg.spsolve_triangular(
            Bs, np.sqrt(r.D) * rng.standard_normal(n), lower=True)
        q += oracle.factor_nll(w.X, w.Z, w.nbr, yy, th).quad
    q /= reps * n
    assert abs(q - 1.0) < 5 * math.sqrt(2.0 / (reps * n))


# ---------------- p8: scalar cases ----------------
def test_p8_scalar_n1_m0():
    th = oracle.Theta("matern32", 1.3, [0.2], 0.4, 0.0)
    X = np.array([[0.3, 0.7]])[:, :1]
    r = oracle.factor_nll(X, np.zeros((0, 1)), np.zeros((1, 0), np.int32), np.array([0.9]), th)
    s = 1.3 + 0.4
    assert r.nll == pytest.approx(0.5 * math.log(2 * math.pi) + 0.5 * math.log(s) + 0.81 / (2 * s), rel=1e-14)


def test_p8_scalar_n1_with_inducing():
    rng = np.random.default_rng(2)
    Z = rng.random((3, 2))
    X = rng.random((1, 2))
    th = oracle.Theta("matern52", 1.0, [0.3, 0.3], 0.05, 1e-10)
    r = oracle.factor_nll(X, Z, np.zeros((1, 2), np.int32) - 1, np.array([0.2]), th)
    Km = sk_cov("matern52", 1.0, [0.3, 0.3], Z) + 1e-10 * np.eye(3)
    k = sk_cov("matern52", 1.0, [0.3, 0.3], Z, X)[:, 0]
    D = 1.0 + 0.05 - k @ np.linalg.solve(Km, k)
    assert r.D[0] == pytest.approx(D, rel=1e-12)
    assert np.all(r.B == 0.0)


# ---------------- sharding algebra: partial sums over a row partition (p11 for the oracle) -------
def test_partial_sums_partition_equals_full():
    w = small(600, 10, 6, seed=91)
    th = theta_of(w)
    full = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, th)
    G = np.zeros((w.m, w.m)); v = np.zeros(w.m); s = np.zeros(2)
    for part in np.array_split(np.random.default_rng(0).permutation(w.n), 3):
        g, vv, ss = oracle.partial(w.X, w.Z, w.nbr, w.y, th, part)
        G += g; v += vv; s += ss
    t = oracle.finish(w.n, G, v, s)
    assert t[0] == pytest.approx(full.nll, rel=1e-12)
    assert t[3] == pytest.approx(full.quad, rel=1e-10)


def test_neighbor_validation():
    nbr = np.array([[-1, -1], [0, -1], [1, 0]], np.int32)
    assert oracle.check_neighbors(nbr) == -1
    assert oracle.check_neighbors(np.array([[-1, -1], [1, -1], [1, 0]], np.int32)) == 1  # j >= i
    assert oracle.check_neighbors(np.array([[-1, -1], [0, -1], [0, 0]], np.int32)) == 2  # duplicate
    assert oracle.check_neighbors(np.array([[-1, -1], [-1, 0], [1, 0]], np.int32)) == 1  # pad not trailing


def test_not_pd_reports_row():
    # two coincident points with zero nugget: C_NN singular at the second row's conditioning set
    X = np.array([[0.1, 0.1], [0.5, 0.5], [0.5, 0.5], [0.7, 0.2]])
    nbr = np.array([[-1, -1], [0, -1], [1, 0], [2, 1]], np.int32)
    th = oracle.Theta("matern32", 1.0, [0.3, 0.3], 0.0, 0.0)
    with pytest.raises(oracle.OracleError) as e:
        oracle.factor_nll(X, np.zeros((0, 2)), nbr, np.zeros(4), th)
    assert e.value.status == 2 and e.value.bad_row in (2, 3)

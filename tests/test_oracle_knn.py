"""Pins of the oracle's correlation-distance neighbour search.

pk1  with m = 0 and an isotropic stationary kernel, |corr| is decreasing in the distance, so N(i) are
     the Euclidean nearest predecessors (brute force with numpy, ties by index);
pk2  against the input generator's independent torch implementation (vifgen.dc_neighbors), with m > 0
     and ARD length-scales: identical sets, except at exact score ties where both must be valid;
pk3  structural rules: predecessors only, i <= m_v takes all predecessors, scores non-increasing.
"""
import numpy as np
import pytest

import oracle
import vifgen


def small(n, m, mv, family="matern32", seed=1, rho=0.15, d=2, ard=None, z="kmeans++"):
    return vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=0.1, seed=seed,
                                device="cpu", ard=ard, z=z if m > 0 else "subset")


@pytest.mark.parametrize("family", ["matern12", "matern32", "gaussian"])
def test_pk1_m0_is_euclidean_knn_among_predecessors(family):
    w = small(400, 0, 9, family=family, seed=80)
    nbr, sc = oracle.dc_neighbors(w.X, w.Z, oracle.Theta(**w.theta_dict()), 9)
    for i in range(400):
        d2 = ((w.X[:i] - w.X[i]) ** 2).sum(1)
        ref = np.lexsort((np.arange(i), d2))[:min(9, i)]
        np.testing.assert_array_equal(nbr[i, :len(ref)], ref)
        assert np.all(nbr[i, len(ref):] == -1)


@pytest.mark.parametrize("m,ard,z", [(20, None, "kmeans++"), (12, (0.5, 2.0), "kmeans++"), (15, None, "subset")])
def test_pk2_matches_generator(m, ard, z):
    w = small(500, m, 10, seed=81, ard=ard, d=3 if ard else 2, z=z)
    th = oracle.Theta(**w.theta_dict())
    nbr, sc = oracle.dc_neighbors(w.X, w.Z, th, 10)
    diff = np.nonzero((nbr != w.nbr).any(1))[0]
    for i in diff:  # only legitimate at (near) ties: the sets' scores must agree to rounding
        a = oracle.dc_scores(w.X, w.Z, th, np.full(10, i), nbr[i][nbr[i] >= 0])
        b = oracle.dc_scores(w.X, w.Z, th, np.full(10, i), w.nbr[i][w.nbr[i] >= 0])
        np.testing.assert_allclose(np.sort(a), np.sort(b), rtol=1e-12, atol=1e-15)
    assert len(diff) <= 2


def test_pk3_structure():
    w = small(300, 10, 8, seed=82)
    nbr, sc = oracle.dc_neighbors(w.X, w.Z, oracle.Theta(**w.theta_dict()), 8)
    for i in range(300):
        row = nbr[i][nbr[i] >= 0]
        assert len(row) == min(i, 8) and np.all(row < i) and len(set(row)) == len(row)
        s = sc[i][:len(row)]
        assert np.all(np.diff(s) <= 0)


# ---------------------------------------------------------------------------------------------
# pk4: the paper's definition written out densely, independently of the oracle and of vifgen
def dense_dc_reference(w, tau_rel=1e-7):
    """Scores of every (i, j < i) pair straight from P:509-513, un-whitened and dense:
    rho_c(i, j) = Sigma_ij - Sigma_mi^T Sigma_m^{-1} Sigma_mj (Sigma WITHOUT the nugget; Sigma_m with the
    theta jitter, reading c3; LU solve, scikit-learn kernels), corr = |rho_c(i,j)| / sqrt(rho_c(i,i) rho_c(j,j)),
    d_c = sqrt(1 - corr): smallest d_c = largest corr.  Reading c7: a candidate j with rho_c(j,j) < 1e-7 sigma_1^2
    has d_c = 1 (corr 0); a degenerate query ranks its predecessors by the length-scale-scaled Euclidean
    distance (score -dist^2).  Returns the n x n score matrix (upper triangle unused)."""
    from refs import sk_cov
    K = sk_cov(w.family, w.sigma2, w.lengthscale, w.X)
    if w.m > 0:
        Km = sk_cov(w.family, w.sigma2, w.lengthscale, w.Z) + w.jitter * np.eye(w.m)
        Knm = sk_cov(w.family, w.sigma2, w.lengthscale, w.X, w.Z)
        rho = K - Knm @ np.linalg.solve(Km, Knm.T)
    else:
        rho = K
    rd = np.diag(rho).copy()
    deg = rd < tau_rel * w.sigma2
    safe = np.where(deg, 1.0, rd)
    corr = np.abs(rho) / np.sqrt(np.outer(safe, safe))
    corr[:, deg] = 0.0
    Xs = w.X / w.lengthscale
    d2 = ((Xs[:, None, :] - Xs[None, :, :]) ** 2).sum(-1)
    corr[deg, :] = -d2[deg, :]
    return corr, deg


def _check_sets_against_dense(w, nbr, corr, tol, max_mismatch):
    n, mv = nbr.shape
    mismatches = 0
    for i in range(n):
        cand = np.arange(i)
        sc = corr[i, :i]
        ref = cand[np.lexsort((cand, -sc))][:min(mv, i)]   # (corr desc, index asc): reading c6
        got = nbr[i][nbr[i] >= 0]
        assert len(got) == min(mv, i) and np.all(got < i) and len(set(got.tolist())) == len(got)
        if np.array_equal(got, ref):
            continue
        mismatches += 1
        # a different choice is only legitimate at a tie under the dense scores' own rounding: the chosen set
        # must be a valid top-m_v (its worst score >= the best unchosen score - tol) in non-increasing order
        rest = np.setdiff1d(cand, got)
        worst = sc[got].min()
        best_rest = sc[rest].max() if len(rest) else -np.inf
        assert worst >= best_rest - tol, (i, worst, best_rest)
        assert np.all(np.diff(sc[got]) <= tol), i
    assert mismatches <= max_mismatch, mismatches


@pytest.mark.parametrize("family,m,ard,z,d", [
    ("matern32", 20, None, "kmeans++", 2),
    ("matern12", 15, None, "kmeans++", 2),
    ("matern52", 12, (0.5, 2.0), "kmeans++", 3),
    ("gaussian", 10, None, "kmeans++", 2),
])
def test_pk4_dense_unwhitened_definition(family, m, ard, z, d):
    """oracle_dc_neighbors / oracle_dc_scores for m > 0 against the dense un-whitened Nystrom form of P:509-513
    (not the generator's whitened copy): sets equal except at rounding-level ties, scores to 1e-9."""
    w = small(350, m, 9, family=family, seed=90 + m, ard=ard, d=d, z=z)
    th = oracle.Theta(**w.theta_dict())
    nbr, sc = oracle.dc_neighbors(w.X, w.Z, th, 9)
    corr, deg = dense_dc_reference(w)
    assert not deg.any()
    _check_sets_against_dense(w, nbr, corr, tol=1e-9, max_mismatch=3)
    # the oracle's scores of its chosen pairs equal the dense definition's
    for i in range(1, w.n, 7):
        got = nbr[i][nbr[i] >= 0]
        np.testing.assert_allclose(sc[i][:len(got)], corr[i, got], rtol=1e-9, atol=1e-12)
    qi = np.repeat(np.arange(50, 60), 8)
    cj = np.concatenate([np.random.default_rng(i).choice(i, 8, replace=False) for i in range(50, 60)])
    np.testing.assert_allclose(oracle.dc_scores(w.X, w.Z, th, qi, cj), corr[qi, cj], rtol=1e-9, atol=1e-12)


def test_pk4_degenerate_inducing_points_at_data_points():
    """Reading c7 with inducing points at data points (config-1 style subset Z): those points have residual
    variance ~ jitter; as candidates they score d_c = 1, as queries they rank predecessors by scaled distance --
    the dense definition and the oracle agree on which points are degenerate and on every set."""
    w = small(300, 25, 8, seed=97, z="subset")
    th = oracle.Theta(**w.theta_dict())
    nbr, sc = oracle.dc_neighbors(w.X, w.Z, th, 8)
    corr, deg = dense_dc_reference(w)
    assert deg.sum() == 25
    _check_sets_against_dense(w, nbr, corr, tol=1e-9, max_mismatch=3)
    for i in np.nonzero(deg)[0]:
        if i == 0:
            continue
        d2 = (((w.X[:i] - w.X[i]) / w.lengthscale) ** 2).sum(1)
        ref = np.lexsort((np.arange(i), d2))[:min(8, i)]
        np.testing.assert_array_equal(nbr[i, :len(ref)], ref)

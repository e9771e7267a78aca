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

"""The input generator's own pruned neighbour search (vifgen.dc_neighbors_pruned) returns exactly the sets of
its brute force (vifgen.dc_neighbors) -- both are vifgen's torch code; the oracle pins the definition itself
(tests/test_oracle_knn.py pk4).  CPU, small n with a small prefix so the pruning is exercised."""
import numpy as np
import pytest

import vifgen


@pytest.mark.parametrize("n,d,m,mv,family,z", [
    (3000, 2, 30, 10, "matern32", "kmeans++"),
    (2500, 3, 20, 8, "matern12", "kmeans++"),
    (2000, 2, 25, 12, "matern32", "subset"),   # degenerate points (reading c7)
    (2000, 2, 0, 6, "gaussian", "subset"),
])
def test_pruned_generator_equals_brute_force(n, d, m, mv, family, z):
    w = vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=0.1, nugget=0.1, seed=5, device="cpu", z=z)
    Xs, Zs = w.X / w.lengthscale, w.Z / w.lengthscale
    a = vifgen.dc_neighbors(Xs, Zs, w.family, w.sigma2, w.jitter, mv, device="cpu")
    b = vifgen.dc_neighbors_pruned(Xs, Zs, w.family, w.sigma2, w.jitter, mv, device="cpu", prefix=200, csize=64,
                                   qsize=128)
    np.testing.assert_array_equal(a, b)

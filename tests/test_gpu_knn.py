"""CUDA correlation-distance neighbour search (vif_neighbors) vs the oracle.

Neighbour sets are integers: bit-exact equality is required except where the oracle's own scores
make the choice ambiguous (two candidates with scores equal to 1e-12 relative at the m_v boundary
or inside the ranking); there every selected neighbour's oracle score must be within 1e-12 of the
oracle's choice at the same rank (the set is valid), and at most 0.5% of rows may differ."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import vifgen  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_05064_b200 as p
    p.load_library()
    return p


def knn_parity(w, mv):
    import paper_2507_05064_b200 as p
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, device=dev)
    th = p.Theta(**w.theta_dict())
    g = model.neighbors(th, mv).cpu().numpy()
    oth = oracle.Theta(**w.theta_dict())
    r, rs = oracle.dc_neighbors(w.X, w.Z, oth, mv)
    diff = np.nonzero((g != r).any(1))[0]
    assert len(diff) <= max(2, 0.005 * w.n), len(diff)
    for i in diff:
        sel = g[i][g[i] >= 0]
        assert len(sel) == (r[i] >= 0).sum() and np.all(sel < i) and len(set(sel)) == len(sel)
        gs = oracle.dc_scores(w.X, w.Z, oth, np.full(len(sel), i), sel)
        np.testing.assert_allclose(gs, rs[i][:len(sel)], rtol=1e-12, atol=1e-14)
    # the factor with the GPU neighbours equals the factor with the oracle's (same NLL to 1e-10)
    model.set_data(nbr=torch.from_numpy(g).to(dev))
    a = model.evaluate(th).nll
    model.set_data(nbr=torch.from_numpy(r).to(dev))
    b = model.evaluate(th).nll
    assert a == pytest.approx(b, rel=1e-10)
    model.close()
    return g


def test_knn_config1():
    knn_parity(vifgen.make_config(1, device="cuda"), 10)


@pytest.mark.parametrize("family", ["matern12", "matern32", "matern52", "gaussian"])
def test_knn_families_ragged(family):
    w = vifgen.make_workload(n=1000, d=2, m=37, mv=13, family=family, rho=0.15, nugget=0.1, seed=90,
                             device="cuda")
    knn_parity(w, 13)


def test_knn_m0_ard_and_large_mv():
    w = vifgen.make_workload(n=900, d=3, m=0, mv=5, family="matern52", ard=(0.5, 2.0), nugget=0.1, seed=91,
                             device="cuda", z="subset")
    knn_parity(w, 5)
    w = vifgen.make_workload(n=700, d=2, m=20, mv=45, family="matern32", rho=0.2, nugget=0.1, seed=92, device="cuda")
    knn_parity(w, 45)


def test_knn_degenerate_inducing_points_at_data():
    # config-1 style: Z is a subset of X, so those points have zero residual variance (reading c7)
    w = vifgen.make_workload(n=800, d=2, m=40, mv=10, family="matern32", rho=0.1, nugget=0.1, seed=93,
                             device="cuda", z="subset")
    knn_parity(w, 10)


def test_knn_matches_generator_config2_subset():
    w = vifgen.make_config(2, device="cuda", n=20000)
    g = knn_parity(w, 20)
    agree = (g == w.nbr).all(1).mean()
    assert agree > 0.995

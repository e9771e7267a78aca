"""CUDA gradient of the NLL (vif_grad, through the C ABI) vs the oracle gradient.

theta = (sigma_1^2, lambda_1..lambda_d, sigma^2).  Bar: per component |g - g_ref| <= 1e-8 x
max(|g_ref|, term scale), the term scale being half the sum of |d sum log D|, |d logdet M_w|,
|d quad| (the gradient at the data-generating theta is a small difference of large terms).
At n = 1M (config 3) the oracle is too slow; there the GPU gradient is checked against
Richardson-extrapolated central differences of the GPU's own NLL (a property at any size)."""
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


def vif():
    import paper_2507_05064_b200 as p
    return p


def model_of(w, world=1):
    p = vif()
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
    return p.VifModel(X, Z, nbr, y, world=world, device=dev)


def small(n, m, mv, family="matern32", seed=1, rho=0.15, nugget=0.1, d=2, ard=None, neighbors="dc"):
    return vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=nugget, seed=seed,
                                device="cuda", ard=ard, z="kmeans++" if m > 0 else "subset", neighbors=neighbors)


def check(g, r, rtol=1e-8):
    scale = np.maximum(np.abs(r.grad), 0.5 * np.abs(r.parts).sum(axis=1))
    err = np.abs(g - r.grad) / scale
    assert np.all(err <= rtol), (g, r.grad, err)


def grad_parity(w, rtol=1e-8, world=1):
    p = vif()
    model = model_of(w, world)
    terms, g = model.grad(p.Theta(**w.theta_dict()))
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    ro = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), want_BD=False)
    assert terms.nll == pytest.approx(ro.nll, rel=1e-8)
    check(g, r, rtol)
    model.close()
    return g, r


def test_grad_config1():
    grad_parity(vifgen.make_config(1, device="cuda"))


@pytest.mark.parametrize("family", ["matern12", "matern32", "matern52", "gaussian"])
@pytest.mark.parametrize("n,m,mv", [(700, 37, 13), (513, 64, 31), (300, 9, 1)])
def test_grad_shapes(family, n, m, mv):
    grad_parity(small(n, m, mv, family=family, seed=n + mv))


@pytest.mark.parametrize("world", [2, 3])
def test_grad_emulated_world(world):
    """Emulated multi-rank handle: per-rank point sums (dU formed in several row blocks) + the reduction."""
    grad_parity(small(1100, 45, 17, seed=world, d=3, ard=(0.5, 2.0)), world=world)


def test_grad_m0_vecchia():
    grad_parity(small(600, 0, 12, seed=5))


def test_grad_mv0_fitc():
    grad_parity(small(600, 40, 0, seed=6))


@pytest.mark.parametrize("n,m,mv,family", [(500, 30, 40, "matern32"), (420, 0, 33, "matern12"),
                                           (600, 45, 47, "gaussian")])
def test_grad_large_conditioning_sets(n, m, mv, family):
    """s = m_v + 1 > 32: the shared-memory state pass (m_v <= 47; config 5 has m_v = 40)."""
    grad_parity(small(n, m, mv, family=family, seed=n + mv))


def test_grad_config5_shape():
    """config 5's dimensions (d = 3, m_v = 40, exponential covariance) on a small n."""
    grad_parity(small(1200, 80, 40, family="matern12", d=3, rho=0.3, seed=45, nugget=0.01))


def test_grad_config4_shape():
    """config 4's dimensions (d = 10, m_v = 20: 12 KB of shared memory per warp in the state pass, over the
    48 KB default with the static arrays) on a small n."""
    grad_parity(small(1500, 120, 20, family="matern52", d=10, ard=(0.5, 5.0), seed=44, nugget=0.1))


def test_grad_ard_10d():
    grad_parity(small(800, 60, 15, family="matern52", d=10, ard=(0.5, 5.0), seed=7, nugget=0.1))


def test_grad_exact_case_all_predecessors():
    grad_parity(small(32, 6, 31, neighbors="all", seed=8))


def test_grad_off_theta():
    w = small(900, 30, 10, seed=9)
    th = dict(w.theta_dict())
    th["sigma2"] *= 1.6
    th["lengthscale"] = np.asarray(th["lengthscale"]) * 0.7
    th["nugget"] *= 2.2
    p = vif()
    model = model_of(w)
    _, g = model.grad(p.Theta(**th))
    r = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**th))
    check(g, r)
    assert np.all(np.abs(r.grad) > 1.0)
    model.close()


def test_grad_repeat_deterministic_and_matches_nll():
    w = small(500, 20, 8, seed=10)
    p = vif()
    model = model_of(w)
    th = p.Theta(**w.theta_dict())
    t1, g1 = model.grad(th)
    t2, g2 = model.grad(th)
    assert np.array_equal(g1, g2) and t1.nll == t2.nll
    assert model.evaluate(th).nll == t1.nll
    model.close()


@pytest.mark.slow
def test_grad_config4_recipe_m1000():
    """m = 1000 (ld = 1008: the gradient buffers, R, T, G2 and the Q / Gamma GEMMs beyond 512 columns) at the
    config-4 recipe (d = 10 ARD Matern 5/2, m_v = 20), n = 3000, all 12 partial derivatives vs the oracle."""
    grad_parity(vifgen.make_config(4, device="cuda", n=3000))


@pytest.mark.slow
def test_grad_config2_full():
    grad_parity(vifgen.make_config(2, device="cuda"))


@pytest.mark.slow
def test_grad_config3_recipe_vs_oracle():
    """The config-3 recipe (m = 500, m_v = 30, Matern 3/2 in 2-D) at n = 200k against the oracle's gradient
    (the full n = 1M is checked by finite differences below: the oracle would need ~15 min there)."""
    grad_parity(vifgen.make_config(3, device="cuda", n=200000))


@pytest.mark.slow
def test_grad_config3_vs_gpu_finite_differences():
    """n = 1M: analytic GPU gradient vs Richardson central differences of the GPU NLL."""
    w = vifgen.make_config(3, device="cuda")
    p = vif()
    model = model_of(w)
    base = w.theta_dict()
    v0 = np.concatenate([[base["sigma2"]], np.asarray(base["lengthscale"], float), [base["nugget"]]])
    d = w.d

    def nll(v):
        th = p.Theta(base["family"], float(v[0]), np.array(v[1:1 + d]), float(v[1 + d]), base["jitter"])
        return model.evaluate(th).nll

    terms, g = model.grad(p.Theta(**base))
    for k in range(len(v0)):
        h = 1e-4 * v0[k]
        e = np.eye(len(v0))[k]
        cen = lambda hh: (nll(v0 + hh * e) - nll(v0 - hh * e)) / (2 * hh)
        fd = (4 * cen(h / 2) - cen(h)) / 3
        # term scale of the NLL (|NLL| << its terms at the data-generating theta)
        scale = max(abs(g[k]), 1e-7 * (abs(terms.logdet_D) + abs(terms.logdet_M) + abs(terms.quad)) / v0[k])
        assert abs(g[k] - fd) <= 1e-6 * scale + 1e-6 * abs(fd), (k, g[k], fd)
    model.close()


def test_lbfgs_fit_recovers_theta():
    """The gradient drives a quasi-Newton fit: from a perturbed start, L-BFGS on the log-parameters
    converges (small projected gradient), lowers the NLL, and lands near the data-generating theta."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples"))
    from fit_lbfgs import fit
    w = vifgen.make_workload(n=20000, d=2, m=60, mv=15, family="matern32", rho=0.05, nugget=0.05, seed=12,
                             device="cuda")
    model = model_of(w)
    truth = np.array([w.sigma2, w.lengthscale[0], w.nugget])
    r, evals, secs = fit(model, w, truth * np.array([2.0, 0.5, 3.0]))
    est = np.exp(r.x)
    assert r.fun < evals[0][0] - 10.0
    assert np.linalg.norm(r.jac) < 1e-2 * max(1.0, abs(r.fun)) ** 0.5
    assert np.all(np.abs(np.log(est / truth)) < np.log(1.6)), (est, truth)
    model.close()

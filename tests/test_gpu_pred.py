"""CUDA predictive means (vif_predict, through the C ABI) vs the oracle (Prop. 1; reading p1).

Bar: mu to 1e-9 relative with an absolute floor 1e-10 max|y|; var and D_p relative 1e-9; B_p = -A_p per row
max|dB| <= 1e-9 max(max|B_p|, 1e-3) (the training B bar)."""
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


def small(n, m, mv, family="matern32", seed=1, rho=0.15, nugget=0.1, d=2, ard=None):
    return vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=nugget, seed=seed,
                                device="cuda", ard=ard, z="kmeans++" if m > 0 else "subset")


def pred_parity(w, npred=300, x="uniform", world=1):
    import paper_2507_05064_b200 as p
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, world=world, device=dev)
    Xp, nbrp = vifgen.make_prediction(w, npred, x=x, device="cuda")
    mu, var, Dp, Bp = model.predict(p.Theta(**w.theta_dict()), Xp, nbrp, want_var=True, want_D=True, want_B=True)
    mu, var, Dp, Bp = mu.cpu().numpy(), var.cpu().numpy(), Dp.cpu().numpy(), Bp.cpu().numpy()
    rmu, rvar, rD, rB = oracle.predict(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), Xp, nbrp)
    np.testing.assert_allclose(mu, rmu, rtol=1e-9, atol=1e-10 * np.abs(w.y).max())
    np.testing.assert_allclose(var, rvar, rtol=1e-9)
    np.testing.assert_allclose(Dp, rD, rtol=1e-9)
    if w.mv > 0:
        err = np.abs(Bp - rB).max(1) / np.maximum(np.abs(rB).max(1), 1e-3)
        assert err.max() <= 1e-9
    model.close()


def test_pred_config1():
    pred_parity(vifgen.make_config(1, device="cuda"), npred=1000)


@pytest.mark.parametrize("family", ["matern12", "matern32", "matern52", "gaussian"])
@pytest.mark.parametrize("n,m,mv", [(700, 37, 13), (513, 64, 31), (400, 9, 40)])
def test_pred_shapes(family, n, m, mv):
    pred_parity(small(n, m, mv, family=family, seed=n + mv), npred=257)


@pytest.mark.parametrize("world", [2, 3])
def test_pred_emulated_world(world):
    """An emulated multi-rank handle (one process) reduces the Gram over its ranks and predicts all points."""
    pred_parity(small(900, 40, 15, seed=world), npred=301, world=world)


def test_pred_m0_and_mv0():
    pred_parity(small(600, 0, 12, seed=5))
    pred_parity(small(600, 40, 0, seed=6))


def test_pred_ard_10d():
    pred_parity(small(800, 60, 15, family="matern52", d=10, ard=(0.5, 5.0), seed=7), x="normal")


def test_pred_single_point_and_repeat():
    import paper_2507_05064_b200 as p
    w = small(400, 20, 8, seed=12)
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, device=dev)
    Xp, nbrp = vifgen.make_prediction(w, 1, device="cuda")
    th = p.Theta(**w.theta_dict())
    a = model.predict(th, Xp, nbrp).cpu().numpy()
    b = model.predict(th, Xp, nbrp).cpu().numpy()
    assert np.array_equal(a, b)
    rmu, _, _, _ = oracle.predict(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), Xp, nbrp)
    np.testing.assert_allclose(a, rmu, rtol=1e-9, atol=1e-10)
    # the training NLL is unchanged by a prediction call
    t1 = model.evaluate(th)
    model.predict(th, Xp, nbrp)
    assert model.evaluate(th).nll == t1.nll
    model.close()


@pytest.mark.slow
def test_pred_config3_vs_oracle():
    pred_parity(vifgen.make_config(3, device="cuda"), npred=2000)


@pytest.mark.parametrize("cid,n", [(4, 8000), (5, 6000)])
def test_pred_large_m_config_recipes(cid, n):
    """m = 1000 (config 4: 10-D prediction inputs, N(0, I)) and m = 1500 with m_v = 40 (config 5): the prediction
    features, rows and the L_M^{-T} product beyond 512 columns."""
    pred_parity(vifgen.make_config(cid, device="cuda", n=n), npred=400, x="normal" if cid == 4 else "uniform")

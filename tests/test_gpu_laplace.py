"""GPU parity of the VIF-Laplace iterative path against oracle/laplace.py.

Operators (Sigma_dagger, W^{-1} + Sigma_dagger, B^{-1}, B^{-T}, the FITC solve, Sigma_dagger^{-1} and
W + Sigma_dagger^{-1} of pcls1): the triangular solves to
a backward error of 1e-13 against the GPU's own latent B (|B x - v| / (|B| |x|)), every operator to a forward
error of 1e-8 relative to the column scale (B and D themselves agree to 1e-9, north_star; the solves
carry that through dependency chains, observed up to ~2e-9 on ill-conditioned residual factors); the mode, -log p and the quadratic term with both sides' CG and Newton tolerances at
1e-12 (bound: the mode is unique and both iterations stop within ~1e-11 of it); the SLQ log-determinant
with the same probe draws and CG tolerance 1e-12 (e1^T log(T) e1 is a Gauss quadrature whose error
after convergence is O(||r||^2): the two sides agree to ~1e-10 relative).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import laplace as la
import vifgen

pytestmark = pytest.mark.gpu


def vif():
    import paper_2507_05064_b200 as p
    return p


def work(n, m, mv, family="matern32", d=2, rho=0.2, seed=1, neighbors="dc", lengthscale=None):
    return vifgen.make_laplace_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, seed=seed, device="cuda",
                                        neighbors=neighbors, z="kmeans++" if m > 0 else "subset",
                                        lengthscale=lengthscale)


def model_of(w, theta, nprobe=0, max_cg=1000):
    p = vif()
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, device=dev)
    model.la_prepare(theta, nprobe=nprobe, max_cg=max_cg)
    return model


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    scale = np.maximum(np.abs(b).max(axis=0), 1e-300)
    return float((np.abs(a - b).max(axis=0) / scale).max())


@pytest.mark.parametrize("n,m,mv,ncol", [(700, 37, 13, 1), (700, 37, 13, 5), (513, 64, 31, 8), (400, 0, 12, 3),
                                         (300, 9, 0, 2), (257, 20, 40, 1), (700, 37, 13, 20), (450, 70, 12, 64),
                                         (700, 37, 9, 33)])
def test_operators(n, m, mv, ncol):
    p = vif()
    w = work(n, m, mv, seed=n + mv)
    th = p.Theta(**w.theta_dict())
    model = model_of(w, th, nprobe=ncol)
    lat = la.latent_factor(w.X, w.Z, w.nbr, oracle.Theta(**w.theta_dict()))
    rng = np.random.default_rng(ncol)
    V = rng.standard_normal((n, ncol)) if ncol > 1 else rng.standard_normal(n)
    W = la.hess_w(rng.normal(0, 1.5, n))
    winv = 1.0 / W
    V2 = V.reshape(n, -1)
    sinv = np.stack([lat.sigma_dagger_inv(V2[:, k]) for k in range(V2.shape[1])], axis=1).reshape(V.shape)
    refs = {"btinv": lat.btinv(V), "binv": lat.binv(V), "sigma": lat.sigma_dagger(V),
            "A": (V / W[:, None] if V.ndim == 2 else V / W) + lat.sigma_dagger(V),
            "fitc_solve": la.fitc(lat, W).solve(V),
            "sigma_inv": sinv, "A1": (V * W[:, None] if V.ndim == 2 else V * W) + sinv}
    errs, gots = {}, {}
    for op, ref in refs.items():
        got = gots[op] = model.la_apply(op, V, winv=winv if op in ("A", "A1", "fitc_solve") else None).cpu().numpy()
        errs[op] = rel_err(got, ref)
    assert max(errs.values()) < 1e-8, errs
    # backward error of the triangular solves against the GPU's own latent B (vif_factor at nugget 0;
    # this invalidates the Laplace workspace, so it comes last): rounding level
    th0 = p.Theta(**{**w.theta_dict(), "nugget": 0.0})
    Bg = torch.zeros((n, max(mv, 1)), dtype=torch.float64, device="cuda")
    model.factor(th0, Bg if mv > 0 else None, torch.empty(n, dtype=torch.float64, device="cuda"))
    Bg = Bg.cpu().numpy()
    import scipy.sparse as sp
    rows = np.repeat(np.arange(n), mv)
    ok = w.nbr.reshape(-1) >= 0 if mv > 0 else np.zeros(0, bool)
    Bm = sp.csr_matrix((np.concatenate([np.ones(n), Bg[:, :mv].reshape(-1)[ok]]),
                        (np.concatenate([np.arange(n), rows[ok]]), np.concatenate([np.arange(n), w.nbr.reshape(-1)[ok]]))),
                       shape=(n, n))
    for op, M in (("binv", Bm), ("btinv", Bm.T.tocsr())):
        G = gots[op].reshape(n, -1)
        res = np.abs(M @ G - V.reshape(n, -1)).max(axis=0) / (abs(M) @ np.abs(G)).max(axis=0)
        assert res.max() < 1e-13, (op, res)
    model.close()


def mode_parity(w, nprobe=0, tol=1e-12, mode_rtol=1e-8, nll_rtol=1e-9):
    p = vif()
    th = p.Theta(**w.theta_dict())
    model = model_of(w, th, nprobe=nprobe)
    eps1, eps2 = vifgen.make_probes(w.n, w.Z.shape[0], nprobe) if nprobe else (None, None)
    opts = p.LaOpts(max_newton=60, newton_tol=tol, max_cg=1000, cg_tol=tol, nprobe=nprobe, slq_tol=tol)
    t, b = model.la_nll(w.y, opts, eps1 if nprobe and w.Z.shape[0] else None, eps2)
    b = b.cpu().numpy()
    r = la.vifla_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), eps1=eps1, eps2=eps2, newton_tol=tol,
                     max_newton=60, cg_tol=tol, max_cg=1000, slq_tol=tol)
    assert np.abs(b - r.b).max() <= mode_rtol * np.abs(r.b).max()
    assert t.neg_loglik == pytest.approx(r.neg_loglik, rel=nll_rtol)
    assert t.quad == pytest.approx(r.quad, rel=mode_rtol)
    if nprobe:
        assert t.logdet_W == pytest.approx(r.logdet_parts["logdet_W"], rel=1e-10)
        assert t.logdet_P == pytest.approx(r.logdet_parts["logdet_P"], rel=1e-10)
        assert t.logdet == pytest.approx(r.logdet, rel=1e-9)
        assert t.nll == pytest.approx(r.nll, rel=1e-9)
    model.close()
    return t, r


@pytest.mark.parametrize("family", ["matern12", "matern32", "matern52", "gaussian"])
def test_mode_families(family):
    mode_parity(work(600, 25, 10, family=family, seed=3))


@pytest.mark.parametrize("n,m,mv", [(800, 40, 15), (500, 0, 12), (400, 16, 31), (300, 10, 40)])
def test_mode_shapes(n, m, mv):
    mode_parity(work(n, m, mv, seed=n))


@pytest.mark.parametrize("nprobe", [1, 7, 32])
def test_slq_logdet(nprobe):
    mode_parity(work(700, 30, 12, seed=11), nprobe=nprobe)


def test_paper_workload_small():
    """The recipe of the paper's Laplace experiments (d = 5, ARD Gaussian covariance, binary
    responses) at n = 2000, m = 50, m_v = 15."""
    w = vifgen.make_laplace_workload(n=2000, m=50, mv=15, seed=21, device="cuda")
    mode_parity(w, nprobe=8)


def test_exact_case_matches_dense_laplace():
    """All predecessors: the GPU mode and L^LA with the oracle's dense log-det equal the textbook
    Laplace approximation on the exact covariance (la6 pins the oracle to it)."""
    w = work(40, 5, 39, neighbors="all", seed=10, rho=0.3)
    t, r = mode_parity(w)
    lat = la.latent_factor(w.X, w.Z, w.nbr, oracle.Theta(**w.theta_dict()))
    assert np.isfinite(la.exact_logdet(lat, la.hess_w(r.b)))


def test_state_checks():
    p = vif()
    w = work(300, 10, 8, seed=5)
    th = p.Theta(**w.theta_dict())
    model = model_of(w, th)
    model.evaluate(th)  # a new factor invalidates the prepared Laplace workspace
    with pytest.raises(p.VifError):
        model.la_apply("sigma", np.ones(300))
    model.close()


@pytest.mark.slow
def test_bench_size_sampled():
    """bench.py's Laplace workload (n = 100k, d = 5 ARD Gaussian, m = 200, m_v = 30) in its launch
    configuration: sampled rows against the oracle, and properties that hold at any size.
      - B^{-1} v and B^{-T} u: the oracle's own B rows (oracle.rows, nugget 0, recomputed from scratch)
        satisfy (B x)_i = v_i on 300 sampled rows and (B^T y)_j = u_j on 40 sampled columns (all their
        children rows) to 1e-9 relative to the row scale;
      - the mode is stationary: b~ = Sigma_dagger (y - pi(b~)) (Sigma_dagger applied by the GPU, whose
        operator parity is pinned above) to the CG tolerance;
      - L^VIFLA is finite and equals its three terms."""
    p = vif()
    w = vifgen.make_laplace_workload(n=100000, m=200, mv=30, device="cuda")
    th = p.Theta(**w.theta_dict())
    model = model_of(w, th, nprobe=50)
    n, mv = w.n, w.mv
    rng = np.random.default_rng(5)
    v = rng.standard_normal(n)
    x = model.la_apply("binv", v).cpu().numpy()
    yv = model.la_apply("btinv", v).cpu().numpy()
    th0 = oracle.Theta(**{**w.theta_dict(), "nugget": 0.0})
    ri = rng.choice(n, 300, replace=False)
    _, Br, _ = oracle.rows(w.X, w.Z, w.nbr, th0, ri)
    nb = w.nbr[ri]
    Bx = x[ri] + np.sum(np.where(nb >= 0, Br * x[np.maximum(nb, 0)], 0.0), axis=1)
    scale = np.abs(x[ri]) + np.sum(np.abs(np.where(nb >= 0, Br * x[np.maximum(nb, 0)], 0.0)), axis=1)
    assert np.max(np.abs(Bx - v[ri]) / scale) < 1e-9
    cols = rng.choice(n, 40, replace=False)
    for j in cols:
        ch, pos = np.nonzero(w.nbr == j)
        _, Bc, _ = oracle.rows(w.X, w.Z, w.nbr, th0, ch) if len(ch) else (None, np.zeros((0, mv)), None)
        terms = Bc[np.arange(len(ch)), pos] * yv[ch] if len(ch) else np.zeros(0)
        res = yv[j] + terms.sum() - v[j]
        assert abs(res) <= 1e-9 * (abs(yv[j]) + np.abs(terms).sum())
    eps1, eps2 = vifgen.make_probes(n, 200, 50)
    opts = p.LaOpts(max_newton=50, newton_tol=1e-10, max_cg=1000, cg_tol=1e-10, nprobe=50, slq_tol=1e-6)
    t, b = model.la_nll(w.y, opts, eps1, eps2)
    b = b.cpu().numpy()
    g = w.y - 1.0 / (1.0 + np.exp(-b))
    sg = model.la_apply("sigma", g).cpu().numpy()
    assert np.max(np.abs(sg - b)) <= 1e-6 * np.abs(b).max()
    assert np.isfinite(t.nll) and t.nll == pytest.approx(t.neg_loglik + 0.5 * t.quad + 0.5 * t.logdet, rel=1e-12)
    model.close()


def test_sigma_inv_inverts_sigma():
    """Sigma_dagger^{-1} (Woodbury, sparse products) inverts Sigma_dagger (triangular solves) on the GPU."""
    p = vif()
    w = work(900, 30, 12, seed=17)
    model = model_of(w, p.Theta(**w.theta_dict()), nprobe=4)
    V = np.random.default_rng(3).standard_normal((900, 4))
    back = model.la_apply("sigma_inv", model.la_apply("sigma", V)).cpu().numpy()
    assert rel_err(back, V) < 1e-8
    model.close()


def test_truncated_cg_iteration_exact():
    """CG capped at 6 iterations (Newton solves and probe solves): both sides stop at the same iteration,
    so the iterates, the Lanczos matrices and L^VIFLA still agree (tests the per-iteration arithmetic,
    not only the converged answer)."""
    p = vif()
    w = work(500, 20, 10, seed=19)
    th = p.Theta(**w.theta_dict())
    model = model_of(w, th, nprobe=5, max_cg=6)
    eps1, eps2 = vifgen.make_probes(w.n, 20, 5)
    opts = p.LaOpts(max_newton=8, newton_tol=1e-14, max_cg=6, cg_tol=1e-14, nprobe=5, slq_tol=1e-14)
    t, b = model.la_nll(w.y, opts, eps1, eps2)
    r = la.vifla_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), eps1=eps1, eps2=eps2, newton_tol=1e-14,
                     max_newton=8, cg_tol=1e-14, max_cg=6, slq_tol=1e-14)
    assert t.newton_iters == r.newton_iters and t.slq_iters_max == max(r.slq_iters) == 6
    np.testing.assert_allclose(b.cpu().numpy(), r.b, rtol=1e-9, atol=1e-10 * np.abs(r.b).max())
    assert t.logdet == pytest.approx(r.logdet, rel=1e-9)
    assert t.nll == pytest.approx(r.nll, rel=1e-9)
    model.close()


def test_tiny_problem_no_neighbours_no_inducing():
    """n = 40 with m = 0 and m_v = 0 (B = I, Sigma_dagger = D diagonal) and n = 7 < 32 rows."""
    for n, m, mv in ((40, 0, 0), (7, 3, 4)):
        mode_parity(work(n, m, mv, seed=n), nprobe=3)

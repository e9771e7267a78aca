"""CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.  Needs a B200."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import vifgen  # noqa: E402
from parity import check_B, check_D, check_terms, check_U  # noqa: E402


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


def run_gpu(w, world=1, emulate=True, want_U=False, host_inputs=False):
    p = vif()
    dev = torch.device("cuda")
    if host_inputs:
        X = torch.from_numpy(w.X).pin_memory()
        Z = torch.from_numpy(w.Z.reshape(-1, w.d)).pin_memory()
        nbr = torch.from_numpy(w.nbr).pin_memory()
        y = torch.from_numpy(w.y).pin_memory()
    else:
        X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                        for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, world=world, device=dev)
    B = torch.zeros((w.n, w.mv), dtype=torch.float64, device=dev)
    D = torch.zeros(w.n, dtype=torch.float64, device=dev)
    th = p.Theta(**w.theta_dict())
    t = model.evaluate(th, B, D)
    U = model.U().cpu().numpy() if want_U else None
    out = (t, B.cpu().numpy(), D.cpu().numpy(), U, model.launch_count())
    model.close()
    return out


def oracle_run(w, want_U=False):
    return oracle.factor_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), want_U=want_U)


def assert_parity(w, world=1, want_U=True, host_inputs=False):
    t, B, D, U, nl = run_gpu(w, world=world, want_U=want_U, host_inputs=host_inputs)
    r = oracle_run(w, want_U=want_U)
    check_terms(t, r.nll, r.logdet_D, r.logdet_M, r.quad)
    check_D(D, r.D)
    check_B(B, r.B)
    if want_U and w.m > 0:
        check_U(U, r.U)
    assert nl > 0
    return t, r


def small(n, m, mv, family="matern32", d=2, seed=1, rho=0.15, nugget=0.1, ard=None, x="uniform", neighbors="dc"):
    return vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=nugget, seed=seed,
                                device="cuda", ard=ard, x=x, z="kmeans++" if m > 0 else "subset",
                                neighbors=neighbors)


def test_config1_full_parity():
    w = vifgen.make_config(1, device="cuda")
    assert_parity(w)


@pytest.mark.parametrize("n,m,mv,family,d", [
    (3001, 37, 7, "matern32", 2),      # odd m, ragged n, RB = 1
    (2500, 64, 31, "matern52", 3),     # RB = 4 (s = 32), m multiple of 64
    (1777, 130, 20, "matern12", 2),    # RB = 3, several GEMM col tiles + ragged
    (1200, 16, 40, "gaussian", 4),     # RB = 6 (s = 41)
    (1100, 25, 36, "matern12", 3),     # RB = 5 (s = 37)
    (900, 9, 47, "matern32", 1),       # max m_v, d = 1
    (2049, 200, 15, "matern52", 5),    # several 64-col SYRK tiles
])
def test_shapes_parity(n, m, mv, family, d):
    w = small(n, m, mv, family=family, d=d, seed=n + m + mv, rho=0.3 if d > 2 else 0.15)
    assert_parity(w)


def test_m0_classical_vecchia():
    w = small(1500, 0, 12, seed=5)
    t, r = assert_parity(w, want_U=False)
    assert t.logdet_M == 0.0


def test_mv0_fitc():
    w = small(1200, 20, 0, seed=6)
    assert_parity(w)


def test_ard_10d_config4_recipe_small():
    w = vifgen.make_workload(n=3000, d=10, m=100, mv=20, family="matern52", ard=(0.5, 5.0), nugget=0.1,
                             x="normal", seed=vifgen.SEED_BASE + 4, device="cuda")
    assert_parity(w)


def test_exact_case_all_predecessors_matches_dense():
    from refs import dense_nll, sk_cov
    n = 40
    w = small(n, 6, n - 1, seed=7, neighbors="all")
    t, B, D, U, _ = run_gpu(w)
    S = sk_cov(w.family, w.sigma2, w.lengthscale, w.X) + w.nugget * np.eye(n)
    assert t.nll == pytest.approx(dense_nll(S, w.y), rel=1e-9)


def test_n1_scalar():
    p = vif()
    for m in (0, 3):
        rng = np.random.default_rng(3)
        w = vifgen.Workload("n1", rng.random((1, 2)), rng.random((m, 2)), np.zeros((1, 2), np.int32) - 1,
                            np.array([0.4]), "matern32", 1.2, np.array([0.3, 0.3]), 0.2, 1e-10)
        assert_parity(w, want_U=m > 0)


@pytest.mark.parametrize("world,d", [(2, 2), (3, 2), (4, 2), (3, 6)])
def test_emulated_sharding_matches_single(world, d):
    """d = 6 takes the neighbour-driven processing order (d > 3) on every emulated rank."""
    w = small(5003, 48, 10, seed=11, d=d, ard=(0.3, 3.0) if d > 3 else None)
    t1, B1, D1, _, _ = run_gpu(w, world=1)
    tg, Bg, Dg, _, _ = run_gpu(w, world=world)
    assert tg.nll == pytest.approx(t1.nll, rel=1e-12)
    assert tg.quad == pytest.approx(t1.quad, rel=1e-11)
    np.testing.assert_array_equal(Dg, D1)   # rows are computed identically, only the sums change order
    np.testing.assert_array_equal(Bg, B1)


def test_host_pinned_inputs_same_result():
    w = small(2000, 32, 9, seed=12)
    t_dev, *_ = run_gpu(w)
    t_host, *_ = run_gpu(w, host_inputs=True)
    assert t_host.nll == t_dev.nll


def test_repeat_evaluations_deterministic_and_theta_change():
    p = vif()
    w = small(4000, 40, 12, seed=13)
    dev = torch.device("cuda")
    model = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
    th = p.Theta(**w.theta_dict())
    a = model.evaluate(th)
    b = model.evaluate(th)
    assert a.nll == b.nll
    th2 = w.theta_dict()
    th2["lengthscale"] = th2["lengthscale"] * 1.1
    c = model.evaluate(p.Theta(**th2))
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**th2))
    check_terms(c, r.nll, r.logdet_D, r.logdet_M, r.quad)
    model.close()


# ---------------- error behaviour ----------------
def test_invalid_neighbors_rejected():
    p = vif()
    w = small(300, 8, 5, seed=14)
    nbr = w.nbr.copy()
    nbr[100, 0] = 150   # not a predecessor
    dev = torch.device("cuda")
    with pytest.raises(p.VifError) as e:
        p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, nbr, w.y)))
    assert e.value.status == 1 and "row 100" in e.value.msg


@pytest.mark.parametrize("width", [2, 35])  # register kernel / blocked shared-memory kernel (m_v > 31)
def test_not_pd_reports_row(width):
    p = vif()
    X = np.array([[0.1, 0.1], [0.5, 0.5], [0.5, 0.5], [0.7, 0.2]])
    nbr = np.full((4, width), -1, np.int32)
    nbr[:, :2] = [[-1, -1], [0, -1], [1, 0], [2, 1]]
    dev = torch.device("cuda")
    model = p.VifModel(torch.from_numpy(X).to(dev), torch.zeros((0, 2), dtype=torch.float64, device=dev),
                       torch.from_numpy(nbr).to(dev), torch.zeros(4, dtype=torch.float64, device=dev))
    with pytest.raises(p.VifError) as e:
        model.evaluate(p.Theta("matern32", 1.0, [0.3, 0.3], 0.0, 0.0))
    assert e.value.status == 2 and e.value.bad_row in (2, 3)


def test_state_and_theta_errors():
    p = vif()
    w = small(200, 8, 4, seed=15)
    dev = torch.device("cuda")
    model = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
    with pytest.raises(p.VifError) as e:
        model.nll()
    assert e.value.status == 6
    with pytest.raises(p.VifError) as e:
        model.factor(p.Theta("matern32", -1.0, [0.1, 0.1], 0.1, 0.0))
    assert e.value.status == 1
    with pytest.raises(p.VifError) as e:
        model.factor(p.Theta("matern32", 1.0, [0.1], 0.1, 0.0))
    assert e.value.status == 1
    model.close()


# ---------------- larger configs (BASELINE.json configs[1], configs[2]) ----------------
def test_config2_full_parity():
    w = vifgen.make_config(2, device="cuda")
    assert_parity(w, want_U=False)


@pytest.mark.slow
def test_config3_full_nll_and_sampled_rows():
    """n = 1M, m = 500, m_v = 30 in the bench's launch configuration: full oracle NLL + 2000 sampled
    rows of U, B, D recomputed one by one by the oracle; invariants at every row."""
    p = vif()
    w = vifgen.make_config(3, device="cuda")
    t, B, D, U, _ = run_gpu(w, want_U=True)
    rows = np.random.default_rng(0).choice(w.n, 2000, replace=False)
    rows = np.concatenate([rows, [0, 1, 29, 30, 31, w.n - 1]])
    Ur, Br, Dr = oracle.rows(w.X, w.Z, w.nbr, oracle.Theta(**w.theta_dict()), rows, want_U=True)
    check_D(D[rows], Dr)
    check_B(B[rows], Br)
    rel = np.linalg.norm(U[rows] - Ur, axis=1) / np.linalg.norm(Ur, axis=1)
    assert rel.max() <= 1e-11
    # invariants at all rows (p6): sigma^2 <= D_i <= C_ii
    Cii = w.sigma2 + w.nugget - (U * U).sum(1)
    assert np.all(D >= w.nugget * (1 - 1e-12)) and np.all(D <= Cii * (1 + 1e-10))
    assert t.logdet_M >= 0 and t.quad >= 0
    r = oracle_run(w)
    check_terms(t, r.nll, r.logdet_D, r.logdet_M, r.quad)
    # the full oracle factor is at hand: every one of the 1M rows of B and D, not only the sample
    check_D(D, r.D)
    check_B(B, r.B)


@pytest.mark.parametrize("cid,n", [(4, 12000), (5, 9000)])
def test_large_m_config_recipes_parity(cid, n):
    """BASELINE configs 4 (d = 10, ARD Matern 5/2, m = 1000, m_v = 20) and 5 (d = 3, Matern 1/2, m = 1500,
    m_v = 40: the s > 32 kernel) at n of ~10k with their own recipes: the W pass beyond 512 columns (ld = 1008 /
    1512), K1 and the SYRK at ld > 512, chol_inv beyond 16 tiles -- NLL, every B and D row and U against the
    oracle."""
    w = vifgen.make_config(cid, device="cuda", n=n)
    assert w.m == (1000 if cid == 4 else 1500)
    assert_parity(w, want_U=True)


def test_large_m_emulated_sharding():
    """m = 1000 on three emulated ranks (per-rank SYRK partials at ld = 1008, rank-ordered reduction)."""
    w = vifgen.make_config(4, device="cuda", n=6000)
    assert_parity(w, world=3, want_U=False)


def test_rounds_schedule_same_result():
    """The optional single-GPU round schedule (VIF_ROUNDS, three streams) gives the serial result:
    B and D bit-identical, NLL to 1e-12 and the gradient to 1e-10 (only the SYRK summation order
    differs).  The round schedule keeps the FP64 DMMA K1 (kx_eval + gemm_tn), so both runs use it
    (VIF_UFEAT_FP64=1) for the bit-identical comparison of B and D.  The knobs are read
    once per process, hence the subprocess."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, %r)
import __graft_entry__; __graft_entry__.build()
import paper_2507_05064_b200 as p, vifgen
w = vifgen.make_workload(n=9000, d=2, m=40, mv=12, seed=77, device="cuda")
dev = torch.device("cuda")
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
B = torch.zeros((w.n, w.mv), dtype=torch.float64, device=dev); D = torch.zeros(w.n, dtype=torch.float64, device=dev)
t = m.evaluate(p.Theta(**w.theta_dict()), B, D)
_, g = m.grad(p.Theta(**w.theta_dict()))  # the factor inside vif_grad writes the gradient state per round
np.save(sys.argv[1], np.concatenate([B.cpu().numpy().ravel(), D.cpu().numpy(), [t.nll], g]))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for R in ("1", "4"):
        path = f"/tmp/vif_rounds_{R}.npy"
        env = dict(os.environ, VIF_ROUNDS=R, VIF_UFEAT_FP64="1")
        subprocess.run([sys.executable, "-c", code, path], env=env, check=True)
        outs.append(np.load(path))
    a, b = outs
    k = a.size - 4  # B, D | NLL | gradient (sigma_1^2, lambda_1, lambda_2, sigma^2)
    assert np.array_equal(a[:k - 1], b[:k - 1])
    assert b[k - 1] == pytest.approx(a[k - 1], rel=1e-12)
    np.testing.assert_allclose(b[k:], a[k:], rtol=1e-10)


def test_stage_data_pipelined_matches_set_data():
    """vif_stage_data (second input slot, copy stream) gives exactly the results of vif_set_data, in the
    pipelined order factor(k) -> stage(k+1) -> nll(k), with pinned-host inputs, and across a switch
    between two different data sets (and back to set_data)."""
    p = vif()
    dev = torch.device("cuda")
    wa = small(3000, 40, 12, seed=101)
    wb = small(3000, 40, 12, seed=102)

    def pinned(w):
        return tuple(torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                     for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
    ha, hb = pinned(wa), pinned(wb)
    th = p.Theta(**wa.theta_dict())
    ref = []
    for h in (ha, hb):
        m = p.VifModel(*(t.to(dev) for t in h), device=dev)
        ref.append(m.evaluate(th).nll)
        m.close()
    model = p.VifModel(*(t.to(dev) for t in ha), device=dev)
    seq = [ha, hb, hb, ha, hb, ha]
    model.stage_data(*seq[0])
    got = []
    for k in range(len(seq)):
        model.factor(th)
        if k + 1 < len(seq):
            model.stage_data(*seq[k + 1])
        got.append(model.nll().nll)
    want = [ref[0] if s is ha else ref[1] for s in seq]
    assert got == want
    model.set_data(*ha)
    assert model.evaluate(th).nll == ref[0]
    model.close()


@pytest.mark.parametrize("world", [1, 3])
def test_owned_rows_map(world):
    """vif_owned_rows describes the chunk-cyclic map: for a single-rank handle the chunks
    tile [0, n) and agree with vif_partition / owned_rows; an emulated handle owns everything."""
    import paper_2507_05064_b200 as p
    w = small(1001, 8, 5, seed=13)
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, world=world, device=dev)
    first, chunk, stride, nchunks = p.vif_owned_rows(model.handle)
    rows = np.concatenate([np.arange(c * chunk, min((c + 1) * chunk, w.n)) for c in range(first, nchunks, stride)])
    np.testing.assert_array_equal(rows, np.arange(w.n))
    if world == 1:
        np.testing.assert_array_equal(np.sort(model.owned_rows()), rows)
    model.close()


_NCCL1 = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2507_05064_b200 as p
import vifgen
w = vifgen.make_workload(n=3001, d=2, m=24, mv={mv}, family="matern32", rho=0.15, nugget=0.1, seed=31, device="cuda")
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
nid = p.vif_nccl_unique_id() if {use_nccl} else None
model = p.VifModel(X, Z, nbr, y, world=1, nccl_id=nid, device=dev)
th = p.Theta(**w.theta_dict())
D = torch.zeros(w.n, dtype=torch.float64, device=dev)
t = model.evaluate(th, None, D)
_, g = model.grad(th)
print(json.dumps(dict(nll=t.nll, D=D.cpu().numpy().tolist()[:50], g=list(map(float, g)), rounds=model.rounds)))
"""


@pytest.mark.parametrize("mv", [9, 35])
def test_nccl_single_rank_schedule(mv):
    """The multi-GPU schedule (8 rounds, per-round NCCL all-gather, NCCL all-reduce of the Gram and of
    the gradient sums) on a one-rank communicator (VIF_NCCL_SINGLE=1): exercises the NCCL plumbing on one
    GPU (no ranks waiting on each other) and must reproduce the single-GPU result (the register kernel at
    m_v = 9, the shared-memory kernel at m_v = 35)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for use in (False, True):
        env = dict(os.environ, VIF_NCCL_SINGLE="1" if use else "0")
        r = subprocess.run([sys.executable, "-c", _NCCL1.format(root=root, use_nccl=use, mv=mv)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    a, b = outs
    assert b["rounds"] == 8 and a["rounds"] >= 1
    assert b["nll"] == pytest.approx(a["nll"], rel=1e-12)
    np.testing.assert_array_equal(np.array(b["D"]), np.array(a["D"]))
    np.testing.assert_allclose(b["g"], a["g"], rtol=1e-11)

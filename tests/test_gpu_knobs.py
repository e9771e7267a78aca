"""Every environment knob of libvif.so that selects another kernel variant, launch shape or ordering is run
against the CPU oracle (the knobs are read once per process, so each setting runs in its own python process).

Knobs covered here (the engine switches VIF_*_FP64, VIF_KNN_*, VIF_ROUNDS, VIF_NCCL_* have their own tests in
test_gpu_gram.py, test_gpu_knn.py, test_gpu_parity.py and test_gpu_robust.py):
  VIF_KX_GENERIC=1         K1a kernel evaluation with runtime-d loops (A1)
  VIF_VECCHIA_GENERIC_D=1  vecchia rows with runtime-d loops at d = 2 (A3-A5, T1 steps 3-5)
  VIF_GRAD_RORDER=0        gradient R rows visited in index order instead of the Morton order
  VIF_GR_BLOCKS=37         gradient R kernel on a small grid
  VIF_ORDER_ND=0           processing order from the first three coordinates for d > 3
  VIF_ORDER_K=2            n-D Morton code over two dimensions only
  VIF_KNN_EW=4             int8 neighbour search with 4 epilogue warps and the 3-stage ring
  VIF_GRAD_STATE=1         gradient state pass recomputes L, A_i, D_i instead of taking them from the factor
The order and grid knobs change only the order in which rows are visited, so the result must stay within the
oracle tolerances of tests/parity.py (B, D elementwise, NLL terms, gradient 1e-8, neighbour sets equal up to
exact ties)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import vifgen  # noqa: E402
from parity import check_B, check_D  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKLOADS = {
    # d = 2: the compile-time-d specialisations are the default path
    "d2": dict(n=2500, d=2, m=60, mv=15, family="matern32", rho=0.15, nugget=0.1, seed=41),
    # d = 5 ARD: the n-D processing order is the default path
    "d5": dict(n=2100, d=5, m=40, mv=12, family="matern52", rho=None, lengthscale=(0.3, 0.5, 0.8, 1.2, 2.0), nugget=0.05,
               seed=43),
}

CODE = r"""
import sys, json
import numpy as np, torch
sys.path.insert(0, %r)
import __graft_entry__; __graft_entry__.build()
import paper_2507_05064_b200 as p, vifgen
kw = json.loads(sys.argv[1])
if kw.get("lengthscale") is not None: kw["lengthscale"] = tuple(kw["lengthscale"])
w = vifgen.make_workload(device="cuda", **kw)
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z.reshape(-1, w.d), w.nbr, w.y))
m = p.VifModel(X, Z, nbr, y, device=dev)
th = p.Theta(**w.theta_dict())
B = torch.zeros((w.n, w.mv), dtype=torch.float64, device=dev)
D = torch.zeros(w.n, dtype=torch.float64, device=dev)
t = m.evaluate(th, B, D)
gt, g = m.grad(th)
nb = m.neighbors(th, w.mv).cpu().numpy()
print(json.dumps({"terms": [t.nll, t.logdet_D, t.logdet_M, t.quad], "B": B.cpu().numpy().tolist(),
                  "D": D.cpu().numpy().tolist(), "grad": [float(x) for x in g], "grad_nll": gt.nll,
                  "nbr": nb.tolist()}))
""" % ROOT


@pytest.fixture(scope="module")
def refs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = {}
    for name, kw in WORKLOADS.items():
        w = vifgen.make_workload(device="cuda", **kw)
        oth = oracle.Theta(**w.theta_dict())
        out[name] = (w, oth, oracle.factor_nll(w.X, w.Z, w.nbr, w.y, oth), oracle.grad(w.X, w.Z, w.nbr, w.y, oth),
                     oracle.dc_neighbors(w.X, w.Z, oth, w.mv))
    return out


def run(wname, env):
    r = subprocess.run([sys.executable, "-c", CODE, json.dumps(WORKLOADS[wname])], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("wname,env", [
    ("d2", {}),
    ("d2", {"VIF_KX_GENERIC": "1", "VIF_VECCHIA_GENERIC_D": "1"}),
    ("d2", {"VIF_GRAD_RORDER": "0", "VIF_GR_BLOCKS": "37"}),
    ("d2", {"VIF_KNN_EW": "4", "VIF_GRAD_STATE": "1"}),
    ("d5", {}),
    ("d5", {"VIF_ORDER_ND": "0"}),
    ("d5", {"VIF_ORDER_K": "2", "VIF_KX_GENERIC": "1"}),
], ids=lambda v: v if isinstance(v, str) else ("+".join(f"{k}={x}" for k, x in v.items()) or "default"))
def test_knob_matches_oracle(refs, wname, env):
    w, oth, r, rg, (rn, rs) = refs[wname]
    g = run(wname, env)
    nll, ld, lm, q = g["terms"]
    scale = abs(r.logdet_D) + abs(r.logdet_M) + abs(r.quad)
    assert abs(nll - r.nll) <= 1e-8 * max(abs(r.nll), 1e-3 * scale), (nll, r.nll)
    for a, b in ((ld, r.logdet_D), (lm, r.logdet_M), (q, r.quad)):
        assert abs(a - b) <= 1e-10 * max(abs(b), 1e-10 * scale), (a, b)
    check_D(np.array(g["D"]), r.D)
    check_B(np.array(g["B"]), r.B)
    # gradient: the tolerance of tests/test_gpu_grad.py
    gv = np.array(g["grad"])
    gscale = np.maximum(np.abs(rg.grad), 0.5 * np.abs(rg.parts).sum(axis=1))
    assert np.all(np.abs(gv - rg.grad) / gscale <= 1e-8), (gv, rg.grad)
    assert g["grad_nll"] == pytest.approx(r.nll, rel=1e-8)
    # neighbour sets: bit-exact except exact ties, whose oracle scores agree (tests/test_gpu_knn.py)
    nb = np.array(g["nbr"], dtype=np.int64)
    diff = np.nonzero((nb != rn).any(1))[0]
    assert len(diff) <= max(2, 0.005 * w.n), len(diff)
    for i in diff:
        sel = nb[i][nb[i] >= 0]
        assert len(sel) == (rn[i] >= 0).sum() and np.all(sel < i) and len(set(sel)) == len(sel)
        gs = oracle.dc_scores(w.X, w.Z, oth, np.full(len(sel), i), sel)
        np.testing.assert_allclose(gs, rs[i][:len(sel)], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("env", [
    {"VIF_LA_LONG": "8"},                                # lanes-over-entries rows from 8 entries on, every ncol
    {"VIF_LA_LONG": "1000000"},                          # never
    {"VIF_LA_LVL_BPS": "2", "VIF_LA_LVL_CTAS": "40"},    # two CTAs per SM allowed, grid capped at 40 CTAs
], ids=lambda v: "+".join(f"{k}={x}" for k, x in v.items()))
def test_laplace_solve_launch_knobs(env):
    """The launch-shape knobs of the level-scheduled triangular solves (k_laplace.cu, section 13): the
    operator, mode and SLQ parity cases of test_gpu_laplace.py (each against oracle/laplace.py) rerun in a
    process with the knob set."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_laplace.py"), "-q", "-x",
                        "-m", "gpu", "-k", "test_operators or test_mode_shapes or test_slq_logdet or "
                        "test_sigma_inv_inverts_sigma"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=1500, cwd=ROOT)
    tail = r.stdout[-1500:] + r.stderr[-500:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout and " skipped" not in r.stdout, tail

"""Robustness of the boundary (include/vif.h error behaviour): non-finite
inputs, invalid prediction neighbours, input marshalling of VifModel.set_data, stale Laplace state,
NOT_PD and the NCCL wait on a communicator, and -- when the box has two GPUs -- the real two-rank NCCL
path against the oracle.  Needs a B200."""
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
from parity import check_D, check_terms  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


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


def small(n=400, m=12, mv=6, seed=5):
    return vifgen.make_workload(n=n, d=2, m=m, mv=mv, family="matern32", rho=0.15, nugget=0.1, seed=seed,
                                device="cuda")


def dev_inputs(w, X=None, Z=None, nbr=None, y=None):
    dev = torch.device("cuda")
    arrs = (w.X if X is None else X, w.Z if Z is None else Z, w.nbr if nbr is None else nbr, w.y if y is None else y)
    return tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs)


@pytest.mark.parametrize("what,row", [("X", 123), ("y", 7), ("y", 399), ("Xinf", 0)])
def test_non_finite_inputs_rejected_at_create(what, row):
    """A NaN / inf in X or y is INVALID_ARG naming the first offending row (validation at vif_create)."""
    p = vif()
    w = small()
    X, y = w.X.copy(), w.y.copy()
    if what == "X":
        X[row, 1] = np.nan
    elif what == "Xinf":
        X[row, 0] = np.inf
    else:
        y[row] = np.nan
    with pytest.raises(p.VifError) as e:
        p.VifModel(*dev_inputs(w, X=X, y=y))
    assert e.value.status == 1 and f"row {row}" in e.value.msg


def test_non_finite_inducing_point_and_set_data_validation():
    p = vif()
    w = small()
    Z = w.Z.copy()
    Z[3, 0] = np.nan
    with pytest.raises(p.VifError) as e:
        p.VifModel(*dev_inputs(w, Z=Z))
    assert e.value.status == 1 and "inducing" in e.value.msg
    model = p.VifModel(*dev_inputs(w))
    t0 = model.evaluate(p.Theta(**w.theta_dict())).nll
    y = w.y.copy()
    y[250] = np.nan
    with pytest.raises(p.VifError) as e:
        model.set_data(y=torch.from_numpy(y).cuda(), validate=True)
    assert e.value.status == 1 and "row 250" in e.value.msg
    model.set_data(y=w.y, validate=True)  # numpy input is marshalled like the constructor's
    assert model.evaluate(p.Theta(**w.theta_dict())).nll == t0
    model.close()


def test_set_data_marshalling_and_sizes():
    """set_data marshals numpy / non-contiguous inputs and rejects wrong dtypes and sizes
    instead of reading raw bytes."""
    p = vif()
    w = small()
    model = p.VifModel(*dev_inputs(w))
    th = p.Theta(**w.theta_dict())
    t0 = model.evaluate(th).nll
    Xt = torch.from_numpy(np.ascontiguousarray(w.X.T)).cuda().t()  # non-contiguous view -> made contiguous
    assert not Xt.is_contiguous()
    model.set_data(X=Xt, y=w.y)
    assert model.evaluate(th).nll == t0
    with pytest.raises(TypeError):
        model.set_data(X=torch.from_numpy(w.X.astype(np.float32)).cuda())
    with pytest.raises(ValueError):
        model.set_data(y=w.y[:-1])
    with pytest.raises(ValueError):
        model.set_data(nbr=w.nbr[:, :-1].copy())
    model.close()


def test_predict_invalid_neighbours_rejected():
    """vif_predict validates nbrp (indices in [0, n), distinct, -1 only trailing) before the vecchia
    kernel gathers them."""
    p = vif()
    w = small()
    Xp, nbrp = vifgen.make_prediction(w, 50, device="cuda")
    model = p.VifModel(*dev_inputs(w))
    th = p.Theta(**w.theta_dict())
    mu = model.predict(th, Xp, nbrp)
    assert np.all(np.isfinite(mu.cpu().numpy()))
    for bad, row in (("range", 11), ("middle", 20), ("dup", 33), ("nan", 44)):
        b = nbrp.copy()
        Xb = Xp.copy()
        if bad == "range":
            b[row, 2] = w.n
        elif bad == "middle":
            b[row, 1] = -1
        elif bad == "dup":
            b[row, 3] = b[row, 0]
        else:
            Xb[row, 0] = np.nan
        with pytest.raises(p.VifError) as e:
            model.predict(th, Xb, b)
        assert e.value.status == 1 and f"row {row}" in e.value.msg, e.value.msg
    mu2 = model.predict(th, Xp, nbrp)  # the handle is still usable
    assert torch.equal(mu, mu2)
    model.close()


def test_set_data_invalidates_laplace_workspace():
    """a prepared VIF-Laplace workspace is stale after vif_set_data (VIF_ERR_STATE), not
    silently combined with the new neighbour structure."""
    p = vif()
    lw = vifgen.make_laplace_workload(n=500, m=16, mv=8, family="matern32", rho=0.2, device="cuda")
    model = p.VifModel(*dev_inputs(lw))
    th = p.Theta(**lw.theta_dict())
    opts = p.LaOpts(max_newton=30, newton_tol=1e-10, max_cg=300, cg_tol=1e-10, nprobe=0, slq_tol=1e-10)
    model.la_prepare(th, nprobe=0, max_cg=300)
    model.la_nll(lw.y, opts)
    nbr = lw.nbr.copy()
    model.set_data(nbr=nbr)
    with pytest.raises(p.VifError) as e:
        model.la_nll(lw.y, opts)
    assert e.value.status == 6
    model.la_prepare(th, nprobe=0, max_cg=300)
    model.la_nll(lw.y, opts)
    model.close()


_NCCL_NOTPD = r"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2507_05064_b200 as p
dev = torch.device("cuda")
X = np.array([[0.1, 0.1], [0.5, 0.5], [0.5, 0.5], [0.7, 0.2]] * 1)
nbr = np.array([[-1, -1], [0, -1], [1, 0], [2, 1]], np.int32)
out = {{}}
model = p.VifModel(torch.from_numpy(X).to(dev), torch.zeros((0, 2), dtype=torch.float64, device=dev),
                   torch.from_numpy(nbr).to(dev), torch.zeros(4, dtype=torch.float64, device=dev),
                   nccl_id=p.vif_nccl_unique_id(), device=dev)
try:
    model.evaluate(p.Theta("matern32", 1.0, [0.3, 0.3], 0.0, 0.0))
    out["status"] = 0
except p.VifError as e:
    out["status"], out["bad_row"] = e.status, e.bad_row
# the same handle recovers with a positive nugget (the failure state is per evaluation)
t = model.evaluate(p.Theta("matern32", 1.0, [0.3, 0.3], 0.1, 0.0))
out["nll"] = t.nll
print(json.dumps(out))
"""


def test_nccl_single_rank_not_pd_and_wait():
    """On a communicator (VIF_NCCL_SINGLE=1: one rank, the multi-GPU schedule) NOT_PD is reported through
    the reduced failure state with the failing row, the polling wait (short VIF_NCCL_TIMEOUT_S) returns
    normally, and the handle is usable afterwards."""
    env = dict(os.environ, VIF_NCCL_SINGLE="1", VIF_NCCL_TIMEOUT_S="30")
    r = subprocess.run([sys.executable, "-c", _NCCL_NOTPD.format(root=ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["status"] == 2 and out["bad_row"] in (2, 3)
    assert np.isfinite(out["nll"])


_TWO_RANK = r"""
import json, os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
import paper_2507_05064_b200 as p
import vifgen
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
dev = torch.device("cuda", rank)
w = vifgen.make_workload(n=6001, d=2, m=40, mv=12, family="matern32", rho=0.12, nugget=0.08, seed=61, device="cpu")
uid = [p.vif_nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
model = p.VifModel(X, Z, nbr, y, rank=rank, world=world, nccl_id=uid[0], device=dev)
th = p.Theta(**w.theta_dict())
D = torch.zeros(w.n, dtype=torch.float64, device=dev)
t = model.evaluate(th, None, D)
_, g = model.grad(th)
rows = model.owned_rows()
out = dict(rank=rank, nll=t.nll, logdet_D=t.logdet_D, logdet_M=t.logdet_M, quad=t.quad, g=list(map(float, g)),
           rows=rows.tolist(), D=D.cpu().numpy()[rows].tolist())
# NOT_PD on one rank's row must reach every rank: a non-finite coordinate loaded without validation
# makes the last point's residual block fail (no other point conditions on it)
X2 = w.X.copy(); X2[w.n - 1, 0] = np.nan
model.set_data(X=torch.from_numpy(X2).to(dev))
try:
    model.evaluate(th)
    out["notpd"] = 0
except p.VifError as e:
    out["notpd"], out["bad_row"] = e.status, e.bad_row
json.dump(out, open(os.environ["OUT"] + f".{{rank}}", "w"))
model.close()
dist.barrier()
dist.destroy_process_group()
"""


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_rank_nccl_matches_oracle(tmp_path):
    """The real multi-GPU path (two processes, per-round NCCL all-gather of U, all-reduce of the Gram,
    the failure state and the gradient sums) against the oracle; NOT_PD found on one rank is returned by
    both with the same row."""
    script = tmp_path / "two_rank.py"
    script.write_text(_TWO_RANK.format(root=ROOT))
    out = str(tmp_path / "out")
    env = dict(os.environ, OUT=out, VIF_NCCL_TIMEOUT_S="120")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2", "--master-addr",
                        "127.0.0.1", "--master-port", "29533", str(script)], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = [json.load(open(f"{out}.{k}")) for k in range(2)]
    w = vifgen.make_workload(n=6001, d=2, m=40, mv=12, family="matern32", rho=0.12, nugget=0.08, seed=61, device="cpu")
    ref = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    for o in res:
        check_terms(type("T", (), o), ref.nll, ref.logdet_D, ref.logdet_M, ref.quad)
        assert o["nll"] == res[0]["nll"] and o["g"] == res[0]["g"]
        check_D(np.array(o["D"]), ref.D[o["rows"]])
        assert o["notpd"] == 2 and o["bad_row"] == w.n - 1
    assert sorted(res[0]["rows"] + res[1]["rows"]) == list(range(w.n))
    g = oracle.grad(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    scale = np.maximum(np.abs(g.grad), 0.5 * np.abs(g.parts).sum(axis=1))
    assert np.max(np.abs(np.array(res[0]["g"]) - g.grad) / scale) <= 1e-8

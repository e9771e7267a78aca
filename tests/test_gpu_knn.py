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


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_world_same_sets(world):
    """An emulated multi-rank handle searches every query block: the sets equal the one-rank result."""
    import paper_2507_05064_b200 as p
    w = vifgen.make_workload(n=1500, d=2, m=30, mv=12, family="matern32", rho=0.15, nugget=0.1, seed=21,
                             device="cuda")
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
    th = p.Theta(**w.theta_dict())
    outs = []
    for wd in (1, world):
        model = p.VifModel(X, Z, nbr, y, world=wd, device=dev)
        outs.append(model.neighbors(th, 12).cpu().numpy())
        model.close()
    np.testing.assert_array_equal(outs[1], outs[0])


def test_u_in_row_blocks_same_sets():
    """u_i computed in row blocks (the multi-rank path; forced small blocks) gives the same sets."""
    import json
    import os
    import subprocess
    import sys
    code = r"""
import sys, json
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2507_05064_b200 as p, vifgen
w = vifgen.make_workload(n=1100, d=2, m=40, mv=10, family="matern52", rho=0.2, nugget=0.1, seed=22, device="cuda")
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
m = p.VifModel(X, Z, nbr, y, device=dev)
print(json.dumps(m.neighbors(p.Theta(**w.theta_dict()), 10).cpu().numpy().tolist()))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for rows in ("0", "137"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, VIF_KNN_UROWS=rows),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(np.array(json.loads(r.stdout.strip().splitlines()[-1])))
    np.testing.assert_array_equal(res[1], res[0])


def test_query_block_shards_cover_every_row():
    """The rank-g query blocks (kb = g, g + G, ...) of G ranks write disjoint rows that together equal the
    one-rank result (VIF_KNN_SHARD test hook: one process plays each rank's search in turn)."""
    import json
    import os
    import subprocess
    import sys
    code = r"""
import sys, json
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2507_05064_b200 as p, vifgen
w = vifgen.make_workload(n=1300, d=2, m=25, mv=11, family="matern32", rho=0.15, nugget=0.1, seed=23, device="cuda")
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
m = p.VifModel(X, Z, nbr, y, device=dev)
out = torch.full((w.n, 11), -7, dtype=torch.int32, device=dev)
p.vif_neighbors(m.handle, p.Theta(**w.theta_dict()), 11, out)
print(json.dumps(out.cpu().numpy().tolist()))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    def run(shard):
        env = dict(os.environ)
        if shard:
            env["VIF_KNN_SHARD"] = shard
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        return np.array(json.loads(r.stdout.strip().splitlines()[-1]))
    full = run(None)
    parts = [run(f"{g},3") for g in range(3)]
    written = [(pt != -7).all(1) for pt in parts]
    assert np.array_equal(sum(wr.astype(int) for wr in written), np.ones(full.shape[0], int))  # disjoint, complete
    merged = np.where(written[0][:, None], parts[0], np.where(written[1][:, None], parts[1], parts[2]))
    np.testing.assert_array_equal(merged, full)


@pytest.mark.slow
def test_search_config3_equals_generator():
    """n = 1M (config 3): vif_neighbors returns the generator's sets (vifgen's own torch brute force) on every
    row except exact ties, whose oracle scores agree."""
    import time
    import paper_2507_05064_b200 as p
    w = vifgen.make_config(3, device="cuda")
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, device=dev)
    th = p.Theta(**w.theta_dict())
    t0 = time.perf_counter()
    g = model.neighbors(th, w.mv).cpu().numpy()
    dt = time.perf_counter() - t0
    diff = np.nonzero((g != w.nbr).any(1))[0]
    assert len(diff) <= 0.001 * w.n, len(diff)
    oth = oracle.Theta(**w.theta_dict())
    for i in diff[:200]:  # differences only at ties: the same multiset of oracle scores
        a = oracle.dc_scores(w.X, w.Z, oth, np.full(w.mv, i), g[i])
        b = oracle.dc_scores(w.X, w.Z, oth, np.full(w.mv, i), w.nbr[i])
        np.testing.assert_allclose(np.sort(a), np.sort(b), rtol=1e-12, atol=1e-14)
    print(f"vif_neighbors n = 1M: {dt:.2f} s")
    model.close()


@pytest.mark.parametrize("family,n,m,mv,d,rho", [("matern32", 3000, 60, 20, 2, 0.15), ("gaussian", 2500, 250, 31, 2, 0.15),
                                                  ("matern12", 1200, 8, 47, 2, 0.15), ("matern52", 2000, 100, 15, 5, 0.6)])
def test_int8_and_dmma_engines_agree(family, n, m, mv, d, rho):
    """vif_neighbors with the Gram blocks on the integer tensor cores (default, reading c18) and on DMMA
    (VIF_KNN_FP64=1, read once per process: subprocesses): the same sets on every row except scores equal
    to rounding, where both choices carry the same oracle score"""
    import json
    import os
    import subprocess
    import sys
    code = r"""
import sys, json
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2507_05064_b200 as p, vifgen
w = vifgen.make_workload(n=%d, d=%d, m=%d, mv=%d, family=%r, rho=%r, nugget=0.1, seed=77, device="cuda")
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
m = p.VifModel(X, Z, nbr, y, device=dev)
print(json.dumps(m.neighbors(p.Theta(**w.theta_dict()), %d).cpu().numpy().tolist()))
""" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), n, d, m, mv, family, rho, mv)
    outs = []
    for fp64 in ("0", "1"):
        # the int8 run places its digit slices in the W buffer (the n > 2^20 placement) for the largest case
        env = dict(os.environ, VIF_KNN_FP64=fp64, VIF_KNN_WSLICES="1" if m >= 100 else "0")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.array(json.loads(r.stdout.strip().splitlines()[-1])))
    a, b = outs
    w = vifgen.make_workload(n=n, d=d, m=m, mv=mv, family=family, rho=rho, nugget=0.1, seed=77, device="cuda")
    diff = np.nonzero((a != b).any(1))[0]
    assert len(diff) <= max(2, 0.005 * n), len(diff)
    oth = oracle.Theta(**w.theta_dict())
    for i in diff:
        sa, sb = a[i][a[i] >= 0], b[i][b[i] >= 0]
        assert len(sa) == len(sb) and np.all(sa < i) and len(set(sa)) == len(sa)
        ga = oracle.dc_scores(w.X, w.Z, oth, np.full(len(sa), i), sa)
        gb = oracle.dc_scores(w.X, w.Z, oth, np.full(len(sb), i), sb)
        np.testing.assert_allclose(ga, gb, rtol=1e-12, atol=1e-14)

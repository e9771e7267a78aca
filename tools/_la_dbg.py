import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import __graft_entry__; __graft_entry__.build()
import paper_2507_05064_b200 as p, vifgen, oracle
from oracle import laplace as la
n, m, mv, ncol = 300, 9, 0, 2
w = vifgen.make_laplace_workload(n=n, m=m, mv=mv, family="matern32", rho=0.2, device="cuda", seed=n + mv) if False else None
import test_gpu_laplace as T
w = T.work(n, m, mv, seed=n + mv)
th = p.Theta(**w.theta_dict())
model = T.model_of(w, th, nprobe=ncol)
rng = np.random.default_rng(ncol)
V = rng.standard_normal((n, ncol))
lat = la.latent_factor(w.X, w.Z, w.nbr, oracle.Theta(**w.theta_dict()))
for op in ["btinv", "binv", "btinv", "sigma"]:
    got = model.la_apply(op, V).cpu().numpy()
    ref = {"btinv": lat.btinv(V), "binv": lat.binv(V), "sigma": lat.sigma_dagger(V)}[op]
    bad = np.nonzero(~np.isfinite(got).all(1))[0]
    print(op, "nonfinite rows", len(bad), bad[:10], "maxerr finite", np.nanmax(np.abs(got - ref)))

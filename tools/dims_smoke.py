"""Every entry point at the dimensions of BASELINE configs 4 and 5 (small n): catches launch-shape
failures (shared-memory opt-ins, template dispatch) that the small parity shapes do not reach."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_05064_b200 as p  # noqa: E402
import vifgen  # noqa: E402


def run(cid, n):
    w = vifgen.make_config(cid, device="cuda", n=n)
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
    th = p.Theta(**w.theta_dict())
    model = p.VifModel(X, Z, nbr, y, device=dev)
    out = {"config": cid, "n": n, "d": w.d, "m": w.Z.shape[0], "mv": w.mv}
    out["nll"] = model.evaluate(th).nll
    if w.mv <= 31:
        out["grad0"] = float(model.grad(th)[1][0])
    Xp, nbrp = vifgen.make_prediction(w, 500, x="normal" if cid == 4 else "uniform", device="cuda")
    mu, var = model.predict(th, Xp, nbrp, want_var=True)
    out["mu0"], out["var_min"] = float(mu[0]), float(var.min())
    nb = model.neighbors(th, w.mv)
    out["nbr_equal_rows"] = float((nb.cpu().numpy() == w.nbr).all(1).mean())
    model.close()
    lw = vifgen.make_laplace_workload(n=n, d=w.d, m=w.Z.shape[0], mv=min(w.mv, 30), family=w.family, rho=0.5,
                                      device="cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (lw.X, lw.Z, lw.nbr, lw.y))
    lm = p.VifModel(X, Z, nbr, y, device=dev)
    lm.la_prepare(p.Theta(**lw.theta_dict()), nprobe=8, max_cg=300)
    e1, e2 = vifgen.make_probes(n, lw.Z.shape[0], 8)
    t, _ = lm.la_nll(lw.y, p.LaOpts(max_newton=30, newton_tol=1e-8, max_cg=300, cg_tol=1e-8, nprobe=8, slq_tol=1e-8),
                     e1, e2)
    out["la_nll"] = t.nll
    lm.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    run(4, 4000)
    run(5, 4000)

"""Small end-to-end run of every library entry point, for compute-sanitizer (SURVEY 4, T-san):
factor + NLL (config 1), emulated 3-rank factor, gradient, prediction, neighbour search, and the
VIF-Laplace path (prepare, operators, mode + SLQ)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_05064_b200 as p  # noqa: E402
import vifgen  # noqa: E402


def main():
    dev = torch.device("cuda")
    w = vifgen.make_workload(n=700, d=2, m=37, mv=13, family="matern32", rho=0.15, nugget=0.1, seed=3, device="cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
    th = p.Theta(**w.theta_dict())
    for world in (1, 3):
        model = p.VifModel(X, Z, nbr, y, world=world, device=dev)
        B = torch.zeros((w.n, w.mv), dtype=torch.float64, device=dev)
        D = torch.zeros(w.n, dtype=torch.float64, device=dev)
        t = model.evaluate(th, B, D)
        _, g = model.grad(th)
        Xp, nbrp = vifgen.make_prediction(w, 50, device="cuda")
        mu, var = model.predict(th, Xp, nbrp, want_var=True)
        print(f"world {world}: nll {t.nll:.6f} grad {g[0]:.6f} mu[0] {float(mu[0]):.6f}")
        if world == 1:
            nb = model.neighbors(th, w.mv)
            print("neighbors equal:", bool((nb.cpu().numpy() == w.nbr).all()))
        model.close()
    lw = vifgen.make_laplace_workload(n=500, m=20, mv=10, family="matern32", rho=0.2, device="cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (lw.X, lw.Z, lw.nbr, lw.y))
    lm = p.VifModel(X, Z, nbr, y, device=dev)
    lm.la_prepare(p.Theta(**lw.theta_dict()), nprobe=33, max_cg=200)
    V = torch.randn(lw.n, 33, dtype=torch.float64, device=dev)
    winv = torch.full((lw.n,), 4.0, dtype=torch.float64, device=dev)
    for op in ("sigma", "A", "binv", "btinv", "fitc_solve"):
        lm.la_apply(op, V, winv=winv)
        lm.la_apply(op, V[:, 0].contiguous(), winv=winv)
    e1, e2 = vifgen.make_probes(lw.n, 20, 33)
    t, _ = lm.la_nll(lw.y, p.LaOpts(max_newton=20, newton_tol=1e-8, max_cg=200, cg_tol=1e-8, nprobe=33, slq_tol=1e-8),
                     e1, e2)
    print(f"laplace nll {t.nll:.6f} newton {t.newton_iters} cg {t.cg_iters}")
    lm.close()
    torch.cuda.synchronize()
    print("sanitize run done")


if __name__ == "__main__":
    main()

"""Debug helper: B/D of the current vecchia variant vs the oracle on a small workload, per row."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import oracle
import paper_2507_05064_b200 as p
import vifgen
np.set_printoptions(precision=6, linewidth=200)
for (n, m, mv) in [(60, 8, 4), (300, 20, 10), (2000, 50, 30)]:
    w = vifgen.make_workload(n=n, d=2, m=m, mv=mv, family="matern32", rho=0.15, nugget=0.1, seed=1, device="cuda")
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, device=dev)
    B = torch.zeros((w.n, w.mv), dtype=torch.float64, device=dev)
    D = torch.zeros(w.n, dtype=torch.float64, device=dev)
    try:
        t = model.evaluate(p.Theta(**w.theta_dict()), B, D)
        print("nll", t.nll)
    except p.VifError as e:
        print("error", e)
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()))
    B, D = B.cpu().numpy(), D.cpu().numpy()
    print(n, m, mv, "oracle nll", r.nll)
    bad = [i for i in range(n) if not (abs(D[i] - r.D[i]) <= 1e-9 * r.D[i])]
    print("bad D rows", len(bad), bad[:20])
    for i in bad[:4] + list(range(3)):
        print(i, "q", int((w.nbr[i] >= 0).sum()), "D", D[i], r.D[i], "\n  B", B[i][:8], "\n  Bo", r.B[i][:8])
    model.close()

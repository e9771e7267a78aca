"""Time the VIF-Laplace path (vif_la_prepare + vif_la_nll) on the paper's Laplace workload recipe
(d = 5, ARD Gaussian covariance, binary responses) at a given n / m / m_v / ell."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import vifgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--m", type=int, default=200)
    ap.add_argument("--mv", type=int, default=30)
    ap.add_argument("--ell", type=int, default=50)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--family", default="gaussian")
    ap.add_argument("--oracle", action="store_true")
    a = ap.parse_args()
    import paper_2507_05064_b200 as p
    t0 = time.time()
    w = vifgen.make_laplace_workload(n=a.n, m=a.m, mv=a.mv, family=a.family, device="cuda")
    gen = time.time() - t0
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (w.X, w.Z, w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, device=dev)
    th = p.Theta(**w.theta_dict())
    eps1, eps2 = vifgen.make_probes(a.n, a.m, a.ell)
    e1 = torch.from_numpy(eps1).to(dev)
    e2 = torch.from_numpy(eps2).to(dev)
    opts = p.LaOpts(max_newton=50, newton_tol=a.tol, max_cg=1000, cg_tol=a.tol, nprobe=a.ell, slq_tol=a.tol)
    out = []
    for r in range(a.reps + 1):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        model.la_prepare(th, nprobe=a.ell, max_cg=1000)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        t, b = model.la_nll(y, opts, e1, e2)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rec = dict(rep=r, prepare_ms=1e3 * (t2 - t1), nll_ms=1e3 * (t3 - t2), nll=t.nll, neg_loglik=t.neg_loglik,
                   quad=t.quad, logdet=t.logdet, newton=t.newton_iters, cg=t.cg_iters, slq_max=t.slq_iters_max,
                   slq_mean=t.slq_iters_mean)
        out.append(rec)
        print(json.dumps(rec), flush=True)
    # one Sigma_dagger apply and one FITC solve (ncol = 1 and ell), timed alone
    for ncol in (1, a.ell):
        V = torch.randn(a.n, ncol, dtype=torch.float64, device=dev) if ncol > 1 else torch.randn(a.n, dtype=torch.float64, device=dev)
        for op in ("btinv", "binv", "sigma", "sigma_inv"):
            model.la_apply(op, V)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            for _ in range(5):
                model.la_apply(op, V)
            torch.cuda.synchronize()
            print(json.dumps(dict(op=op, ncol=ncol, ms=1e3 * (time.perf_counter() - t1) / 5)), flush=True)
    print(json.dumps(dict(gen_s=gen)))
    if a.oracle:
        import oracle
        from oracle import laplace as la
        t1 = time.time()
        r = la.vifla_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), eps1=eps1, eps2=eps2,
                         newton_tol=a.tol, cg_tol=a.tol, slq_tol=a.tol)
        print(json.dumps(dict(oracle_s=time.time() - t1, nll=r.nll, logdet=r.logdet, newton=r.newton_iters,
                              cg=r.cg_iters)))


if __name__ == "__main__":
    main()

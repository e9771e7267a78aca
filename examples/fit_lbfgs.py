"""Fit theta = (sigma_1^2, range, sigma^2) by L-BFGS on the GPU NLL and its gradient (the paper
fits its GP models by minimising L_dagger with a quasi-Newton method).

  python examples/fit_lbfgs.py [--config 2] [--n 100000]

Optimises over log-parameters (isotropic range: dNLL/drho = sum_j dNLL/dlambda_j), starting from a
perturbed theta; every function/gradient evaluation is one vif_grad call (factor + NLL + gradient)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
from scipy.optimize import minimize

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def fit(model, w, start, maxiter=40, verbose=False):
    import paper_2507_05064_b200 as p
    d = w.d
    evals = []

    def fun(logv):
        s2, rho, nug = np.exp(logv)
        th = p.Theta(w.family, float(s2), np.full(d, rho), float(nug), w.jitter)
        terms, g = model.grad(th)
        gl = np.array([g[0], g[1:1 + d].sum(), g[1 + d]]) * np.exp(logv)  # chain rule to log-parameters
        evals.append((float(terms.nll), [float(x) for x in np.exp(logv)]))
        if verbose:
            print(json.dumps({"nll": terms.nll, "theta": evals[-1][1], "grad_log": list(map(float, gl))}))
        return terms.nll, gl

    t = time.perf_counter()
    r = minimize(fun, np.log(start), jac=True, method="L-BFGS-B", options={"maxiter": maxiter, "gtol": 1e-5})
    return r, evals, time.perf_counter() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_05064_b200 as p
    import vifgen
    w = vifgen.make_config(args.config, device="cuda", n=args.n)
    dev = torch.device("cuda")
    model = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
    truth = np.array([w.sigma2, w.lengthscale[0], w.nugget])
    start = truth * np.array([2.0, 0.5, 3.0])
    r, evals, secs = fit(model, w, start, verbose=args.verbose)
    print(json.dumps({"config": args.config, "n": w.n, "truth": truth.tolist(), "start": start.tolist(),
                      "estimate": np.exp(r.x).tolist(), "nll_start": evals[0][0], "nll_end": float(r.fun),
                      "evaluations": len(evals), "seconds": secs, "converged": bool(r.success)}))


if __name__ == "__main__":
    main()

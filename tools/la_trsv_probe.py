"""Triangular-solve timings of the VIF-Laplace path vs the number of columns (tools/la_probe.py workload)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import vifgen  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
    import paper_2507_05064_b200 as p
    w = vifgen.make_laplace_workload(n=n, m=200, mv=30, device="cuda")
    dev = torch.device("cuda")
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (w.X, w.Z, w.nbr, w.y))
    model = p.VifModel(X, Z, nbr, y, device=dev)
    model.la_prepare(p.Theta(**w.theta_dict()), nprobe=64, max_cg=100)
    cnt = np.bincount(w.nbr[w.nbr >= 0].ravel(), minlength=n)
    lev = np.zeros(n, np.int64)
    nb = w.nbr
    for i in range(n):
        r = nb[i][nb[i] >= 0]
        if len(r):
            lev[i] = lev[r].max() + 1
    hist = np.bincount(lev)
    print(json.dumps(dict(children_max=int(cnt.max()), children_mean=float(cnt.mean()),
                          children_p99=float(np.percentile(cnt, 99)), depth=int(lev.max()) + 1,
                          level_width_min=int(hist.min()), level_width_median=float(np.median(hist)))))
    for ncol in (1, 2, 4, 8, 16, 32, 33, 50, 64):
        V = torch.randn(n, ncol, dtype=torch.float64, device=dev) if ncol > 1 else torch.randn(n, dtype=torch.float64, device=dev)
        rec = dict(ncol=ncol)
        for op in ("btinv", "binv"):
            model.la_apply(op, V)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            for _ in range(5):
                model.la_apply(op, V)
            torch.cuda.synchronize()
            rec[op] = 1e3 * (time.perf_counter() - t1) / 5
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

"""Three Sigma_dagger applications (ncol = 1) on the n = 100k Laplace recipe, for ncu launch lists."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import vifgen  # noqa: E402
import paper_2507_05064_b200 as p  # noqa: E402
n = 100000
w = vifgen.make_laplace_workload(n=n, m=200, mv=30, device="cuda")
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (w.X, w.Z, w.nbr, w.y))
model = p.VifModel(X, Z, nbr, y, device=dev)
model.la_prepare(p.Theta(**w.theta_dict()), nprobe=1, max_cg=10)
v = torch.randn(n, dtype=torch.float64, device=dev)
for _ in range(3):
    model.la_apply("sigma", v)
torch.cuda.synchronize()

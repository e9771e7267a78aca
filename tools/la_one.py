import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import vifgen, paper_2507_05064_b200 as p
n = 100000
w = vifgen.make_laplace_workload(n=n, m=200, mv=30, device="cuda")
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (w.X, w.Z, w.nbr, w.y))
model = p.VifModel(X, Z, nbr, y, device=dev)
model.la_prepare(p.Theta(**w.theta_dict()), nprobe=64, max_cg=100)
V = torch.randn(n, 2, dtype=torch.float64, device=dev)
for _ in range(3):
    model.la_apply("btinv", V)
    model.la_apply("binv", V)
torch.cuda.synchronize()
print("done")

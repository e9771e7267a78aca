import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import vifgen, paper_2507_05064_b200 as p
n = 100000
w = vifgen.make_laplace_workload(n=n, m=200, mv=30, device="cuda")
dev = torch.device("cuda")
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (w.X, w.Z, w.nbr, w.y))
model = p.VifModel(X, Z, nbr, y, device=dev)
th = p.Theta(**w.theta_dict())
e1, e2 = (torch.from_numpy(a).to(dev) for a in vifgen.make_probes(n, 200, 50))
opts = p.LaOpts(max_newton=50, newton_tol=1e-6, max_cg=1000, cg_tol=1e-6, nprobe=50, slq_tol=1e-6)
model.la_prepare(th, nprobe=50, max_cg=1000)
t, b = model.la_nll(y, opts, e1, e2)
torch.cuda.synchronize()
print(t)

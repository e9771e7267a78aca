import os, sys, json, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import vifgen, paper_2507_05064_b200 as p
w = vifgen.make_config(4, device="cuda", n=int(sys.argv[1]))
dev = torch.device("cuda")
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)), device=dev)
th = p.Theta(**w.theta_dict())
m.grad(th); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(2): _, g = m.grad(th)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(2): m.evaluate(th)
torch.cuda.synchronize()
print(json.dumps({"n": w.n, "d": w.d, "m": w.Z.shape[0], "grad_ms": (t1 - t) / 2 * 1e3, "nll_ms": (time.perf_counter() - t1) / 2 * 1e3, "g0": float(g[0])}))

"""Timing probe for vif_grad at the config-3 recipe (n points, default 300k); workload cached in /tmp."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2507_05064_b200 as p
import vifgen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cache = f"/tmp/vif_probe_c3_{n}.npz"
if os.path.exists(cache):
    z = np.load(cache)
    X, Z, nbr, y = z["X"], z["Z"], z["nbr"], z["y"]
    td = json.loads(str(z["theta"])); td["lengthscale"] = np.array(td["lengthscale"])
else:
    w = vifgen.make_config(3, device="cuda", n=n)
    X, Z, nbr, y = w.X, w.Z, w.nbr, w.y
    td = {**w.theta_dict(), "lengthscale": [float(v) for v in w.lengthscale]}
    np.savez(cache, X=X, Z=Z, nbr=nbr, y=y, theta=json.dumps(td))
    td["lengthscale"] = np.array(td["lengthscale"])
dev = torch.device("cuda")
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (X, Z, nbr, y)))
th = p.Theta(**td)
m.grad(th)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(reps):
    terms, g = m.grad(th)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / reps
t = time.perf_counter()
for _ in range(reps):
    m.evaluate(th)
torch.cuda.synchronize()
de = (time.perf_counter() - t) / reps
print(json.dumps({"n": n, "grad_ms": dt * 1e3, "nll_ms": de * 1e3, "grad": list(map(float, g))}))

"""vif_grad timing for any BASELINE config recipe at n points: python tools/grad_config_probe.py <config> <n> [reps]"""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2507_05064_b200 as p
import vifgen
cid, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = vifgen.make_config(cid, device="cuda", n=n)
dev = torch.device("cuda")
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
th = p.Theta(**w.theta_dict())
m.grad(th)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(reps):
    terms, g = m.grad(th)
torch.cuda.synchronize()
gms = (time.perf_counter() - t) / reps * 1e3
t = time.perf_counter()
for _ in range(reps):
    m.evaluate(th)
torch.cuda.synchronize()
print(json.dumps({"config": cid, "n": n, "grad_ms": gms, "nll_ms": (time.perf_counter() - t) / reps * 1e3,
                  "grad": [float(v) for v in g], "env": {k: v for k, v in os.environ.items() if k.startswith("VIF_")}}))

"""Whole-evaluation timing (factor + NLL, CUDA events on the library stream) at the config-3 recipe;
for A/B of schedule knobs (VIF_ROUNDS, ...).  Workload cached in /tmp between processes of one call.
  python tools/step_probe.py [n] [steps]"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2507_05064_b200 as p
import vifgen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
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
stream = torch.cuda.current_stream(dev)
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (X, Z, nbr, y)), stream=stream)
th = p.Theta(**td)
for _ in range(3):
    t = m.evaluate(th)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(steps):
    t = m.evaluate(th)
e1.record(stream)
torch.cuda.synchronize()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("VIF_")}, "n": n,
                  "ms_per_eval": e0.elapsed_time(e1) / steps, "nll": t.nll}))

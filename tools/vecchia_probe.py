"""Timing probe: vecchia kernel time, optionally with the Gram / scalar phases skipped
(VIF_DEBUG_VECCHIA), for A/B runs of kernel variants (VIF_VREG_CFG, VIF_VECCHIA_VARIANT).
  python tools/vecchia_probe.py [n] [flags, e.g. 0,1,2]
The workload (config-3 recipe at n points) is cached under /tmp between processes of one call."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2507_05064_b200 as p
import vifgen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
flags = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"]
cache = f"/tmp/vif_probe_c3_{n}.npz"
if os.path.exists(cache):
    z = np.load(cache)
    X, Z, nbr, y = z["X"], z["Z"], z["nbr"], z["y"]
    td = json.loads(str(z["theta"])); td["lengthscale"] = np.array(td["lengthscale"]); th = p.Theta(**td)
else:
    w = vifgen.make_config(3, device="cuda", n=n)
    X, Z, nbr, y = w.X, w.Z, w.nbr, w.y
    th = p.Theta(**w.theta_dict())
    np.savez(cache, X=X, Z=Z, nbr=nbr, y=y, theta=json.dumps({**w.theta_dict(), "lengthscale": [float(v) for v in w.lengthscale]}))
dev = torch.device("cuda")
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (X, Z, nbr, y)))
tag = {k: os.environ[k] for k in os.environ if k.startswith("VIF_")}
m.factor(th)  # warm-up: lazy module loading of the kernels happens at their first launch
try:
    m.nll()
except p.VifError:
    pass
for flag in flags:
    os.environ["VIF_DEBUG_VECCHIA"] = flag
    m.profile(True)
    for k in range(5):
        m.factor(th)
        try:
            t = m.nll()
        except p.VifError:
            t = None
    st, ev = m.stage_times()
    m.profile(False)
    print(json.dumps({"env": tag, "flag": flag, "n": n, "evals": ev,
                      "stages_ms": {k.split(" ")[0]: round(v / max(ev, 1), 3) for k, v in st.items()},
                      "nll": None if t is None else t.nll}))

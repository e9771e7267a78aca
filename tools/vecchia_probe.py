"""Timing probe: vecchia kernel time with the Gram / scalar phases skipped (VIF_DEBUG_VECCHIA)."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2507_05064_b200 as p
import vifgen
w = vifgen.make_config(3, device="cuda", n=int(sys.argv[1]) if len(sys.argv) > 1 else 300000)
dev = torch.device("cuda")
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
th = p.Theta(**w.theta_dict())
for flag in ("0", "1", "2", "3", "0"):
    os.environ["VIF_DEBUG_VECCHIA"] = flag
    m.profile(True)
    for k in range(4):
        m.factor(th)
        try:
            m.nll()
        except p.VifError:
            pass
    st, ev = m.stage_times()
    m.profile(False)
    print(json.dumps({"flag": flag, "vecchia_ms": st[[k for k in st if "vecchia" in k][0]] / max(ev, 1), "evals": ev}))

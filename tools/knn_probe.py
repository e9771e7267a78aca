"""Time vif_neighbors at the config-3 recipe (n points) and compare with the generator's sets."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2507_05064_b200 as p
import vifgen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
t = time.perf_counter()
w = vifgen.make_config(3, device="cuda", n=n)
tg = time.perf_counter() - t
dev = torch.device("cuda")
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)))
th = p.Theta(**w.theta_dict())
g = m.neighbors(th, w.mv)
torch.cuda.synchronize()
t = time.perf_counter()
g = m.neighbors(th, w.mv)
torch.cuda.synchronize()
tk = time.perf_counter() - t
g = g.cpu().numpy()
print(json.dumps({"n": n, "knn_s": tk, "generator_neighbors_s": w.timings["neighbors"], "gen_total_s": tg,
                  "rows_equal_frac": float((g == w.nbr).all(1).mean())}))

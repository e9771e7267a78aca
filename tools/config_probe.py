"""Factor + NLL timing and per-stage breakdown for any BASELINE config recipe (optionally truncated n).
  python tools/config_probe.py <config> [n] [steps]"""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
import paper_2507_05064_b200 as p
import vifgen
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload_flops, FP64_PEAK_TFLOPS
cid = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "full" else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
t = time.perf_counter()
w = vifgen.make_config(cid, device="cuda", n=n)
gen = time.perf_counter() - t
dev = torch.device("cuda")
stream = torch.cuda.current_stream(dev)
m = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y)), stream=stream)
th = p.Theta(**w.theta_dict())
for _ in range(2):
    m.evaluate(th)
m.profile(True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(steps):
    tt = m.evaluate(th)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
st, ev = m.stage_times()
fl = workload_flops(w.nbr, w.m)
stages = {k: v / ev for k, v in st.items()}
names = list(stages)
out = {"config": cid, "n": w.n, "d": w.d, "m": w.m, "mv": w.mv, "family": w.family, "ms_per_eval": ms,
       "points_per_s": w.n / ms * 1e3, "path_tflops": sum(fl.values()) / ms / 1e9,
       "vecchia_tflops": fl["vecchia"] / stages[names[3]] / 1e9, "ufeat_tflops": fl["ufeat"] / stages[names[1]] / 1e9,
       "syrk_tflops": fl["syrk"] / stages[names[4]] / 1e9, "stages_ms": {k.split(" ")[0]: round(v, 3) for k, v in stages.items()},
       "nll": tt.nll, "input_generation_s": gen}
print(json.dumps(out))

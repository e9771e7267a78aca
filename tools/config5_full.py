"""BASELINE config 5 at full size on one B200: n = 4,000,000 uniform on [0,1]^3, Matern 1/2
(sigma^2 = 1, range 0.1), nugget 0.01, m = 1500 kMeans++ inducing points, m_v = 40 correlation-distance
neighbours, random ordering.
  1. inputs from vifgen (its own torch code: kMeans++, the exact d_c brute force, the RFF draw of y); timed;
  2. vif_factor + vif_nll on the GPU: warm-up, then `steps` evaluations with CUDA events (median), stage times;
  3. parity: `rows` sampled rows of U, B, D recomputed one by one by the oracle; invariants at every row;
  4. (optional, --oracle-nll) the oracle's full factor + NLL on the host cores, against the GPU NLL and terms.
Writes one JSON line.  python tools/config5_full.py [--n N] [--steps K] [--rows R] [--oracle-nll]"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import oracle  # noqa: E402
import paper_2507_05064_b200 as p  # noqa: E402
import vifgen  # noqa: E402
from bench import FP64_PEAK_TFLOPS, workload_flops  # noqa: E402
from parity import check_B, check_D, check_terms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--rows", type=int, default=2000)
ap.add_argument("--oracle-nll", action="store_true")
args = ap.parse_args()

out = {"config": 5}
t0 = time.perf_counter()
w = vifgen.make_config(5, device="cuda", n=args.n)
out["input_generation_s"] = {"total": time.perf_counter() - t0, **{k: round(v, 2) for k, v in w.timings.items()}}
out.update(n=w.n, d=w.d, m=w.m, mv=w.mv, family=w.family)
print(json.dumps({"generated": out}), flush=True)
torch.cuda.empty_cache()

dev = torch.device("cuda")
stream = torch.cuda.current_stream(dev)
X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
model = p.VifModel(X, Z, nbr, y, device=dev, stream=stream)
out["workspace_gb"] = model.workspace.numel() / 1e9
th = p.Theta(**w.theta_dict())
B = torch.zeros((w.n, w.mv), dtype=torch.float64, device=dev)
D = torch.zeros(w.n, dtype=torch.float64, device=dev)
model.evaluate(th, B, D)
model.profile(True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
torch.cuda.synchronize()
ev[0].record(stream)
for k in range(args.steps):
    t = model.evaluate(th)
    ev[k + 1].record(stream)
torch.cuda.synchronize()
ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
st, nev = model.stage_times()
model.profile(False)
fl = workload_flops(w.nbr, w.m)
med = statistics.median(ms)
stages = {k: v / max(nev, 1) for k, v in st.items()}
names = list(stages)
out.update(ms_per_eval=med, points_per_s=w.n / med * 1e3, path_tflops=sum(fl.values()) / med / 1e9,
           path_frac=sum(fl.values()) / med / 1e9 / FP64_PEAK_TFLOPS,
           vecchia_tflops=fl["vecchia"] / stages[names[3]] / 1e9, ufeat_tflops=fl["ufeat"] / stages[names[1]] / 1e9,
           syrk_tflops=fl["syrk"] / stages[names[4]] / 1e9,
           stages_ms={k.split(" ")[0]: round(v, 3) for k, v in stages.items()},
           nll=t.nll, logdet_D=t.logdet_D, logdet_M=t.logdet_M, quad=t.quad)
print(json.dumps({"timed": out}), flush=True)

# parity on sampled rows (the oracle recomputes each row from scratch)
rows = np.random.default_rng(5).choice(w.n, args.rows, replace=False)
rows = np.concatenate([rows, [0, 1, 39, 40, 41, w.n - 1]])
Bh, Dh = B.cpu().numpy(), D.cpu().numpy()
t1 = time.perf_counter()
Ur, Br, Dr = oracle.rows(w.X, w.Z, w.nbr, oracle.Theta(**w.theta_dict()), rows, want_U=True)
Ufull = model.U()  # n x m on the device (48 GB at n = 4M)
Ug = Ufull[torch.from_numpy(rows).to(dev)].cpu().numpy()
Cii = np.concatenate([(w.sigma2 + w.nugget - (Ufull[a:a + (1 << 18)] ** 2).sum(1)).cpu().numpy()
                      for a in range(0, w.n, 1 << 18)])
del Ufull
torch.cuda.empty_cache()
check_D(Dh[rows], Dr)
check_B(Bh[rows], Br)
urel = float((np.linalg.norm(Ug - Ur, axis=1) / np.linalg.norm(Ur, axis=1)).max())
assert urel <= 1e-11, urel
out["sampled_rows"] = {"rows": int(len(rows)), "D_max_rel": float(np.max(np.abs(Dh[rows] - Dr) / Dr)),
                       "B_max_rowrel": float(np.max(np.abs(Bh[rows] - Br).max(1) / np.maximum(np.abs(Br).max(1), 1e-3))),
                       "U_max_rowrel": urel, "oracle_s": time.perf_counter() - t1}
out["invariants"] = {"D_ge_nugget": bool(np.all(Dh >= w.nugget * (1 - 1e-12))),
                     "D_le_Cii": bool(np.all(Dh <= Cii * (1 + 1e-10))), "logdet_M_ge_0": t.logdet_M >= 0,
                     "quad_ge_0": t.quad >= 0}
print(json.dumps({"parity_rows": out["sampled_rows"], "invariants": out["invariants"]}), flush=True)
model.close()
del X, Z, nbr, y, B, D
torch.cuda.empty_cache()

if args.oracle_nll:
    t2 = time.perf_counter()
    r = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, oracle.Theta(**w.theta_dict()), want_BD=False)
    out["oracle"] = {"nll": r.nll, "logdet_D": r.logdet_D, "logdet_M": r.logdet_M, "quad": r.quad,
                     "s": time.perf_counter() - t2, "threads": oracle.num_threads()}
    check_terms(t, r.nll, r.logdet_D, r.logdet_M, r.quad)
    out["oracle"]["nll_rel"] = abs(t.nll - r.nll) / abs(r.nll)
print(json.dumps(out), flush=True)

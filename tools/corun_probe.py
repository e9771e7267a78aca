"""Co-run probe: how much does a concurrent U replication slow the factor down on ONE GPU?
A rank of an 8-GPU run receives ~3.6 GB of U rows per evaluation at config 3 while its vecchia rows run.  On one
GPU we replay that traffic beside a full vif_factor + vif_nll (config-3 recipe, n points):
  alone       the evaluation by itself;
  ce_copy     + a 3.6 GB device-to-device cudaMemcpyAsync on a side stream (the driver's D2D memcpy; peer
              copies between GPUs would run on the copy engines);
  sm_copy     + the same bytes moved by an SM kernel (torch's copy kernel, 16 chunks) on a side stream (what
              NCCL's SM-based all-gather kernels need: CTAs on the SMs the vecchia kernel fills).
Reported: evaluation time (events on the library stream), the side copy's time, and both run alone.
VIF_RESERVE_SMS=k (environment) makes the vecchia rows leave k SMs free, as multi-GPU handles do.
  python tools/corun_probe.py [n]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2507_05064_b200 as p  # noqa: E402
import vifgen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
cache = f"/tmp/vif_probe_c3_{n}.npz"
if os.path.exists(cache):
    z = np.load(cache)
    X, Z, nbr, y = z["X"], z["Z"], z["nbr"], z["y"]
    td = json.loads(str(z["theta"]))
    td["lengthscale"] = np.array(td["lengthscale"])
else:
    w = vifgen.make_config(3, device="cuda", n=n)
    X, Z, nbr, y = w.X, w.Z, w.nbr, w.y
    td = {**w.theta_dict(), "lengthscale": [float(v) for v in w.lengthscale]}
    np.savez(cache, X=X, Z=Z, nbr=nbr, y=y, theta=json.dumps(td))
    td["lengthscale"] = np.array(td["lengthscale"])
dev = torch.device("cuda")
main = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev)
model = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (X, Z, nbr, y)), stream=main)
th = p.Theta(**td)
nbytes = int(3.6e9 * n / 1e6)
src = torch.empty(nbytes // 8, dtype=torch.float64, device=dev).normal_()
dst = torch.empty_like(src)


def ev():
    return torch.cuda.Event(enable_timing=True)


def side_copy(kind):
    with torch.cuda.stream(side):
        if kind == "ce_copy":
            dst.copy_(src, non_blocking=True)  # contiguous same-device copy_: cudaMemcpyAsync D2D
        else:
            for a, b in zip(dst.chunk(16), src.chunk(16)):
                b2 = b.view(-1, 2)  # an elementwise kernel (strided view forces the SM copy path)
                a.view(-1, 2)[:, 0].copy_(b2[:, 0])
                a.view(-1, 2)[:, 1].copy_(b2[:, 1])


def timed(kind, reps=3):
    res = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1, s0, s1 = ev(), ev(), ev(), ev()
        if kind != "alone":
            s0.record(side)
            side_copy(kind)
            s1.record(side)
        e0.record(main)
        model.evaluate(th)
        e1.record(main)
        torch.cuda.synchronize()
        res.append((e0.elapsed_time(e1), s0.elapsed_time(s1) if kind != "alone" else None))
    return res[-1]


model.evaluate(th)
out = {"n": n, "side_bytes": nbytes, "reserve_sms": os.environ.get("VIF_RESERVE_SMS", "0")}
out["alone_ms"] = timed("alone")[0]
for kind in ("ce_copy", "sm_copy"):
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(side)
    side_copy(kind)
    b.record(side)
    torch.cuda.synchronize()
    out[f"{kind}_alone_ms"] = a.elapsed_time(b)
    out[f"eval_with_{kind}_ms"], out[f"{kind}_beside_eval_ms"] = timed(kind)
print(json.dumps(out))

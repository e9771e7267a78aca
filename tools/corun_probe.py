"""Co-run probe: how much does a concurrent U replication slow the factor down on ONE GPU?
A rank of an 8-GPU run receives ~3.6 GB of U rows per evaluation at config 3 while its vecchia rows run.  On one
GPU we replay that traffic beside a full vif_factor + vif_nll (config-3 recipe, n points):
  alone       the evaluation by itself;
  ce_copy     + a 3.6 GB device-to-device cudaMemcpyAsync on a side stream (the driver's D2D memcpy; peer
              copies between GPUs would run on the copy engines);
  sm_copy     + the same bytes moved by an SM kernel (torch's copy kernel, 16 chunks) on a side stream (what
              NCCL's SM-based all-gather kernels need: CTAs on the SMs the vecchia kernel fills).
Reported: evaluation time (events on the library stream), the side copy's time, and both run alone.
CORUN_PRIORITY=1 puts the side stream at the highest stream priority.
  python tools/corun_probe.py [n]"""
import json
import os
import sys
import time

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
# CORUN_PRIORITY=1: the side stream at the highest priority (the block scheduler then prefers its CTAs as SMs
# free up) -- what the library's communication stream uses
prio = torch.cuda.Stream.priority_range()[1] if os.environ.get("CORUN_PRIORITY") == "1" else 0
side = torch.cuda.Stream(dev, priority=prio)
model = p.VifModel(*(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (X, Z, nbr, y)), stream=main)
th = p.Theta(**td)
nbytes = int(3.6e9 * n / 1e6)
DELAY_MS = float(os.environ.get("CORUN_DELAY_MS", "14"))
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
                torch.mul(b, 1.0, out=a)  # an elementwise SM kernel moving the same bytes


def timed(kind, reps=3):
    """the evaluation is enqueued first; the side copy is enqueued `delay` ms later (host clock), when the
    vecchia rows are running (K1 takes ~10 ms at n = 1M), as a per-round all-gather would be"""
    res = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1, s0, s1 = ev(), ev(), ev(), ev()
        e0.record(main)
        model.factor(th)
        e1.record(main)
        if kind != "alone":
            time.sleep(DELAY_MS * 1e-3)
            s0.record(side)
            side_copy(kind)
            s1.record(side)
        torch.cuda.synchronize()
        model.nll()
        res.append((e0.elapsed_time(e1), s0.elapsed_time(s1) if kind != "alone" else None))
    return res[-1]


model.evaluate(th)
out = {"n": n, "side_bytes": nbytes, "side_priority": prio, "delay_ms": DELAY_MS,
       "note": "factor times (vif_factor only; the copy is enqueued delay_ms after it, during the vecchia rows)"}
out["alone_ms"] = timed("alone")[0]
for kind in ("ce_copy", "sm_copy"):
    for _ in range(2):  # the second one is timed (the first loads the kernels)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(side)
        side_copy(kind)
        b.record(side)
        torch.cuda.synchronize()
    out[f"{kind}_alone_ms"] = a.elapsed_time(b)
    out[f"eval_with_{kind}_ms"], out[f"{kind}_beside_eval_ms"] = timed(kind)
print(json.dumps(out))

"""Time vif_gram's two engines on an n x c matrix (CUDA events, median of reps).  python tools/gram_bench.py [n] [c]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2507_05064_b200 as p  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
c = int(sys.argv[2]) if len(sys.argv) > 2 else 512
W = torch.randn(n, c, dtype=torch.float64, device="cuda")
out = {"n": n, "c": c}
for eng in ("int8", "fp64"):
    ms = []
    for r in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p.vif_gram(W, eng)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    med = statistics.median(ms[1:])
    out[eng + "_ms"] = med
    out[eng + "_tflops"] = n * c * (c + 1) / med / 1e9
print(json.dumps(out))

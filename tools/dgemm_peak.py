"""Measure cuBLAS DGEMM (torch.matmul float64) peak: best-of-10 burst and 4 s sustained."""
import json, time, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); c = a @ b; e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
flops = 2.0 * n ** 3
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(True); e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e1 = torch.cuda.Event(True); e1.record(); e1.synchronize()
sus = e0.elapsed_time(e1) / cnt
print(json.dumps({"bench": "cublas_dgemm", "n": n, "burst_tflops": flops / best / 1e9,
                  "sustained_tflops": flops / sus / 1e9, "iters": cnt}))

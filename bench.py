#!/usr/bin/env python3
"""Benchmark: VIF factor + NLL evaluations, points/s at n = 1M (BASELINE.json configs[2]).

One "step" = one whole pass of the hot path (vif_factor + vif_nll: K_m, L_m^-1, U, all-gather,
per-point residual Vecchia rows, W, SYRK, all-reduce, M Cholesky, NLL) over the n = 1M workload,
with inputs already resident in HBM; theta alternates between the data-generating value and the
range x 1.1 so nothing theta-dependent can be reused across steps.  U (4.1 GB) and W (4.1 GB) are
rewritten every step, far larger than the 126 MB L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl vif|reference]

Multi-GPU: one process per GPU, launched by torchrun -- or by `bench.py --gpus N` itself, which
re-executes under torch.distributed.run when WORLD_SIZE is unset; rows are sharded chunk-cyclically,
U is all-gathered and the Gram all-reduced by NCCL inside libvif; the problem size stays n = 1M
(strong scaling).  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VIF factor+NLL evals: points/s at n=1M (1/2/4/8 B200), % FP64-tensor/HBM roofline"
FP64_PEAK_TFLOPS = 37.1   # measured: tools/microbench_fp64.cu DMMA.8x8x4 register loop (profiles/r01_fp64_peaks.json)
FP64_CUBLAS_TFLOPS = 35.5  # measured: cuBLAS DGEMM 8192^3 (torch.matmul float64)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=None, help="override n (same recipe)")
    ap.add_argument("--impl", default="vif", choices=["vif", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-grad", action="store_true", help="skip the NLL-gradient timing (vif_grad)")
    ap.add_argument("--npred", type=int, default=100000, help="prediction points for the vif_predict timing (0: skip)")
    ap.add_argument("--no-knn", action="store_true", help="skip the vif_neighbors timing")
    ap.add_argument("--la-n", type=int, default=100000,
                    help="points of the VIF-Laplace (Bernoulli) timing, paper recipe P:600 (0: skip)")
    ap.add_argument("--la-ell", type=int, default=50, help="SLQ probe vectors of the VIF-Laplace timing")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU seconds of the oracle sample")
    return ap.parse_args()


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            h = None
            try:
                props = torch.cuda.get_device_properties(device_index)
                bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.nvml, self.h = pynvml, h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nvml, self.h = None, None
            self.error = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.h is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.h is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------ flops
def per_point_flops(s, m):
    """SURVEY 8(d) algorithmic FP64 work per point, split by kernel (FMA = 2, symmetric once)."""
    mv = s - 1
    return {"ufeat": float(m) * m,                                   # A1  U = K L^-T (triangular)
            "vecchia": s * (s + 1.0) * m + s ** 3 / 3.0 + mv ** 2 + 2.0 * mv * m,  # A3 + A4 + A5
            "syrk": (m + 1.0) * (m + 2.0)}                            # A6


def vecchia_executed_flops(nbr, m):
    """FP64 flops the vecchia kernel EXECUTES per launch (k_vecchia.cuh, s <= 32): the Gram on 8 x 8 DMMA tiles of
    the RB = ceil(s / 8) row blocks (RB (RB + 1) / 2 tiles x 64 entries x mk, the padding included), the Cholesky of
    the padded 8 RB rows, the back substitution and the W row over the ld columns -- against the algorithmic
    count of per_point_flops, which counts only the s (s + 1) / 2 needed Gram entries"""
    mk = -(-m // 8) * 8
    ld = -(-(mk + 1) // 8) * 8
    s = (nbr >= 0).sum(1).astype(np.float64) + 1.0 if nbr.shape[1] > 0 else np.ones(nbr.shape[0])
    rb = np.ceil(s / 8.0)
    sp = 8.0 * rb
    gram = rb * (rb + 1) / 2 * 64 * mk * 2.0
    chol = sp ** 3 / 3.0
    solve = (s - 1) ** 2
    wrow = 2.0 * s * ld
    return float(np.sum(gram + chol + solve + wrow))


INT8_PEAK_TOPS = 2 * 1665.1  # MEASURED_PEAKS.json bf16_tflops (burst) x the guide's nominal int8 : bf16 ratio of 2


def syrk_int8_ops(n, m):
    """int8 tensor-core ops (2 per MAC) the K4 Gram executes on the integer-slice engine (k_ozaki.cu): 28 digit
    products per (128 x 64 tile, row) over the tiles touching the lower triangle of the ld x ld Gram"""
    ld = -(-(((m + 7) // 8) * 8 + 1) // 8) * 8
    nI, nJ = -(-ld // 128), -(-ld // 64)
    tiles = sum(min(2 * i + 2, nJ) for i in range(nI))
    nrp = -(-n // 64) * 64
    return 2.0 * 28 * nrp * tiles * 128 * 64


def ufeat_int8_ops(n, m):
    """int8 tensor-core ops (2 per MAC) of the K1 GEMM on the integer-slice engine (k_ozaki.cu oz_gemm_kernel): per
    128-row block, 64-column tiles J with the triangular k range min(kb, 2J + 2) blocks of 32, 28 digit products each"""
    mk = -(-m // 8) * 8
    kb, nJ = -(-mk // 32), -(-mk // 64)
    kblocks = sum(min(kb, 2 * J + 2) for J in range(nJ))
    return 2.0 * 28 * (-(-n // 128)) * kblocks * 128 * 64 * 32


def workload_flops(nbr, m):
    s = (nbr >= 0).sum(1).astype(np.float64) + 1.0 if nbr.shape[1] > 0 else np.ones(nbr.shape[0])
    f = per_point_flops(s, m)
    return {k: float(np.sum(v)) if np.ndim(v) else float(v) * len(s) for k, v in f.items()}


def describe(w, cid):
    return {"workload": f"config{cid}: n={w.n}, d={w.d}, {w.family}, m={w.m} inducing, m_v={w.mv}, "
                        f"nugget={w.nugget}, random ordering, correlation-distance neighbours",
            "n": w.n, "d": w.d, "m": w.m, "mv": w.mv, "family": w.family,
            "l2": "inputs > L2: U and W (n x 512 fp64 = 4.1 GB each) rewritten every step",
            "theta": "alternating data-generating theta and range x 1.1"}


def thetas(w):
    t0 = w.theta_dict()
    t1 = w.theta_dict()
    t1["lengthscale"] = t1["lengthscale"] * 1.1
    return t0, t1


# ------------------------------------------------------------------------------------ CPU oracle
def cpu_oracle_sample(w, target_s):
    """Time the oracle (as it stands) on a prefix of the same workload: X[:ns], nbr[:ns] (neighbours are
    predecessors, so a prefix is self-contained), same Z, theta, m, m_v.  Returns (points/s, cores, sample, s)."""
    import oracle
    th = oracle.Theta(**w.theta_dict())
    ns = min(w.n, 4000)
    t = time.perf_counter()
    oracle.factor_nll(w.X[:ns], w.Z, w.nbr[:ns], w.y[:ns], th, want_BD=False)
    dt = time.perf_counter() - t
    ns2 = int(min(w.n, max(ns, ns * target_s / max(dt, 1e-3))))
    t = time.perf_counter()
    oracle.factor_nll(w.X[:ns2], w.Z, w.nbr[:ns2], w.y[:ns2], th, want_BD=False)
    dt2 = time.perf_counter() - t
    return ns2 / dt2, oracle.num_threads(), ns2, dt2


_ONE_THREAD = r'''
import json, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle
z = np.load(sys.argv[2])
th = oracle.Theta(**json.loads(str(z["theta"])))
ns = int(sys.argv[3])
t = time.perf_counter()
oracle.factor_nll(z["X"][:ns], z["Z"], z["nbr"][:ns], z["y"][:ns], th, want_BD=False)
print(json.dumps({"s": time.perf_counter() - t, "threads": oracle.num_threads()}))
'''


def cpu_oracle_one_thread(dev, target_s=6.0):
    """SURVEY 8(d) / BASELINE.md section 3: the oracle on ONE host thread (OMP_NUM_THREADS=1, separate
    process) on a prefix of config 2, a per-core figure beside the all-core cpu_baseline."""
    import tempfile
    import vifgen
    w2 = vifgen.make_config(2, device=str(dev))
    td = {**w2.theta_dict(), "lengthscale": [float(v) for v in w2.lengthscale]}
    path = os.path.join(tempfile.gettempdir(), f"vif_cfg2_{os.getpid()}.npz")
    np.savez(path, X=w2.X, Z=w2.Z, nbr=w2.nbr, y=w2.y, theta=json.dumps(td))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        ns = 2000
        r = json.loads(subprocess.run([sys.executable, "-c", _ONE_THREAD, ROOT, path, str(ns)], env=env, check=True,
                                      capture_output=True, text=True).stdout.strip().splitlines()[-1])
        ns = int(min(w2.n, max(ns, ns * target_s / max(r["s"], 1e-3))))
        r = json.loads(subprocess.run([sys.executable, "-c", _ONE_THREAD, ROOT, path, str(ns)], env=env, check=True,
                                      capture_output=True, text=True).stdout.strip().splitlines()[-1])
    finally:
        os.remove(path)
    fl = sum(workload_flops(w2.nbr[:ns], w2.m).values())
    return {"value": ns / r["s"], "unit": "points/s", "cores": r["threads"], "kind": "oracle",
            "gflops": fl / r["s"] / 1e9,
            "sample": f"oracle (C, OMP_NUM_THREADS=1) on the first {ns} points of config 2 (n = 100k, m = 200, "
                      f"m_v = 20), {r['s']:.1f} s"}


def grad_flops(nbr, m, d, ld):
    """FP64 work of one vif_grad as this library organises it (FMA = 2): the factor
     + Gamma = W (2Q) (2 n ld^2) + T = R L_m^{-1} (n m^2, triangular) + G2 = R^T U (2 n m^2) + the
    gathered dots, adjoint rows and R scatter (~10 s m per point) + per kernel parameter the s(s-1)/2 point-pass
    derivative evaluations and the n m fused dK evaluations contracted with T (2 n m).  Not a lower bound: the
    method's minimum for the gradient is not fixed by the paper."""
    n = nbr.shape[0]
    s = (nbr >= 0).sum(1).astype(np.float64) + 1.0 if nbr.shape[1] > 0 else np.ones(n)
    f = sum(workload_flops(nbr, m).values())
    dense = 2.0 * n * ld * ld + n * float(m) * m + 2.0 * n * float(m) * m
    gathers = float(np.sum(10.0 * s * m))
    per_param = (d + 1) * (2.0 * n * m)
    return {"total": f + dense + gathers + per_param, "factor": f, "dense_contractions": dense, "gathers": gathers,
            "per_parameter": per_param}


# ------------------------------------------------------------------------------------ main
def relaunch_multi_gpu(args):
    """`python bench.py --gpus N` outside torchrun: start N ranks (one process per GPU) through
    torch.distributed.run on this node and return its exit code; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + (os.getpid() % 1000)),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_multi_gpu(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    import vifgen
    cid = args.config

    # ---------------- input generation (timed separately, rank 0, broadcast) ----------------
    t_gen = time.perf_counter()
    if rank == 0:
        w = vifgen.make_config(cid, device=str(dev), n=args.n)
    else:
        w = None
    gen_s = time.perf_counter() - t_gen

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, w, cid, world, gen_s)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    import __graft_entry__
    __graft_entry__.build()
    import paper_2507_05064_b200 as vp

    if world > 1:
        meta = [None]
        if rank == 0:
            meta = [dict(n=w.n, d=w.d, m=w.m, mv=w.mv, theta=w.theta_dict(), name=w.name, timings=w.timings)]
        dist.broadcast_object_list(meta, src=0)
        meta = meta[0]
        if rank == 0:
            X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
        else:
            X = torch.empty((meta["n"], meta["d"]), dtype=torch.float64, device=dev)
            Z = torch.empty((meta["m"], meta["d"]), dtype=torch.float64, device=dev)
            nbr = torch.empty((meta["n"], meta["mv"]), dtype=torch.int32, device=dev)
            y = torch.empty(meta["n"], dtype=torch.float64, device=dev)
        for t in (X, Z, nbr, y):
            dist.broadcast(t, src=0)
        if rank != 0:
            th = meta["theta"]
            w = vifgen.Workload(meta["name"], X.cpu().numpy(), Z.cpu().numpy(), nbr.cpu().numpy(), y.cpu().numpy(),
                                th["family"], th["sigma2"], np.asarray(th["lengthscale"]), th["nugget"], th["jitter"],
                                meta["timings"])
        uid = [vp.vif_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        nccl_id = uid[0]
    else:
        X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.X, w.Z, w.nbr, w.y))
        nccl_id = None

    stream = torch.cuda.current_stream(dev)
    t_create = time.perf_counter()
    model = vp.VifModel(X, Z, nbr, y, rank=rank, world=world, nccl_id=nccl_id, device=dev, stream=stream)
    create_s = time.perf_counter() - t_create
    th = [vp.Theta(**t) for t in thetas(w)]

    def step(k):
        model.factor(th[k % 2])
        return model.nll()

    for k in range(args.warmup):
        step(k)
    launches_per_step = model.launch_count()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- timed region (device events on the library's stream) ----------------
    model.profile(True)
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with sampler:
        ev[0].record(stream)
        last = None
        for k in range(args.steps):
            last = step(k)
            ev[k + 1].record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    ms = statistics.median(step_ms)          # median of >= 10 steps
    ms_mean = ev[0].elapsed_time(ev[-1]) / args.steps
    stages, nev = model.stage_times()
    model.profile(False)
    ms_t = torch.tensor([ms, ms_mean], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max, ms_mean_max = float(ms_t[0].item()), float(ms_t[1].item())

    # ---------------- end-to-end through the public API with HOST buffers ----------------
    hX, hZ, hnbr, hy = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (w.X, w.Z, w.nbr, w.y))
    h2d = sum(t.numel() * t.element_size() for t in (hX, hZ, hnbr, hy))
    d2h = 4 * 8 + 8  # vif_terms (4 doubles + bad_row) read back by vif_nll
    e2e_steps = max(3, min(args.steps, 10))

    def e2e_run(nsteps):
        # pipelined through the public API: step k's inputs are staged (copied from pinned host memory
        # into the second input slot, order sorted, on the library's copy stream) while step k-1
        # computes; vif_factor swaps them in after their copies; vif_nll reads the terms back
        model.stage_data(hX, hZ, hnbr, hy)
        for k in range(nsteps):
            model.factor(th[k % 2])
            if k + 1 < nsteps:
                model.stage_data(hX, hZ, hnbr, hy)
            model.nll()

    e2e_run(2)
    barrier()
    torch.cuda.synchronize(dev)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_run(e2e_steps)
    f1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_ms = torch.tensor([f0.elapsed_time(f1) / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # ---------------- NLL gradient (vif_grad, single GPU): reported beside the headline ----------------
    grad = None
    if world == 1 and not args.no_grad and w.mv <= 31:
        model.grad(th[0])
        g_steps = 3
        torch.cuda.synchronize(dev)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for k in range(g_steps):
            gterms, gvec = model.grad(th[k % 2])
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gms = g0.elapsed_time(g1) / g_steps
        gf = grad_flops(w.nbr, w.m, w.d, (((w.m + 7) // 8 * 8 + 1) + 7) // 8 * 8)
        grad = {"ms_per_eval": gms, "points_per_s": w.n / (gms * 1e-3), "params": len(gvec),
                "ratio_to_evaluation": gms / ms_max,
                "roofline": {"bound": "tensor", "flops_per_eval": gf, "achieved": gf["total"] / (gms * 1e-3) / 1e12,
                             "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                             "frac": gf["total"] / (gms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                             "note": "flops of the library's gradient algorithm (bench.grad_flops), whole call"},
                "grad_at_theta1": [float(x) for x in gvec],
                "note": "vif_grad: factor + NLL + d+2 partial derivatives (sigma_1^2, lambda_1..d, sigma^2; "
                        "P:126-133, App. A), device events around the synchronous calls"}

    # ---------------- predictive means (vif_predict, single GPU) ----------------
    pred = None
    if world == 1 and args.npred > 0:
        t_pg = time.perf_counter()
        Xp, nbrp = vifgen.make_prediction(w, args.npred, x="normal" if cid == 4 else "uniform", device=str(dev))
        pgen = time.perf_counter() - t_pg
        Xp_d, nbrp_d = torch.from_numpy(Xp).to(dev), torch.from_numpy(nbrp).to(dev)
        model.predict(th[0], Xp_d, nbrp_d, want_var=True)
        p_steps = 3
        torch.cuda.synchronize(dev)
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for k in range(p_steps):
            mu, var = model.predict(th[k % 2], Xp_d, nbrp_d, want_var=True)
        q1.record(stream)
        torch.cuda.synchronize(dev)
        pms = q0.elapsed_time(q1) / p_steps
        pred = {"ms_per_call": pms, "npred": args.npred,
                "note": "vif_predict: factor + NLL at theta (training, n points) + prediction features + "
                        "Vecchia rows of the prediction points + means and variances (Prop. 1, P:137-152; "
                        "App. C.1); "
                        f"prediction inputs and their d_c neighbours generated in {pgen:.1f} s (not timed)",
                "mu_mean": float(mu.mean().item()), "var_mean": float(var.mean().item())}

    # ---------------- correlation-distance neighbour search (vif_neighbors, single GPU) ----------------
    knn = None
    if world == 1 and not args.no_knn:
        torch.cuda.synchronize(dev)
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        g = model.neighbors(th[0], w.mv)
        k1.record(stream)
        torch.cuda.synchronize(dev)
        ks = k0.elapsed_time(k1) * 1e-3
        same = float((g.cpu().numpy() == w.nbr).all(1).mean())
        knn = {"s": ks, "rows_equal_to_generator": same, "generator_s": w.timings.get("neighbors"),
               "tflops": w.n * (w.n - 1) / 2 * w.m * 2 / ks / 1e12,
               "note": "vif_neighbors: exact d_c neighbour sets (P:499-513) by brute force (n^2 m / 2 FMA), the Gram "
                       "blocks as int8 digit-slice products on tcgen05 (reading c18; tflops = FP64-equivalent); "
                       "generator_s = the torch brute force of the input generator (vifgen) on the same GPU"}
        model.factor(th[0])  # vif_neighbors invalidates the factor; leave the handle evaluated
        model.nll()

    # ---------------- VIF-Laplace, Bernoulli likelihood (vif_la_*, single GPU) ----------------
    lap = None
    if world == 1 and args.la_n > 0:
        lap = run_laplace(args, dev, stream)

    if rank == 0:
        fl = workload_flops(w.nbr, w.m)
        # per-rank share of the row-sharded kernels (strong scaling: each rank does ~1/world of the rows)
        share = 1.0 / world
        stage_avg = {k: v / max(nev, 1) for k, v in stages.items()}
        names = list(stage_avg.keys())
        kern = {"ufeat": names[1], "vecchia": names[3], "syrk": names[4]}
        fl_launch = {k: fl[k] * share for k in kern}
        achieved = {k: fl_launch[k] / (stage_avg[kern[k]] * 1e-3) / 1e12 if stage_avg[kern[k]] > 0 else 0.0
                    for k in kern}
        dom = max(kern, key=lambda k: stage_avg[kern[k]])
        total_flops = sum(fl.values())
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            try:
                tr = json.load(open(tpath))
                traffic = tr.get(f"config{cid}", {}).get(dom)
            except Exception:
                traffic = None
        cpu = None
        if not args.no_cpu_baseline:
            v, cores, ns, dt = cpu_oracle_sample(w, args.cpu_seconds)
            cpu = {"value": v, "unit": "points/s", "cores": cores, "kind": "oracle",
                   "sample": f"oracle (C, OpenMP, {cores} threads) on the first {ns} points of the same workload "
                             f"(same Z, theta, m, m_v; neighbours are predecessors so the prefix is self-contained); "
                             f"{dt:.1f} s",
                   "gflops": sum(workload_flops(w.nbr[:ns], w.m).values()) / dt / 1e9}
            try:
                cpu["one_thread_config2"] = cpu_oracle_one_thread(dev)
            except Exception as e:  # reported, never fatal for the bench line
                cpu["one_thread_config2"] = {"error": str(e)[-300:]}
        out = {
            "metric": METRIC,
            "value": w.n / (ms_max * 1e-3),
            "unit": "points/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "ms_per_step_mean": ms_mean_max,
            "timing": f"median of {args.steps} per-step CUDA-event intervals on the library stream (max over ranks); "
                      f"mean {ms_mean_max:.3f} ms",
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded; BASELINE.json configs recipe, see DESIGN.md)",
            "config": dict(describe(w, cid), parallelism=f"rows chunk-cyclic over {world} GPU(s); U all-gather + "
                                                          f"Gram all-reduce (NCCL)" if world > 1 else "single GPU"),
            "roofline": {"bound": "tensor", "kernel": kern[dom], "achieved": achieved[dom], "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved[dom] / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "peak_source": "measured FP64 DMMA peak on this pool's B200 (tools/microbench_fp64.cu; "
                                        "MEASURED_PEAKS.json has no FP64 entry); cuBLAS DGEMM 35.5",
                         "flops_per_launch": fl_launch[dom], "avg_launch_ms": stage_avg[kern[dom]],
                         "executed": ({"flops_per_launch": vecchia_executed_flops(w.nbr, w.m) * share,
                                       "tflops": vecchia_executed_flops(w.nbr, w.m) * share /
                                       (stage_avg[kern["vecchia"]] * 1e-3) / 1e12,
                                       "frac": vecchia_executed_flops(w.nbr, w.m) * share /
                                       (stage_avg[kern["vecchia"]] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                                       "note": "flops the kernel executes (8 x 8 DMMA tile padding of the s x s "
                                               "Gram, padded Cholesky, W row over ld columns); frac above counts "
                                               "only the algorithmic flops"}
                                      if dom == "vecchia" and w.mv <= 31 else None),
                         "per_kernel": dict({k: {"stage": kern[k], "avg_ms": stage_avg[kern[k]], "tflops": achieved[k],
                                                 "frac": achieved[k] / FP64_PEAK_TFLOPS} for k in kern},
                                            ufeat={"stage": kern["ufeat"], "avg_ms": stage_avg[kern["ufeat"]],
                                                   "tflops": achieved["ufeat"],
                                                   "frac": achieved["ufeat"] / FP64_PEAK_TFLOPS,
                                                   "engine": "FP64 emulated by int8 digit slices on "
                                                             "tcgen05.mma.kind::i8 (k_ozaki.cu): tflops/frac are "
                                                             "FP64-equivalent (algorithmic FP64 flops / time, vs the "
                                                             "DMMA peak)",
                                                   "int8_tops": ufeat_int8_ops(w.n / world, w.m) /
                                                   (stage_avg[kern["ufeat"]] * 1e-3) / 1e12,
                                                   "int8_peak_tops": INT8_PEAK_TOPS,
                                                   "int8_frac": ufeat_int8_ops(w.n / world, w.m) /
                                                   (stage_avg[kern["ufeat"]] * 1e-3) / 1e12 / INT8_PEAK_TOPS,
                                                   "int8_note": "stage time includes kx_slice (the kernel "
                                                                "evaluations written as digit slices, ~2.0 of 5.6 ms "
                                                                "at config 3)"},
                                            syrk={"stage": kern["syrk"], "avg_ms": stage_avg[kern["syrk"]],
                                                  "tflops": achieved["syrk"],
                                                  "frac": achieved["syrk"] / FP64_PEAK_TFLOPS,
                                                  "engine": "FP64 emulated by int8 digit slices on tcgen05.mma.kind::i8 "
                                                            "(k_ozaki.cu): tflops/frac are FP64-equivalent (the "
                                                            "algorithmic FP64 flops / time, vs the DMMA peak)",
                                                  "int8_tops": syrk_int8_ops(w.n / world, w.m) /
                                                  (stage_avg[kern["syrk"]] * 1e-3) / 1e12,
                                                  "int8_peak_tops": INT8_PEAK_TOPS,
                                                  "int8_frac": syrk_int8_ops(w.n / world, w.m) /
                                                  (stage_avg[kern["syrk"]] * 1e-3) / 1e12 / INT8_PEAK_TOPS,
                                                  "int8_note": "stage time includes the digit-slicing pass over W "
                                                               "(~1.4 of 4.8 ms at config 3; the column maxima come "
                                                               "with the vecchia W rows)"}),
                         "contractions_frac": {"U = K(X,Z) L_m^-T (K1)": achieved["ufeat"] / FP64_PEAK_TFLOPS,
                                               "M Gram W^T W (K4)": achieved["syrk"] / FP64_PEAK_TFLOPS,
                                               "north_star_target": 0.6},
                         "path_effective_tflops": total_flops / (ms_max * 1e-3) / 1e12 / 1.0,
                         "path_frac": total_flops / (ms_max * 1e-3) / 1e12 / FP64_PEAK_TFLOPS},
            "cpu_baseline": cpu,
            "e2e": {"value": w.n / (e2e_ms * 1e-3), "unit": "points/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "note": "every step: vif_stage_data from pinned host X, Z, nbr, y (H2D copies + processing-order "
                            "sort on the library's copy stream, overlapping the previous step) + vif_factor + vif_nll "
                            "(terms read back)"},
            "clocks": sampler.summary(),
            "gpu_launches": launches_per_step * args.steps,
            "stages_ms_per_step": stage_avg,
            "nll": last.nll,
            "grad": grad,
            "predict": pred,
            "neighbors": knn,
            "laplace": lap,
            "input_generation_s": {"total": gen_s, **{k: round(v, 3) for k, v in w.timings.items()}},
            "create_s": create_s,
        }
        print(json.dumps(out), flush=True)
    model.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_laplace(args, dev, stream):
    """One L^VIFLA evaluation = vif_la_prepare (latent factor at nugget 0, transposed structure, levels)
    + vif_la_nll (Newton mode with FITC-preconditioned CG, exact quadratic term, SLQ log-det with ell
    probes) on the paper's Laplace recipe (d = 5, ARD Gaussian covariance, lambda = 0.15..0.75,
    binary responses), m = 200 (the paper's best FITC rank k = 200), m_v = 30."""
    import torch
    import paper_2507_05064_b200 as p
    import vifgen
    n, m, mv, ell = args.la_n, 200, 30, args.la_ell
    t0 = time.perf_counter()
    lw = vifgen.make_laplace_workload(n=n, m=m, mv=mv, device=str(dev))
    gen = time.perf_counter() - t0
    X, Z, nbr, y = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (lw.X, lw.Z, lw.nbr, lw.y))
    eps1, eps2 = vifgen.make_probes(n, m, ell)
    e1, e2 = torch.from_numpy(eps1).to(dev), torch.from_numpy(eps2).to(dev)
    lm = p.VifModel(X, Z, nbr, y, device=dev, stream=stream)
    th = p.Theta(**lw.theta_dict())
    tol = 1e-6
    opts = p.LaOpts(max_newton=50, newton_tol=tol, max_cg=1000, cg_tol=tol, nprobe=ell, slq_tol=tol)
    lm.la_prepare(th, nprobe=ell, max_cg=1000)
    lm.la_nll(y, opts, e1, e2)  # warm-up
    reps, times = 2, []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(stream)
        lm.la_prepare(th, nprobe=ell, max_cg=1000)
        t, _ = lm.la_nll(y, opts, e1, e2)
        b.record(stream)
        torch.cuda.synchronize(dev)
        times.append(a.elapsed_time(b))
    ops = {}
    for ncol in (1, ell):
        V = torch.randn(n, ncol, dtype=torch.float64, device=dev) if ncol > 1 else torch.randn(n, dtype=torch.float64, device=dev)
        for op in ("btinv", "binv", "sigma", "sigma_inv"):
            lm.la_apply(op, V)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(3):
                lm.la_apply(op, V)
            b.record(stream)
            torch.cuda.synchronize(dev)
            ops[f"{op}_ncol{ncol}_ms"] = a.elapsed_time(b) / 3
    lm.close()
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        from oracle import laplace as la
        ns = 2000
        sw = vifgen.make_laplace_workload(n=ns, m=50, mv=mv, device=str(dev))
        s1, s2 = vifgen.make_probes(ns, 50, ell)
        c0 = time.perf_counter()
        la.vifla_nll(sw.X, sw.Z, sw.nbr, sw.y, oracle.Theta(**sw.theta_dict()), eps1=s1, eps2=s2, newton_tol=tol,
                     cg_tol=tol, slq_tol=tol)
        cpu = {"s_per_eval": time.perf_counter() - c0, "n": ns, "m": 50, "mv": mv, "ell": ell,
               "note": "oracle/laplace.py (numpy + scipy sparse triangular solves) on n = 2000 of the same recipe"}
    return {"n": n, "d": 5, "m": m, "mv": mv, "ell": ell, "tol": tol, "ms_per_eval": statistics.median(times),
            "points_per_s": n / (statistics.median(times) * 1e-3), "nll": t.nll, "neg_loglik": t.neg_loglik,
            "quad": t.quad, "logdet": t.logdet, "newton_iters": t.newton_iters, "cg_iters": t.cg_iters,
            "slq_iters_max": t.slq_iters_max, "slq_iters_mean": t.slq_iters_mean, "operators": ops,
            "input_generation_s": gen, "cpu_oracle": cpu,
            "note": "vif_la_prepare + vif_la_nll (Bernoulli-logit VIF-Laplace: Newton + FITC-PCG, pcls2; SLQ "
                    "log-det slq_v2 with ell probe vectors; P:224-345, App. FITC); every CG iteration applies "
                    "Sigma_dagger = B^-1 D B^-T + U U^T (two level-scheduled sparse triangular solves, latency-bound "
                    "by the DAG depth) and the FITC solve"}


def run_reference(args, w, cid, world, gen_s):
    """--impl reference: the oracle, as it stands, on the host cores; each step a bounded prefix sample."""
    import oracle
    th = oracle.Theta(**w.theta_dict())
    # size the sample so one step takes ~ (150 s / (steps + warmup)) of CPU time, at most 10 s
    per_step = min(10.0, 150.0 / max(1, args.steps + args.warmup))
    ns = min(w.n, 4000)
    t = time.perf_counter()
    oracle.factor_nll(w.X[:ns], w.Z, w.nbr[:ns], w.y[:ns], th, want_BD=False)
    dt = time.perf_counter() - t
    ns = int(min(w.n, max(ns, ns * per_step / max(dt, 1e-3))))
    for _ in range(args.warmup):
        oracle.factor_nll(w.X[:ns], w.Z, w.nbr[:ns], w.y[:ns], th, want_BD=False)
    t = time.perf_counter()
    for _ in range(args.steps):
        r = oracle.factor_nll(w.X[:ns], w.Z, w.nbr[:ns], w.y[:ns], th, want_BD=False)
    dt = (time.perf_counter() - t) / args.steps
    v = ns / dt
    cores = oracle.num_threads()
    sample = (f"oracle (C, OpenMP, {cores} threads) on the first {ns} of the {w.n} points of the same workload "
              f"(same Z, theta, m, m_v), {dt:.2f} s per step")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; BASELINE.json configs recipe, see DESIGN.md)",
           "config": dict(describe(w, cid), parallelism="CPU oracle (host cores)"),
           "cpu_baseline": {"value": v, "unit": "points/s", "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "nll_sample": r.nll, "input_generation_s": gen_s}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""Build libvif.so in-tree for sm_100a (nvcc, static cudart, NCCL loaded at run time with dlopen)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libvif.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = os.path.join(base, "nccl", "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


def _flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(), "--expt-relaxed-constexpr"]


def _stale(srcs, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + [os.path.join(ROOT, "include", "vif.h")])
    if not force and not _stale(cus + hdrs, LIB):
        return LIB
    jobs = []
    for cu in cus:
        obj = os.path.join(OBJ, os.path.basename(cu)[:-3] + ".o")
        if force or _stale([cu] + hdrs, obj):
            jobs.append((cu, obj))

    def compile_one(job):
        cu, obj = job
        cmd = [NVCC] + _flags() + ["-c", cu, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = obj[:-2] + ".ptxas.log"
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {cu}:\n{r.stderr[-6000:]}")
        return cu

    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for cu in ex.map(compile_one, jobs):
                if verbose:
                    print("compiled", os.path.basename(cu), file=sys.stderr)
    objs = [os.path.join(OBJ, os.path.basename(c)[:-3] + ".o") for c in cus]
    if force or jobs or _stale(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB + ".tmp"] + objs + ["-ldl"]
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

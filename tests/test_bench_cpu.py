"""bench.py host logic (no GPU): the multi-GPU launcher contract and the flop accounting."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """`bench.py --gpus N` without WORLD_SIZE re-executes itself with N ranks through torch.distributed.run
    (one process per GPU, 127.0.0.1 rendezvous) instead of silently benchmarking one GPU."""
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "12"])
    try:
        bench.main()
    except SystemExit as e:
        assert e.code == 0
    assert len(calls) == 1
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "12"]


def test_world_size_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


def test_flop_accounting_matches_survey_table():
    """F per point at config 3 (m = 500, m_v = 30) = 1,038,332 flops (with every point at s = 31)."""
    nbr = np.zeros((10, 30), np.int32)
    f = bench.workload_flops(nbr, 500)
    assert abs(sum(f.values()) / 10 - 1038332) < 1.0
    g = bench.grad_flops(nbr, 500, 2, 512)
    assert g["total"] > sum(f.values())

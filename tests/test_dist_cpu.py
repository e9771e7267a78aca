"""N > 1 host logic on CPU with 2 gloo ranks: the library's chunk-cyclic partition (vif_partition,
host-only C code) tiles the rows exactly once, and summing per-rank partial Grams over the owned rows
(here computed by the oracle, standing in for the GPU kernels) then finishing reproduces the
single-process NLL -- the algebra of the A6/A7 all-reduce step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2507_05064_b200 as p
    import vifgen
    w = vifgen.make_workload(n=1003, d=2, m=12, mv=7, seed=4242, device="cpu")
    rounds, chunk = p.vif_partition(w.n, w.d, w.m, w.mv, rank, world)
    rows = p.owned_rows(w.n, rank, world, rounds, chunk)
    # partition check: every row exactly once across ranks
    lens = [None] * world
    dist.all_gather_object(lens, rows.tolist())
    allr = np.sort(np.concatenate([np.asarray(r, dtype=np.int64) for r in lens]))
    ok_part = bool(np.array_equal(allr, np.arange(w.n)))
    th = oracle.Theta(**w.theta_dict())
    G, v, sums = oracle.partial(w.X, w.Z, w.nbr, w.y, th, rows)
    buf = torch.from_numpy(np.concatenate([G.ravel(), v, sums]))
    dist.all_reduce(buf)
    b = buf.numpy()
    m = w.m
    terms = oracle.finish(w.n, b[:m * m].reshape(m, m), b[m * m:m * m + m], b[m * m + m:])
    full = oracle.factor_nll(w.X, w.Z, w.nbr, w.y, th)
    out[rank] = (ok_part, float(terms[0]), float(full.nll), len(rows))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_partition_and_reduction():
    import __graft_entry__
    __graft_entry__.build()
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]
    for ok_part, nll, ref, nrows in res:
        assert ok_part
        assert nll == pytest.approx(ref, rel=1e-12)
        assert nrows > 0
    assert res[0][1] == res[1][1]  # identical on every rank

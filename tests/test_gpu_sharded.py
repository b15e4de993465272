"""Scenario-sharded solve: two ranks on one GPU exchanging
through the host-staged gloo all-reduce must reproduce the single-GPU solve
and the reference (iterations, objective, controls)."""
import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, case_path

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, N, sigma, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2301_04869_b200 import _native as nat
    from paper_2301_04869_b200.distributed import sharded_context
    p = nat.Problem(case_path(case), N, sigma, 0)
    ctx = sharded_context(p, world, rank, device=0, backend="gloo")
    r = nat.Solver(ctx).solve()
    out[rank] = {"iterations": r["iterations"], "objective": r["objective"],
                 "u": r["u"].tolist(), "status": r["status_name"]}
    dist.destroy_process_group()


@pytest.mark.parametrize("case,N,sigma,world", [("case9", 8, 0.05, 2), ("case118", 4, 0.05, 2),
                                                ("case118", 64, 0.05, 3)])
def test_sharded_solve_matches_single_and_reference(case, N, sigma, world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, N, sigma, out), nprocs=world, join=True)
    ref = json.load(open(os.path.join(GOLDEN, "solves.json")))[f"{case}_N{N}_s{sigma}_seed0"]
    r0 = out[0]
    for r in range(1, world):  # every rank steps identically
        assert out[r]["iterations"] == r0["iterations"]
        assert out[r]["u"] == r0["u"]
    assert r0["status"] == "Optimal"
    assert r0["iterations"] == ref["iterations"]
    assert abs(r0["objective"] - ref["objective"]) <= 1e-6 * abs(ref["objective"])
    u_ref = np.array(ref["u"])
    assert np.abs(np.array(r0["u"]) - u_ref).max() <= 1e-6 * max(1.0, np.abs(u_ref).max())


def test_nccl_path_one_rank(goldens, monkeypatch):
    """The NCCL exchange (dlopen'd libnccl, ncclCommInitRank, ncclAllReduce on
    the engine stream) exercised on one GPU: a one-rank communicator routed
    through every exchange point must leave the solve unchanged."""
    from paper_2301_04869_b200 import _native as nat
    monkeypatch.setenv("BIPM_FORCE_COMM", "1")
    p = nat.Problem(case_path("case118"), 16, 0.05, 0)
    ctx = nat.Context(p, device=0)
    ctx.set_nccl(nat.nccl_unique_id(), 1, 0)
    r = nat.Solver(ctx).solve()
    monkeypatch.delenv("BIPM_FORCE_COMM")
    ref = nat.Solver(nat.Context(p, device=0)).solve()
    assert r["status_name"] == "Optimal"
    assert r["iterations"] == ref["iterations"]
    assert abs(r["objective"] - ref["objective"]) <= 1e-12 * abs(ref["objective"])
    assert np.max(np.abs(r["u"] - ref["u"])) <= 1e-10

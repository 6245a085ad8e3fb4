"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): max-over-ranks timing,
whole-job throughput of the replicas ("replicas only"), and the reference arm's
rank ≠ 0 early exit."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t_local = 10.0 + 5.0 * rank                      # rank 1 is the slow one
    t = bench.max_over_ranks(t_local, world, "cpu")
    v = bench.job_throughput(20000, world, t)
    out[rank] = torch.tensor([t, v], dtype=torch.float64)
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    world = 2
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        t, v = out[r].tolist()
        assert t == 15.0                              # the slowest rank's time on every rank
        assert v == pytest.approx(2 * 20000 / 15e-3)  # units of all ranks / that time


def test_single_rank_is_identity():
    assert bench.max_over_ranks(3.5, 1) == 3.5
    assert bench.job_throughput(100, 1, 1.0) == pytest.approx(1e5)


def test_reference_arm_nonzero_rank_exits_without_work(monkeypatch):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")

    class A:
        warmup, steps, gpus = 3, 2, 2
    assert bench.run_reference(A()) == 0

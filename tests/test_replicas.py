"""The N > 1 path of bench.py (N independent replicas, barrier + max over
ranks) with world_size 2 on CPU over gloo."""
from __future__ import annotations

import os
import socket
import sys

import pytest

from conftest import ROOT


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    from paper_2411_12690_b200.replicas import Ranks, aggregate_throughput
    r = Ranks(backend="gloo")
    r.barrier()
    ms = 100.0 + 50.0 * rank            # rank 1 is the slow one
    m = r.max(ms)
    s = r.sum(1.0)
    q.put((rank, m, s, aggregate_throughput(10000, r.world, m)))
    r.barrier()
    r.close()


def test_two_rank_gloo_replicas():
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, s, v in out:
        assert m == 150.0 and s == 2.0                       # max over ranks / all ranks counted
        assert v == pytest.approx(2 * 10000 / 0.150)          # whole-job blocks/s, slowest rank's time


def test_single_process_is_identity():
    from paper_2411_12690_b200.replicas import Ranks
    r = Ranks()
    assert r.world == 1 and r.max(3.0) == 3.0 and r.sum(2.0) == 2.0

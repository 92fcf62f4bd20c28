"""Replica (multi-GPU) host logic on CPU with gloo, world_size 2 (no data-path collective)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1901_01685_b200.replicas import cells_for_rank, job_throughput


def test_cells_round_robin():
    cells = list(range(11))
    parts = [cells_for_rank(cells, r, 3) for r in range(3)]
    assert sorted(sum(parts, [])) == cells
    assert parts[0] == [0, 3, 6, 9]
    with pytest.raises(ValueError):
        cells_for_rank(cells, 3, 3)


def test_single_process_throughput():
    assert job_throughput(100.0, 2.0) == (50.0, 100.0, 2.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r "solved" (r + 1) systems of 1000 DOF x 4 cycles in (r + 1) seconds
    val, units, secs = job_throughput(4000.0 * (rank + 1), float(rank + 1))
    q.put((rank, val, units, secs))
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, val, units, secs in res:
        assert units == 12000.0 and secs == 2.0 and val == 6000.0

"""Multi-process host logic of the replicas-only scaling (bench.py --gpus N):
world_size 2 over gloo on CPU. Each rank times its own sequence; the job's
time is the max over ranks; no data-path collective is involved."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = bench.max_over_ranks(1.5 + rank, dist)
        bench.barrier(dist)
        # replicas: every rank draws its own seeded sequence (seed offset by rank)
        from paper_1512_05820_b200.problems import elasticity_sequence

        b = next(iter(elasticity_sequence((2, 2, 2), p=1, seed=3 + rank))).A.values
        gathered = [torch.zeros(b.shape[0], dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(b))
        out[rank] = (t, bool(torch.equal(gathered[0], gathered[1])))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_max_over_ranks_and_distinct_replicas():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 2.5        # job time = slowest rank
    assert res[0][1] is False                     # replicas solve different sequences

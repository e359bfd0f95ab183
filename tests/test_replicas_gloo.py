"""Multi-process host logic of the replicas-only scaling (bench.py --gpus N):
world_size 2 over gloo on CPU. Each rank times its own replica of the
sequence; the job's time is the max over ranks; no data-path collective is
involved; rank 0 generates the host arrays once and every rank maps them."""

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


def _worker(rank, world, port, out, shm):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      RK_BENCH_SHM=shm)
    import types

    import numpy as np

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = bench.max_over_ranks(1.5 + rank, dist)
        bench.barrier(dist)
        # replicas: rank 0 writes the seeded sequence once, every rank maps it (C1: one
        # invariant matrix); an affine sequence (C3) instead keeps its two value
        # arrays per rank and forms every system's values on the device
        res = []
        for workload, mapped in (("c1", True), ("c3", False)):
            args = types.SimpleNamespace(workload=workload, grid=4, systems=3)
            specs = bench._shared_host_specs(args, bench.make_sequence(args), rank, world, dist)
            vals = np.concatenate([np.asarray(s.A.values) for s in specs] + [np.asarray(s.b) for s in specs])
            gathered = [torch.zeros(vals.shape[0], dtype=torch.float64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(vals))
            ref = list(bench.make_sequence(args))
            same_as_generator = all(np.array_equal(a.A.values, b.A.values) and np.array_equal(a.b, b.b)
                                    for a, b in zip(specs, ref))
            how = isinstance(specs[0].A.values, np.memmap) if mapped else getattr(specs[0].A, "affine", None) is not None
            res.append((bool(torch.equal(gathered[0], gathered[1])), same_as_generator, bool(how)))
        out[rank] = (t, all(r[0] for r in res), all(r[1] for r in res), all(r[2] for r in res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_max_over_ranks_and_shared_replicas(tmp_path):
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out, str(tmp_path)), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 2.5                # job time = slowest rank
    assert res[0][1] is True                             # both replicas see the same sequence
    assert res[0][2] and res[1][2]                       # ... which is the seeded generator's
    assert res[0][3] and res[1][3]                       # mapped from one host copy / affine parts

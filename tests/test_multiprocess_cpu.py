"""CPU, world_size 2 over gloo: the N>1 plumbing of bench.py — units are sharded with no
data-path collective and the timing is the max over ranks."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = bench.shard_range(4096, rank, world)
    # every rank solves its own systems with the CPU oracle (test infra), no collective on data
    from oracle.pyoracle import Restated
    import numpy as np
    O = Restated()
    rng = np.random.default_rng(rank)
    a = rng.standard_normal((16, 16)) + 16 * np.eye(16)
    b = rng.standard_normal(16)
    y, rep, _ = O.randomized_genp(a, b, "circulant_sign", "right", 0, seed=1, sid=lo)
    t = bench.max_over_ranks(float(rank + 1), dist)
    out[rank] = (lo, hi, t, float(rep[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_timing():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    spans = sorted((v[0], v[1]) for v in res.values())
    assert spans == [(0, 2048), (2048, 4096)]
    assert all(v[2] == 2.0 for v in res.values())  # max over ranks
    assert all(v[3] < 1e-7 for v in res.values())


@pytest.mark.parametrize("total,world", [(4096, 3), (10, 4), (1, 2), (0, 2)])
def test_shard_range_partitions(total, world):
    import bench
    covered = []
    for r in range(world):
        lo, hi = bench.shard_range(total, r, world)
        covered.extend(range(lo, hi))
    assert covered == list(range(total))

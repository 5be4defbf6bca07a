"""CPU, world_size 2 over gloo: the row-sharded range finder's host logic (TSQR of the
sketch, one all_reduce for B; paper_1212_4560_b200/sharded.py) with the per-rank arithmetic
done by numpy + the restated oracle's Gaussian stream (test infrastructure), against the
single-process answer on the whole matrix."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

M, N, R, K = 512, 96, 12, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix():
    rng = np.random.default_rng(11)
    u, _ = np.linalg.qr(rng.standard_normal((M, R)))
    v, _ = np.linalg.qr(rng.standard_normal((N, R)))
    return (u * np.logspace(0, -3, R)) @ v.T + 1e-11 * rng.standard_normal((M, N))


def _qr_positive(y):
    q, r = np.linalg.qr(y)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s, r * s[:, None]


class NumpyOps:
    def __init__(self, oracle, dist):
        self.o, self.dist = oracle, dist

    def shape(self, a):
        return a.shape

    def gaussian(self, m, n, stream):
        return self.o.gaussian_matrix(m, n, stream.seed, stream.stream_id)

    def matmul(self, a, b, trans_a=False):
        return (a.T if trans_a else a) @ b

    def qr_positive(self, y):
        return _qr_positive(y)

    def rows(self, a, lo, hi):
        return a[lo:hi]

    def numerical_rank(self, b, tol):
        s = np.linalg.svd(b, compute_uv=False)
        return int(np.sum(s >= tol * s[0])) if s[0] > 0 else 0, s

    def all_gather_rows(self, r, group):
        import torch
        parts = [torch.empty(r.shape, dtype=torch.float64) for _ in range(group.get_world_size())]
        self.dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(r)))
        return np.concatenate([p.numpy() for p in parts], axis=0)

    def all_reduce_sum(self, b, group):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(b))
        self.dist.all_reduce(t)
        return t.numpy()


def _worker(rank, world, port, out):
    import torch.distributed as dist
    import bench
    from oracle.pyoracle import Restated
    from paper_1212_4560_b200 import RngStream
    from paper_1212_4560_b200.sharded import DistGroup, range_finder_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = _matrix()
    lo, hi = bench.shard_range(M, rank, world)
    sg, rk, q, b = range_finder_sharded(a[lo:hi], K, RngStream(3, 4), 1e-8, DistGroup(dist),
                                        NumpyOps(Restated(), dist))
    out[rank] = (lo, hi, sg, rk, q, b)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_range_finder_matches_single_process():
    from oracle.pyoracle import Restated
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    a = _matrix()
    h = Restated().gaussian_matrix(N, K, 3, 4)
    q1, _ = _qr_positive(a @ h)
    b1 = q1.T @ a
    s1 = np.linalg.svd(b1, compute_uv=False)
    q = np.concatenate([res[r][4] for r in range(world)], axis=0)
    assert [res[r][:2] for r in range(world)] == [(0, M // 2), (M // 2, M)]
    for r in range(world):
        sg, rk, _, b = res[r][2:]
        assert rk == int(np.sum(s1 >= 1e-8 * s1[0]))
        assert np.abs(sg - s1).max() <= 1e-12
        assert np.abs(b - b1).max() <= 1e-12 * np.abs(a).max()
    # Y has R signal columns and K - R at the 1e-11 noise level: the leading columns of the
    # unique positive-diagonal Q are well determined, the trailing ones only span the noise
    assert np.abs(q[:, :R] - q1[:, :R]).max() < 1e-9
    assert np.abs(q.T @ q - np.eye(K)).max() < 1e-13
    y = a @ h
    assert np.linalg.norm(y - q @ (q.T @ y)) <= 1e-13 * np.linalg.norm(y)

"""Row-sharded randomized range finder over torch.distributed.

A (m x n) is row-partitioned across the ranks; each rank holds its block A_g.  The path is
the reference's approx_basis -> qr_positive -> project_onto_basis -> numerical_rank
(lowrank.cpp:67-84, dense_core.cpp:86-115, lowrank.cpp:61-64, dense_core.cpp:161-175) with
the QR done as TSQR and one exchange step for B:

    H     = gaussian_matrix(n, rho+, stream)       every rank draws the same H (no collective)
    Y_g   = A_g H                                  local
    Y_g   = Q_g R_g                                local qr_positive (needs m_g >= rho+)
    S     = [R_0; R_1; ...]                        all_gather of rho+ x rho+ factors
    S     = Q_S R                                  every rank, same bytes -> same Q_S, R
    Q|_g  = Q_g Q_S[g rho+ : (g+1) rho+]           rows of Q = qr_positive(Y) on rank g
    B     = sum_g Q|_g^T A_g                       one all_reduce (rho+ x n)
    rank  = numerical_rank(B, tol)                 every rank

R has a positive diagonal, so Q and R equal the unique qr_positive(Y) up to rounding.  The
per-rank arithmetic goes through `ops`: `CudaOps` (the library's kernels through the C-ABI,
the product path) or any object with the same methods (the CPU tests pass a numpy one).
"""
from __future__ import annotations

from typing import Any, Tuple


class CudaOps:
    """Per-rank pieces on CUDA tensors through librl_b200 (fails loudly without it)."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())

    def empty(self, m: int, n: int):
        return self.torch.empty(m, n, dtype=self.torch.float64, device=self.device)

    def shape(self, a) -> Tuple[int, int]:
        return int(a.shape[0]), int(a.shape[1])

    def gaussian(self, m: int, n: int, stream):
        from . import dev_gaussian_matrix
        h = self.empty(m, n)
        dev_gaussian_matrix(h, 0.0, 1.0, stream)
        return h

    def matmul(self, a, b, trans_a: bool = False):
        from . import dev_gemm
        m = a.shape[1] if trans_a else a.shape[0]
        c = self.empty(m, b.shape[1])
        dev_gemm(a, b, c, trans_a=trans_a)
        return c

    def qr_positive(self, y):
        from . import dev_qr_positive
        m, n = self.shape(y)
        q, r = self.empty(m, n), self.empty(n, n)
        dev_qr_positive(y, q, r)
        return q, r

    def rows(self, a, lo: int, hi: int):
        return a[lo:hi]  # a contiguous row range: a view, no copy

    def numerical_rank(self, b, tol: float):
        from . import dev_numerical_rank
        return dev_numerical_rank(b, tol)

    def all_gather_rows(self, r, group):
        world = group.get_world_size()
        if world == 1:
            return r
        out = self.empty(world * r.shape[0], r.shape[1])
        group.all_gather_into_tensor(out, r)
        return out

    def all_reduce_sum(self, b, group):
        if group.get_world_size() > 1:
            group.all_reduce(b)
        return b


class DistGroup:
    """torch.distributed (default group) behind the two collectives the path uses."""

    def __init__(self, dist=None):
        if dist is None:
            import torch.distributed as dist
        self.dist = dist

    def get_world_size(self) -> int:
        return self.dist.get_world_size() if self.dist.is_initialized() else 1

    def get_rank(self) -> int:
        return self.dist.get_rank() if self.dist.is_initialized() else 0

    def all_gather_into_tensor(self, out, t) -> None:
        self.dist.all_gather_into_tensor(out, t)

    def all_reduce(self, t) -> None:
        self.dist.all_reduce(t)


def range_finder_sharded(a_local: Any, rho_plus: int, stream, rank_tol: float, group=None, ops=None):
    """Rows of Q and all of B, sigma(B), numerical rank for the row-sharded A.

    Returns (sigma, rank, q_local, b).  Every rank gets the same sigma, rank and B.
    """
    group = group if group is not None else DistGroup()
    ops = ops if ops is not None else CudaOps()
    world, me = group.get_world_size(), group.get_rank()
    m_loc, n = ops.shape(a_local)
    if m_loc < rho_plus:
        raise ValueError("range_finder_sharded: every rank needs at least rho_plus rows")
    h = ops.gaussian(n, rho_plus, stream)        # approx_basis, LeftSpace (lowrank.cpp:67-84)
    y = ops.matmul(a_local, h)
    q_g, r_g = ops.qr_positive(y)                # TSQR leaf
    s = ops.all_gather_rows(r_g, group)          # (world rho+) x rho+, rank order
    if world > 1:
        q_s, _ = ops.qr_positive(s)              # TSQR root, identical on every rank
        q = ops.matmul(q_g, ops.rows(q_s, me * rho_plus, (me + 1) * rho_plus))
    else:
        q = q_g
    b = ops.all_reduce_sum(ops.matmul(q, a_local, trans_a=True), group)  # sta = Q^T A (lowrank.cpp:61-64)
    rank, sigma = ops.numerical_rank(b, rank_tol)
    return sigma, rank, q, b

"""Bitwise run-to-run determinism of the GPU path at n = 8192: factor, solve, gemm, rng."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dev = torch.device("cuda", 0)
A = torch.empty(n, n, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(5, 6))
A += 3 * n ** 0.5 * torch.eye(n, dtype=torch.float64, device=dev)
B = torch.empty(n, 16, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(B, 0.0, 1.0, rl.RngStream(5, 7))


def check(name, fn):
    outs = [fn().clone() for _ in range(reps)]
    bad = [i for i in range(1, reps) if not torch.equal(outs[0], outs[i])]
    diff = max((outs[0] - outs[i]).abs().max().item() for i in range(1, reps))
    print(f"{name:12s}: {'DETERMINISTIC' if not bad else 'DIFFERS in runs ' + str(bad)}  max|d| {diff:.3e}", flush=True)


def fac():
    LU = A.clone()
    rl.dev_genp_factor(LU, 0.0)
    return LU


LU0 = fac()


def sol():
    X = B.clone()
    rl.dev_genp_solve(LU0, X)
    return X


def gem():
    C = torch.empty_like(A)
    rl.dev_gemm(A, A, C)
    return C


def rng():
    G = torch.empty_like(A)
    rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(1, 2))
    return G


check("rng", rng)
check("gemm", gem)
check("genp_factor", fac)
check("genp_solve", sol)

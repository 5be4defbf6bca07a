"""Accuracy of the GENP solve vs a float64 reference solve (torch.linalg.solve) on a
diagonally dominant system, and the per-attempt residuals of one randomized_genp call."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nrhs = 16
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) + 2 * n ** 0.5 * torch.eye(
    n, dtype=torch.float64, device="cuda")
B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda", generator=g)
LU = A.clone()
rl.dev_genp_factor(LU, 0.0)
X = B.clone()
rl.dev_genp_solve(LU, X)
Xr = torch.linalg.solve(A, B)
res = ((A @ X - B).norm(dim=0) / B.norm(dim=0)).max().item()
resr = ((A @ Xr - B).norm(dim=0) / B.norm(dim=0)).max().item()
print(f"n={n}: rel dx {((X - Xr).abs().max() / Xr.abs().max()).item():.3e}  residual {res:.3e}  (torch {resr:.3e})")
if n == 8192:
    import bench
    Ac, Bc = bench.make_config3_inputs(torch, torch.device("cuda", 0))
    Xo = torch.empty_like(Bc)
    os.environ["RL_DEBUG"] = "1"
    rep = rl.dev_randomized_genp(Ac, Bc, Xo, rl.MultiplierKind(), rl.MulSide.RIGHT, 0, rl.RngStream(bench.SEED, 11),
                                 skip_raw_arm=True)
    print("config3 attempt", rep.attempt, "residual", rep.residual, "drawn", rep.attempts_drawn)

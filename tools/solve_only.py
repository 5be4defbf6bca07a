"""Time genp_solve alone (n, 16 RHS) for launch lists / ncu captures."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
A = torch.randn(n, n, dtype=torch.float64, device="cuda") + 2 * n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
rl.dev_genp_factor(A, 0.0)
B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda")
for i in range(4):
    X = B.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rl.dev_genp_solve(A, X)
    e1.record()
    torch.cuda.synchronize()
    print(f"solve n={n} nrhs={nrhs}: {e0.elapsed_time(e1):.3f} ms", flush=True)

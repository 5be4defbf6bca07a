"""Time the 8192^2 Gaussian generation alone (for ncu captures)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
G = torch.empty(n, n, dtype=torch.float64, device="cuda")
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(1, 2))
    e1.record()
    torch.cuda.synchronize()
    print(f"gaussian {n}^2: {e0.elapsed_time(e1):.3f} ms", flush=True)

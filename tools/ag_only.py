"""The config-3 A*G DGEMM alone (8192^3), for ncu captures of the dominant kernel."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = 8192
A = torch.empty(n, n, dtype=torch.float64, device="cuda")
G = torch.empty(n, n, dtype=torch.float64, device="cuda")
rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(1, 1))
rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(1, 2))
C = torch.empty_like(A)
for i in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rl.dev_gemm(A, G, C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"A*G 8192^3: {ms:.3f} ms {2 * n ** 3 / ms / 1e9:.2f} TF/s", flush=True)

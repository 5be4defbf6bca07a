"""A·G at 8192^3 through the library GEMM: prints the CUDA-event time and a SHA-256 of the result
(run once with RL_GEMM_NO_TMA=1 and once without: the TMA-fed kernel must return the same bits)."""
import hashlib
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = 8192
dev = torch.device("cuda", 0)
A = torch.empty(n, n, dtype=torch.float64, device=dev)
G = torch.empty_like(A)
C = torch.empty_like(A)
rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(1, 2))
rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(1, 3))
for _ in range(2):
    rl.dev_gemm(A, G, C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    rl.dev_gemm(A, G, C)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"{ms:.3f} ms {2 * n ** 3 / ms / 1e9:.2f} TFLOP/s sha {hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()[:16]}")

"""Config-4 range finder output hashes (Q, B, sigma) — run twice, with and without
RL_GEMM_NO_TMA=1, to show a GEMM-kernel change leaves the bits alone."""
import hashlib
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

m, n, k = 16384, 4096, 72
dev = torch.device("cuda", 0)
A = torch.empty(m, n, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(4, 3))
Q = torch.empty(m, k, dtype=torch.float64, device=dev)
B = torch.empty(k, n, dtype=torch.float64, device=dev)
sg, rank, _ = rl.dev_range_finder(A, k, rl.RngStream(4, 9), 1e-8, Q, B, want_residual=False)
torch.cuda.synchronize()
h = lambda t: hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]  # noqa: E731
print(f"rank {rank} Q {h(Q)} B {h(B)} sigma {hashlib.sha256(sg.tobytes()).hexdigest()[:16]}")

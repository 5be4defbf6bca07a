"""Config 4 at full size (16384 x 4096, rho+ = 72): the fused range finder's time, numerical
rank and ||A - Q B||_F / ||A||_F against SURVEY.md §8(d)'s expectations (rank 72, ~9.7e-7)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

m, n, r, k = 16384, 4096, 64, 72
dev = torch.device("cuda", 0)
g1 = torch.empty(m, r, dtype=torch.float64, device=dev)
g2 = torch.empty(n, r, dtype=torch.float64, device=dev)
E = torch.empty(m, n, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(g1, 0.0, 1.0, rl.RngStream(4, 1))
rl.dev_gaussian_matrix(g2, 0.0, 1.0, rl.RngStream(4, 2))
rl.dev_gaussian_matrix(E, 0.0, 1.0, rl.RngStream(4, 3))
U, _ = torch.linalg.qr(g1)
V, _ = torch.linalg.qr(g2)
sig = torch.logspace(0, -2, r, dtype=torch.float64, device=dev)
A = (U * sig) @ V.T + 1e-10 * E
del E, g1, g2
Q = torch.empty(m, k, dtype=torch.float64, device=dev)
B = torch.empty(k, n, dtype=torch.float64, device=dev)
sg, rank, res = rl.dev_range_finder(A, k, rl.RngStream(4, 9), 1e-8, Q, B)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sg, rank, _ = rl.dev_range_finder(A, k, rl.RngStream(4, 9), 1e-8, Q, B, want_residual=False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
orth = (Q.T @ Q - torch.eye(k, dtype=torch.float64, device=dev)).abs().max().item()
res2 = torch.linalg.matrix_norm(A - Q @ B, ord=2).item() / torch.linalg.matrix_norm(A, ord=2).item()
print(f"C4 16384x4096 rho+=72: {ms:.3f} ms ({1.967e10 / ms / 1e9:.2f} TFLOP/s of 1.967e10 flop), rank(1e-8) {rank}, "
      f"||A-QB||_F/||A||_F {res:.2e}, ||A-QB||_2/||A||_2 {res2:.2e}, ||Q^T Q - I||_max {orth:.1e}, "
      f"sigma(B) {sg[0]:.4f} .. {sg[-1]:.3e}")
if len(sys.argv) > 1 and sys.argv[1] == "timeline":
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        rl.dev_range_finder(A, k, rl.RngStream(4, 9), 1e-8, Q, B, want_residual=False)
        torch.cuda.synchronize()
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA")
    t0 = ks[0][0]
    for st, en, nm in ks:
        nm = nm.replace("void rl::(anonymous namespace)::", "").replace("rl::(anonymous namespace)::", "")
        print(f"{st - t0:9.1f} {en - t0:9.1f} {en - st:8.1f}  {nm[:70]}")

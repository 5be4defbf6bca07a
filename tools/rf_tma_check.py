"""The range finder's skinny products (A·H: N = 72, Q^T A: M = 72) through the TMA kernel: prints
the config-4 range-finder time and SHA-256s of Q and B (run once with RL_GEMM_NO_TMA=1 and once
without: the bits must agree), and checks ragged dev_gemm shapes against torch's fp64 matmul."""
import hashlib
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402

dev = torch.device("cuda", 0)
rl.lib().rl_init(0)
g = torch.Generator(device=dev).manual_seed(3)
worst = 0.0
for (m, n, k, ta) in [(1000, 72, 777, False), (16384, 72, 4096, False), (72, 1000, 777, True),
                      (72, 4096, 16384, True), (333, 70, 2048, False), (70, 333, 2048, True),
                      (4096, 72, 100000 // 16 * 16, False)]:
    a = torch.randn(k, m, dtype=torch.float64, device=dev, generator=g) if ta else \
        torch.randn(m, k, dtype=torch.float64, device=dev, generator=g)
    b = torch.randn(k, n, dtype=torch.float64, device=dev, generator=g)
    c = torch.empty(m, n, dtype=torch.float64, device=dev)
    rl.dev_gemm(a, b, c, trans_a=ta)
    ref = (a.t() if ta else a) @ b
    err = ((c - ref).abs().max() / ref.abs().max()).item()
    worst = max(worst, err)
    print(f"gemm {m}x{n}x{k} ta={ta}: rel err {err:.2e}")
assert worst < 1e-13, worst
A = bench.make_config4_rows(torch, dev, 0, bench.M4)
Q = torch.empty(bench.M4, bench.K4, dtype=torch.float64, device=dev)
B = torch.empty(bench.K4, bench.N4, dtype=torch.float64, device=dev)
for _ in range(3):
    rl.dev_range_finder(A, bench.K4, rl.RngStream(bench.SEED, 64), 1e-8, Q, B, want_residual=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    rl.dev_range_finder(A, bench.K4, rl.RngStream(bench.SEED, 64), 1e-8, Q, B, want_residual=False)
e1.record()
torch.cuda.synchronize()
h = hashlib.sha256(Q.cpu().numpy().tobytes() + B.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"range finder {e0.elapsed_time(e1) / 10:.4f} ms sha {h}")

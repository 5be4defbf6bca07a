"""Circulant right product A C at n = 8192 through the FFT path vs the dense DMMA product
(dev aid): CUDA-event times, HBM GB/s over 2 n^2 8 bytes, max relative difference."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
A = torch.empty(n, n, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(9, 1))
c = torch.from_numpy(rl.rng_draws(rl.RngStream(9, 2), "sign", n)).to(dev)
out = torch.empty_like(A)


def timed(f, reps=10):
    for _ in range(2):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed(lambda: rl.dev_circulant_apply_right(c, A, out))
idx = (torch.arange(n, device=dev)[:, None] - torch.arange(n, device=dev)[None, :]) % n
C = c[idx]
ref = torch.empty_like(A)
ms_d = timed(lambda: rl.dev_gemm(A, C, ref), 3)
print(f"circulant A C n={n}: FFT {ms:.3f} ms ({2 * n * n * 8 / ms / 1e6:.0f} GB/s), dense DMMA {ms_d:.2f} ms; "
      f"max rel diff {float((out - ref).abs().max() / ref.abs().max()):.2e}", flush=True)

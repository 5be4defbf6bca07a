"""genp_factor + genp_solve at n = 8192 (16 right-hand sides): CUDA-event time of each and a SHA-256
of the packed LU and the solution (dev: RL_LU_RESERVE sweeps must leave the bits unchanged)."""
import hashlib
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
rl.lib().rl_init(0)
g = torch.Generator(device=dev).manual_seed(1)
A = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g) + 4 * n ** 0.5 * torch.eye(
    n, dtype=torch.float64, device=dev)
LU = torch.empty_like(A)
X = torch.randn(n, 16, dtype=torch.float64, device=dev, generator=g)
Y = torch.empty_like(X)
tf = ts = 0.0
reps = 5
for r in range(reps + 2):
    LU.copy_(A)
    Y.copy_(X)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    rl.dev_genp_factor(LU, 0.0)
    e[1].record()
    rl.dev_genp_solve(LU, Y)
    e[2].record()
    torch.cuda.synchronize()
    if r >= 2:
        tf += e[0].elapsed_time(e[1]) / reps
        ts += e[1].elapsed_time(e[2]) / reps
h = hashlib.sha256(LU.cpu().numpy().tobytes() + Y.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"n={n} factor {tf:.3f} ms ({2 * n ** 3 / 3 / tf / 1e9:.2f} TFLOP/s) solve {ts:.3f} ms sha {h}", flush=True)

"""Config 5 (n = 16384, 8 RHS): randomized_genp with the Householder-pair, sparse +-1 and
Gaussian right multipliers (raw arm skipped), timed per call, plus the multiplier-stage kernels
from a CUPTI timeline."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nrhs = 8
dev = torch.device("cuda", 0)
A = torch.empty(n, n, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(9, 1))
h = n // 2
P = torch.empty(h, h - 1, dtype=torch.float64, device=dev)
Q = torch.empty(h - 1, h, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(P, 0.0, 1.0, rl.RngStream(9, 2))
rl.dev_gaussian_matrix(Q, 0.0, 1.0, rl.RngStream(9, 3))
A[:h, :h] = P @ Q
del P, Q
Xt = torch.empty(n, nrhs, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(Xt, 0.0, 1.0, rl.RngStream(9, 4))
B = A @ Xt
X = torch.empty_like(B)
for name, tag in (("householder_pair", rl.MultiplierTag.HOUSEHOLDER_PAIR), ("sparse_sign", rl.MultiplierTag.SPARSE_SIGN),
                  ("gaussian", rl.MultiplierTag.GAUSSIAN)):
    kind = rl.MultiplierKind(tag)
    rep = rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(9, 11), skip_raw_arm=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(9, 11), skip_raw_arm=True)
    e1.record()
    torch.cuda.synchronize()
    res = ((A @ X - B).norm(dim=0) / (A.norm() * X.norm(dim=0))).max().item()
    print(f"{name:17s}: {e0.elapsed_time(e1):9.2f} ms  attempts {rep.attempts_drawn}  residual {rep.residual:.2e}  "
          f"bwd {res:.2e}", flush=True)
    if tag != rl.MultiplierTag.GAUSSIAN:
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(9, 11), skip_raw_arm=True)
            torch.cuda.synchronize()
        for e in prof.events():
            nm = e.name
            if e.device_type.name == "CUDA" and ("hh2" in nm or "sparse" in nm):
                print(f"    {(e.time_range.end - e.time_range.start):8.1f} us  {nm.replace('rl::(anonymous namespace)::', '').split('(')[0][:40]}")

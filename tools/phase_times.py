"""Per-phase device times of the config-3 pipeline (CUDA events, warm)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n, nrhs = 8192, 16
dev = torch.device("cuda", 0)
torch.manual_seed(0)
A = torch.randn(n, n, dtype=torch.float64, device=dev) + 4 * n ** 0.5 * torch.eye(n, dtype=torch.float64, device=dev)
B = torch.randn(n, nrhs, dtype=torch.float64, device=dev)
G = torch.empty_like(A)
C = torch.empty_like(A)


def timeit(name, fn, reps=3, flops=None):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    m = min(ms)
    extra = f"  {flops / m / 1e9:.2f} TF/s" if flops else ""
    print(f"{name:28s} {m:9.3f} ms{extra}", flush=True)


timeit("gaussian 8192^2", lambda: rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(1, 2)))
timeit("dgemm A*G", lambda: rl.dev_gemm(A, G, C), flops=2 * n ** 3)
LU = A.clone()


def fac():
    LU.copy_(A)
    rl.dev_genp_factor(LU, 0.0)


timeit("copy + genp_factor", fac, flops=2 * n ** 3 / 3)
X = B.clone()


def sol():
    X.copy_(B)
    rl.dev_genp_solve(LU, X)


timeit("genp_solve 16 rhs", sol)
Y = torch.empty(n, nrhs, dtype=torch.float64, device=dev)
timeit("G*Y (n x 16)", lambda: rl.dev_gemm(G, X, Y), flops=2 * n * n * nrhs)
kind = rl.MultiplierKind()
Xo = torch.empty_like(B)
timeit("randomized_genp (no raw)", lambda: rl.dev_randomized_genp(A, B, Xo, kind, rl.MulSide.RIGHT, 0,
                                                                   rl.RngStream(1, 2), skip_raw_arm=True))
for m in (1024, 2048, 4096):
    Am = A[:m, :m].contiguous()
    L2 = Am.clone()

    def f2():
        L2.copy_(Am)
        rl.dev_genp_factor(L2, 0.0)
    timeit(f"genp_factor n={m}", f2, flops=2 * m ** 3 / 3)

"""Small workloads for ncu captures of the non-DGEMM kernels:
python tools/prof_kernels.py <c4|c2|hh|sparse|circfft|rng|lu|all> [--time]
Each workload runs the product path once warm and once more (the captured launch); with --time it
prints the CUDA-event time of the second run instead (no profiler)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402

dev = torch.device("cuda", 0)
rl.lib().rl_init(0)
which = sys.argv[1]
timing = "--time" in sys.argv


def run(name, fn, reps=2):
    for _ in range(reps - 1):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    if timing:
        print(f"{name}: {e0.elapsed_time(e1):.4f} ms", flush=True)


if which in ("c4", "all"):
    A = bench.make_config4_rows(torch, dev, 0, bench.M4)
    Q = torch.empty(bench.M4, bench.K4, dtype=torch.float64, device=dev)
    B = torch.empty(bench.K4, bench.N4, dtype=torch.float64, device=dev)
    st = rl.RngStream(bench.SEED, 64)
    run("c4 range finder", lambda: rl.dev_range_finder(A, bench.K4, st, 1e-8, Q, B, want_residual=False), reps=3)
    del A, Q, B
if which in ("c2", "all"):
    A2, b2, sids = bench.make_config2_inputs(torch, dev, bench.BATCH2)
    x2 = torch.empty_like(b2)
    kind = rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN)
    run("c2 batched", lambda: rl.dev_randomized_genp_batched(A2, b2, x2, kind, rl.MulSide.RIGHT, 0, bench.SEED, sids),
        reps=3)
    del A2, b2, x2
if which in ("hh", "sparse", "circfft", "all"):
    n = 16384
    A = torch.empty(n, n, dtype=torch.float64, device=dev)
    rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(9, 1))
    out = torch.empty_like(A)
    if which in ("hh", "all"):
        u = torch.from_numpy(rl.rng_draws(rl.RngStream(9, 3), "sign", 2 * n)).to(dev)
        u1, u2 = u[:n].contiguous(), u[n:].contiguous()
        run("hh pair apply", lambda: rl.dev_householder_pair_apply_right(u1, u2, A, out))
    if which in ("sparse", "all"):
        rows_h, signs_h = rl.sparse_sign(n, rl.RngStream(9, 2))
        rows, signs = torch.from_numpy(rows_h).to(dev), torch.from_numpy(signs_h).to(dev)
        run("sparse apply", lambda: rl.dev_sparse_apply_right(rows, signs, A, out))
    if which in ("circfft", "all"):
        m = 8192
        A8 = A[:m, :m].contiguous()
        o8 = torch.empty_like(A8)
        c = torch.from_numpy(rl.rng_draws(rl.RngStream(9, 4), "sign", m)).to(dev)
        run("circulant fft apply", lambda: rl.dev_circulant_apply_right(c, A8, o8))
        del A8, o8
    del A, out
if which in ("rng", "all"):
    G = torch.empty(8192, 8192, dtype=torch.float64, device=dev)
    run("gaussian_matrix 8192^2", lambda: rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(bench.SEED, 11)))
    del G
if which in ("lu", "all"):
    n = 8192
    g = torch.Generator(device=dev).manual_seed(1)
    A = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g) + 4 * n ** 0.5 * torch.eye(
        n, dtype=torch.float64, device=dev)
    LU = torch.empty_like(A)
    X = torch.randn(n, 16, dtype=torch.float64, device=dev, generator=g)

    def lu():
        LU.copy_(A)
        rl.dev_genp_factor(LU, 0.0)
        Y = X.clone()
        rl.dev_genp_solve(LU, Y)
    run("genp factor + solve n=8192", lu)
torch.cuda.synchronize()

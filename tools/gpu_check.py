"""Development sweep on a GPU box: parity spot checks + timings, prints a report.
(Not part of the test suite; tests/ hold the gated checks.)"""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
import paper_1212_4560_b200 as rl  # noqa: E402
from oracle.pyoracle import Restated  # noqa: E402

O = Restated()


def section(name, fn):
    print(f"=== {name}", flush=True)
    t = time.time()
    try:
        fn()
    except Exception:
        traceback.print_exc()
    print(f"    ({time.time() - t:.2f}s)", flush=True)


def peaks():
    print("peaks fp64 TF/s, hbm GB/s:", rl.probe_peaks())


def rng():
    for cnt in (1000, 70000, 3_000_000):
        g = rl.raw_u64(rl.RngStream(5, 9), cnt)
        o = O.raw_u64(5, 9, cnt)
        bad = np.nonzero(g != o)[0]
        print(f"raw_u64 {cnt}: mismatches {len(bad)} first {bad[:5]}")
    for (m, n) in ((3, 5), (257, 255), (2048, 2048)):
        g = rl.gaussian_matrix(m, n, 0.0, 1.0, rl.RngStream(1, 0))
        o = O.gaussian_matrix(m, n, 1, 0)
        eq = np.mean(g == o)
        ulp = np.max(np.abs(g - o) / np.spacing(np.abs(o)))
        print(f"gaussian {m}x{n}: exact {eq * 100:.4f}% max ulp {ulp:.2f}")
    s = rl.rng_draws(rl.RngStream(7, 3), "sign", 100)
    print("signs eq", np.array_equal(s, O.sign_vector(100, 7, 3)))
    u = rl.uniform_matrix(100, 77, rl.RngStream(2, 2))
    print("uniform eq", np.array_equal(u, O.uniform_matrix(100, 77, 2, 2)))
    r1, s1 = rl.sparse_sign(4096, rl.RngStream(3, 4))
    r2, s2 = O.sparse_pm1(4096, 3, 4)
    print("sparse eq", np.array_equal(r1, r2), np.array_equal(s1, s2))


def gemm():
    rng_ = np.random.default_rng(0)
    for (m, k, n) in ((5, 7, 3), (128, 128, 128), (300, 257, 129), (1000, 64, 72), (64, 4096, 72)):
        a = rng_.standard_normal((m, k))
        b = rng_.standard_normal((k, n))
        c = rl.multiply(a, b)
        ref = a @ b
        print(f"gemm {m}x{k}x{n}: rel err {np.abs(c - ref).max() / np.abs(ref).max():.2e}")
    import torch
    for ta, tb in ((False, False), (True, False), (False, True), (True, True)):
        m, n, k = 333, 222, 190
        A = torch.randn(k if ta else m, m if ta else k, dtype=torch.float64, device="cuda")
        B = torch.randn(n if tb else k, k if tb else n, dtype=torch.float64, device="cuda")
        Cm = torch.zeros(m, n, dtype=torch.float64, device="cuda")
        rl.dev_gemm(A, B, Cm, trans_a=ta, trans_b=tb)
        ref = (A.T if ta else A) @ (B.T if tb else B)
        print(f"dev_gemm ta={ta} tb={tb}: {((Cm - ref).abs().max() / ref.abs().max()).item():.2e}")
    n = 8192
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    B = torch.randn(n, n, dtype=torch.float64, device="cuda")
    Cm = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        rl.dev_gemm(A, B, Cm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        rl.dev_gemm(A, B, Cm)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"dgemm 8192^3: {ms:.2f} ms = {2 * n ** 3 / ms / 1e9:.2f} TF/s; "
          f"err {((Cm - A @ B).abs().max() / 8192 ** 0.5).item():.2e}")


def genp():
    rng_ = np.random.default_rng(1)
    for n in (8, 130, 256, 300):
        a = rng_.standard_normal((n, n)) + n * np.eye(n)
        f = rl.genp_factor(a)
        L, U, piv, _ = O.genp_factor(a)
        print(f"genp n={n}: relL {np.abs(f.L - L).max() / np.abs(L).max():.2e} "
              f"relU {np.abs(f.U - U).max() / np.abs(U).max():.2e} piv {np.abs(f.pivot_abs - piv).max():.2e}")
        b = rng_.standard_normal((n, 3))
        x = rl.genp_solve(f, b)
        print(f"   solve resid {np.abs(a @ x - b).max():.2e}")
    try:
        rl.genp_factor(np.array([[0.0, 1.0], [1.0, 0.0]]), 1e-12)
        print("breakdown NOT raised")
    except rl.PivotBreakdown as e:
        print("breakdown raised:", e)


def config1():
    n = 256
    seed = 20260825
    A = O.gaussian_matrix(n, n, seed, 1)
    P = O.gaussian_matrix(128, 127, seed, 2)
    Q = O.gaussian_matrix(127, 128, seed, 3)
    A[:128, :128] = O.matmul(P, Q)
    xt = O.gaussian_matrix(n, 1, seed, 4).ravel()
    b = O.matvec(A, xt)
    for kind in ("gaussian", "circulant_sign", "householder_pair", "sparse_sign"):
        tag = rl.MultiplierTag.__dict__[kind.upper()]
        x, rep = rl.randomized_genp(A, b, rl.MultiplierKind(tag), rl.MulSide.RIGHT, 0, rl.RngStream(seed, 11))
        xo, ro, eo = O.randomized_genp(A, b, kind, "right", 0, seed, 11)
        be = np.linalg.norm(A @ x - b) / (np.linalg.norm(A, 'fro') * np.linalg.norm(x))
        beo = np.linalg.norm(A @ xo - b) / (np.linalg.norm(A, 'fro') * np.linalg.norm(xo))
        print(f"C1 {kind}: rel dx {np.abs(x - xo).max() / np.abs(xo).max():.2e} res {rep.residual:.2e} "
              f"oracle {ro[0]:.2e} raw {rep.raw_residual:.2e}/{ro[1]:.2e} attempt {rep.attempt}/{eo[0]} "
              f"bwd {be:.2e}/{beo:.2e}")


def diag1():
    # where does C1 accuracy go?  factor A*G (oracle G) on GPU vs oracle
    n = 256
    seed = 20260825
    A = O.gaussian_matrix(n, n, seed, 1)
    P = O.gaussian_matrix(128, 127, seed, 2)
    Q = O.gaussian_matrix(127, 128, seed, 3)
    A[:128, :128] = O.matmul(P, Q)
    xt = O.gaussian_matrix(n, 1, seed, 4).ravel()
    b = O.matvec(A, xt)
    G = O.gaussian_matrix(n, n, seed, 11 ^ 0x5000000000000000)
    Gg = rl.gaussian_matrix(n, n, 0.0, 1.0, rl.RngStream(seed, 11 ^ 0x5000000000000000))
    print("G exact frac", np.mean(G == Gg))
    AG = O.matmul(A, G)
    AGg = rl.multiply(A, G)
    print("AG rel", np.abs(AG - AGg).max() / np.abs(AG).max())
    f = rl.genp_factor(AG)
    L, U, piv, w = O.genp_factor(AG)
    print("L rel", np.abs(f.L - L).max() / np.abs(L).max(), "U rel", np.abs(f.U - U).max() / np.abs(U).max())
    z = rl.genp_solve(f, b)
    zo = O.genp_solve_packed(w, b)
    print("z rel", np.abs(z - zo).max() / np.abs(zo).max())
    print("resid gpu", np.linalg.norm(AG @ z - b) / np.linalg.norm(b), "oracle", np.linalg.norm(AG @ zo - b) / np.linalg.norm(b))


def config2():
    batch, n = 512, 64
    seed = 7
    rng_ = np.random.default_rng(3)
    A = rng_.standard_normal((batch, n, n))
    A[:, :32, :32] = rng_.standard_normal((batch, 32, 31)) @ rng_.standard_normal((batch, 31, 32))
    xt = rng_.standard_normal((batch, n))
    b = np.einsum("bij,bj->bi", A, xt)
    sids = np.arange(batch, dtype=np.uint64) * 3 + 1
    x, reps = rl.randomized_genp_batched(A, b, rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN),
                                         rl.MulSide.RIGHT, 0, seed, sids)
    worst, att_mis = 0.0, 0
    for t in range(batch):
        xo, ro, eo = O.randomized_genp(A[t], b[t], "circulant_sign", "right", 0, seed, int(sids[t]))
        worst = max(worst, np.abs(x[t] - xo).max() / np.abs(xo).max())
        att_mis += int(reps[t].attempt != eo[0])
    print(f"C2 batched {batch}: worst rel dx {worst:.2e}, attempt mismatches {att_mis}, "
          f"attempts>0: {sum(r.attempt > 0 for r in reps)}")


def config4():
    import torch
    m, n, r = 2048, 512, 16
    rng_ = np.random.default_rng(5)
    U, _ = np.linalg.qr(rng_.standard_normal((m, r)))
    V, _ = np.linalg.qr(rng_.standard_normal((n, r)))
    A = (U * np.logspace(0, -2, r)) @ V.T + 1e-10 * rng_.standard_normal((m, n))
    k = 24
    Ad = torch.tensor(A, device="cuda")
    Q = torch.empty(m, k, dtype=torch.float64, device="cuda")
    B = torch.empty(k, n, dtype=torch.float64, device="cuda")
    sg, rank, res = rl.dev_range_finder(Ad, k, rl.RngStream(9, 9), 1e-8, Q, B)
    Y = A @ O.gaussian_matrix(n, k, 9, 9)
    qo, ro = O.qr_positive(Y)
    print(f"C4 small: rank {rank} resid {res:.2e}, |Q - Qo| {np.abs(Q.cpu().numpy() - qo).max():.2e}, "
          f"sigma {sg[:3]} .. {sg[-3:]}, oracle sv {O.singular_values(qo.T @ A)[[0, 1, 2, -3, -2, -1]]}")


def big():
    import torch
    n, nrhs = 8192, 16
    torch.manual_seed(0)
    A = torch.randn(n, n, dtype=torch.float64, device="cuda")
    Xt = torch.randn(n, nrhs, dtype=torch.float64, device="cuda")
    B = A @ Xt
    X = torch.empty_like(B)
    kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)
    rep = rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(1, 2), skip_raw_arm=True)
    torch.cuda.synchronize()
    for _ in range(2):
        t = time.time()
        rep = rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(1, 2), skip_raw_arm=True)
        torch.cuda.synchronize()
        dt = time.time() - t
        print(f"n=8192 nrhs=16: {dt * 1e3:.1f} ms -> {1.4704e12 / dt / 1e12:.2f} TF/s; res {rep.residual:.2e}"
              f" attempt {rep.attempt}")
    G = torch.empty(n, n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t = time.time()
    rl.dev_gaussian_matrix(G, 0.0, 1.0, rl.RngStream(1, 3))
    torch.cuda.synchronize()
    print(f"gaussian 8192^2: {(time.time() - t) * 1e3:.2f} ms")
    LU = A.clone()
    torch.cuda.synchronize()
    t = time.time()
    rl.dev_genp_factor(LU, 0.0)
    torch.cuda.synchronize()
    dt = time.time() - t
    print(f"genp_factor 8192: {dt * 1e3:.1f} ms -> {2 * n ** 3 / 3 / dt / 1e12:.2f} TF/s")


for name in sys.argv[1:] or ["peaks", "rng", "gemm", "genp", "diag1", "config1", "config2", "config4", "big"]:
    section(name, globals()[name])
print("launches", rl.launch_count())

"""Config-5 multiplier stages alone (dev aid): A S (sparse +-1) and A H1 H2 (Householder pair)
at n = 16384 through the device C-ABI, CUDA-event timed, with achieved HBM GB/s over the
algorithmic bytes (2 n^2 8 and 3 n^2 8) and a full-size check against torch (bit-exact for S).
python tools/mult_apply.py [n]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda", 0)
A = torch.empty(n, n, dtype=torch.float64, device=dev)
rl.dev_gaussian_matrix(A, 0.0, 1.0, rl.RngStream(9, 1))
out = torch.empty_like(A)
rows_h, signs_h = rl.sparse_sign(n, rl.RngStream(9, 2))
rows, signs = torch.from_numpy(rows_h).to(dev), torch.from_numpy(signs_h).to(dev)
u = torch.from_numpy(rl.rng_draws(rl.RngStream(9, 3), "sign", 2 * n)).to(dev)
u1, u2 = u[:n].contiguous(), u[n:].contiguous()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(f, reps=20):
    for _ in range(3):
        f()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


ms = timed(lambda: rl.dev_sparse_apply_right(rows, signs, A, out))
print(f"sparse  A S   n={n}: {ms:.3f} ms  {2 * n * n * 8 / ms / 1e6:.0f} GB/s", flush=True)
ok = True
for c0 in range(0, n, 2048):
    r, s = rows[c0:c0 + 2048].long(), signs[c0:c0 + 2048]
    v = [A[:, r[:, t]] * s[:, t] for t in range(4)]
    ref = (v[0] + v[1]) + (v[2] + v[3])  # the defined order (oracle rlo_pairwise)
    ok &= bool(torch.equal(ref, out[:, c0:c0 + 2048]))
print("sparse bit-exact vs torch gather:", ok, flush=True)
ms = timed(lambda: rl.dev_householder_pair_apply_right(u1, u2, A, out))
print(f"hh pair A H1 H2 n={n}: {ms:.3f} ms  {2 * n * n * 8 / ms / 1e6:.0f} GB/s (A read once + written once)", flush=True)
t1 = (2.0 / n) * (A @ u1)
t2 = (2.0 / n) * (A @ u2 - t1 * float(u1 @ u2))
ref = A - torch.outer(t1, u1) - torch.outer(t2, u2)
print(f"hh pair max rel diff vs torch: {float((ref - out).abs().max() / ref.abs().max()):.2e}", flush=True)

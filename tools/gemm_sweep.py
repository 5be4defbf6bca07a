import os, sys
sys.path.insert(0, ".")
import torch
import paper_1212_4560_b200 as rl
shapes = [(8192, 8192, 8192), (8064, 8064, 128), (4096, 4096, 128), (2048, 2048, 128), (8064, 128, 128), (128, 8064, 128)]
if len(sys.argv) > 1 and sys.argv[1] == "small":
    shapes = [(7936, 128, 128), (128, 7936, 128), (7936, 256, 256), (256, 7680, 256), (2048, 256, 256),
              (256, 2048, 256), (1024, 1024, 256), (2048, 2048, 256), (4096, 4096, 256), (7680, 7680, 256)]
big = torch.randn(2 * 8192 * 8192 + 1024, dtype=torch.float64, device="cuda")
C = torch.randn(8192 * 8192, dtype=torch.float64, device="cuda")
for (m, n, k) in shapes:
    A = big[: m * k].view(m, k)
    B = big[m * k: m * k + k * n].view(k, n)
    Cm = C[: m * n].view(m, n)
    for _ in range(2):
        rl.dev_gemm(A, B, Cm, alpha=-1.0, beta=1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3 if k > 1024 else 20
    e0.record()
    for _ in range(reps):
        rl.dev_gemm(A, B, Cm, alpha=-1.0, beta=1.0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"force={os.environ.get('RL_GEMM_FORCE','-')} {m}x{n}x{k}: {ms*1e3:9.1f} us {2*m*n*k/ms/1e9:6.2f} TF/s", flush=True)

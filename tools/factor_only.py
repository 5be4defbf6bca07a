import sys, time
sys.path.insert(0, ".")
import torch
import paper_1212_4560_b200 as rl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
A = torch.randn(n, n, dtype=torch.float64, device="cuda") + 4 * n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
LU = A.clone()
rl.dev_genp_factor(LU, 0.0)
torch.cuda.synchronize()
for i in range(3):
    LU.copy_(A)
    torch.cuda.synchronize()
    t = time.perf_counter()
    rl.dev_genp_factor(LU, 0.0)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"n={n}: host enqueue {1e3*(t1-t):.3f} ms, total {1e3*(t2-t):.3f} ms", flush=True)

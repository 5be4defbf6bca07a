import os, sys
sys.path.insert(0, ".")
import torch
import paper_1212_4560_b200 as rl
n = 8192
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
B = torch.randn(n, n, dtype=torch.float64, device="cuda")
C = torch.empty(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    rl.dev_gemm(A, B, C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    rl.dev_gemm(A, B, C)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cfg {os.environ.get('RL_GEMM_CFG')}: {ms:.2f} ms {2*n**3/ms/1e9:.2f} TF/s err {((C - A@B).abs().max()).item():.2e}")

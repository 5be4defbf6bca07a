import sys
sys.path.insert(0, ".")
import torch
import paper_1212_4560_b200 as rl
n = 8192
A = torch.randn(n, n, dtype=torch.float64, device="cuda")
B = torch.randn(n, n, dtype=torch.float64, device="cuda")
C = torch.empty(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    rl.dev_gemm(A, B, C)
torch.cuda.synchronize()
print("ok")

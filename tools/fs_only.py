import sys
sys.path.insert(0, ".")
import torch
import paper_1212_4560_b200 as rl
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.randn(n, n, dtype=torch.float64, device="cuda") + 4 * n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
B = torch.randn(n, 16, dtype=torch.float64, device="cuda")
LU = A.clone()
rl.dev_genp_factor(LU, 0.0)
X = B.clone()
rl.dev_genp_solve(LU, X)
torch.cuda.synchronize()
print("ok")

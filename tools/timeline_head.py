"""First N kernels of a genp_factor timeline (CUPTI via torch.profiler)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
first = int(sys.argv[2]) if len(sys.argv) > 2 else 40
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A = torch.randn(n, n, dtype=torch.float64, device="cuda") + 4 * n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
LU = A.clone()
rl.dev_genp_factor(LU, 0.0)
LU.copy_(A)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rl.dev_genp_factor(LU, 0.0)
    torch.cuda.synchronize()
ks = sorted((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0), e.name)
            for e in prof.events() if e.device_type.name == "CUDA")
t0 = ks[0][0]
for st, en, sid, nm in ks[skip:skip + first]:
    nm = nm.replace("void rl::(anonymous namespace)::", "").replace("rl::(anonymous namespace)::", "")
    print(f"{st - t0:9.1f} {en - t0:9.1f} {en - st:8.1f} s{sid} {nm[:55]}")

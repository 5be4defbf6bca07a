"""Kernel timeline (CUPTI via torch.profiler) of one genp_factor (or other call): prints
per-kernel start/end (us, relative), stream and name for the last N kernels.
usage: python tools/timeline.py factor 8192 [last_n]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "factor"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
last = int(sys.argv[3]) if len(sys.argv) > 3 else 60
A = torch.randn(n, n, dtype=torch.float64, device="cuda") + 4 * n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
LU = A.clone()
rl.dev_genp_factor(LU, 0.0)
torch.cuda.synchronize()
LU.copy_(A)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rl.dev_genp_factor(LU, 0.0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
ks = []
for e in evs:
    st = e.time_range.start
    en = e.time_range.end
    ks.append((st, en, getattr(e, "device_resource_id", None) or getattr(e, "stream", None), e.name))
ks.sort()
t0 = ks[0][0]
print(f"{len(ks)} device events, span {(ks[-1][1] - t0):.1f} us")
for st, en, strm, name in ks[-last:]:
    print(f"{st - t0:10.1f} {en - t0:10.1f} {en - st:8.1f}  s{strm}  {name[:60]}")

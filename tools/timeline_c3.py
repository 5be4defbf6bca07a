"""CUPTI timeline (torch.profiler) of one config-3 randomized_genp call: kernel time by name
and the idle gaps on the main stream (host syncs between phases)."""
import collections
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402

dev = torch.device("cuda", 0)
A, B = bench.make_config3_inputs(torch, dev)
X = torch.empty_like(B)
kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)
step = lambda: rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(bench.SEED, 11),  # noqa: E731
                                      skip_raw_arm=True)
step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep = step()
    torch.cuda.synchronize()
ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA")
t0, t1 = ks[0][0], max(k[1] for k in ks)
print(f"attempts {rep.attempts_drawn}; span {(t1 - t0) / 1e3:.2f} ms, {len(ks)} device events")
by = collections.Counter()
for st, en, nm in ks:
    key = nm.replace("void ", "").replace("rl::(anonymous namespace)::", "").replace("rl::", "")
    by[key.split("(")[0][:60]] += en - st
for nm, us in by.most_common(20):
    print(f"{us / 1e3:9.3f} ms  {nm}")
# device-idle time: union of busy intervals
busy, cur_s, cur_e = 0.0, None, None
for st, en, _ in ks:
    if cur_e is None or st > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = st, en
    else:
        cur_e = max(cur_e, en)
busy += cur_e - cur_s
print(f"device busy {busy / 1e3:.2f} ms of {(t1 - t0) / 1e3:.2f} ms (idle {(t1 - t0 - busy) / 1e3:.2f} ms)")
# the largest idle gaps (device-wide) with the kernels on either side
gaps = []
cur_e, prev = None, None
for st, en, nm in ks:
    if cur_e is not None and st > cur_e:
        gaps.append((st - cur_e, (cur_e - t0) / 1e3, prev, nm))
    if cur_e is None or en > cur_e:
        cur_e, prev = en, nm
for g, at, a_, b_ in sorted(gaps, reverse=True)[:10]:
    print(f"gap {g:8.1f} us at {at:8.3f} ms: {a_.split('(')[0][-40:]} -> {b_.split('(')[0][-40:]}")
if len(sys.argv) > 1 and sys.argv[1] == "head":  # the first device events in order
    for st, en, nm in ks[:12]:
        print(f"{(st - t0) / 1e3:9.3f} {(en - t0) / 1e3:9.3f} ms  {nm.replace('(anonymous namespace)::', '')[:70]}")

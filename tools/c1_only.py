import sys, time
sys.path.insert(0, ".")
import torch, bench
import paper_1212_4560_b200 as rl
class A: warmup=3; steps=20; no_cpu_baseline=True
print(bench.run_config1(torch, rl, torch.device("cuda",0), None, A, 37.0))
if len(sys.argv) > 1 and sys.argv[1] == "timeline":
    from torch.profiler import ProfilerActivity, profile
    n = 256
    dev = torch.device("cuda", 0)
    Am = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, 1, dtype=torch.float64, device=dev)
    x = torch.empty_like(b)
    kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)
    for _ in range(3):
        rl.dev_randomized_genp(Am, b, x, kind, rl.MulSide.RIGHT, 0, rl.RngStream(1, 2), skip_raw_arm=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        rl.dev_randomized_genp(Am, b, x, kind, rl.MulSide.RIGHT, 0, rl.RngStream(1, 2), skip_raw_arm=True)
        torch.cuda.synchronize()
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA")
    t0 = ks[0][0]
    for st, en, nm in ks:
        nm = nm.replace("void rl::(anonymous namespace)::", "").replace("rl::(anonymous namespace)::", "")
        print(f"{st - t0:9.1f} {en - t0:9.1f} {en - st:8.1f}  {nm[:70]}")

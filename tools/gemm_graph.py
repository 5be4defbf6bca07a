"""Device time of small GEMMs without host launch overhead: 20 back-to-back dev_gemm calls
captured in a CUDA graph, replayed and timed with events.  RL_GEMM_FORCE selects a config."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1212_4560_b200 as rl  # noqa: E402

shapes = [(7168, 7168, 512), (5120, 5120, 512), (3072, 3072, 512), (2048, 2048, 512), (7936, 128, 128), (128, 7936, 128), (7936, 256, 256), (256, 7680, 256), (2048, 256, 256),
          (256, 2048, 256), (1024, 1024, 256), (2048, 2048, 256), (4096, 4096, 256), (7680, 7680, 256),
          (512, 512, 256), (768, 768, 256), (128, 128, 256), (128, 128, 128), (128, 1024, 256), (1024, 256, 256),
          (896, 128, 128), (128, 896, 128)]
big = torch.randn(2 * 8192 * 8192 + 1024, dtype=torch.float64, device="cuda")
C = torch.randn(8192 * 8192, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
for (m, n, k) in shapes:
    A = big[: m * k].view(m, k)
    B = big[m * k: m * k + k * n].view(k, n)
    Cm = C[: m * n].view(m, n)
    with torch.cuda.stream(s):
        rl.dev_gemm(A, B, Cm, alpha=-1.0, beta=1.0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        reps = 20
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                rl.dev_gemm(A, B, Cm, alpha=-1.0, beta=1.0)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"force={os.environ.get('RL_GEMM_FORCE', '-')} {m}x{n}x{k}: {us:8.1f} us {2 * m * n * k / us / 1e6:6.2f} TF/s",
          flush=True)

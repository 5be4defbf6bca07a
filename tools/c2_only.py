"""Config 2 batched solve time (dev aid): python tools/c2_only.py"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402
dev = torch.device("cuda", 0)
A2, b2, sids = bench.make_config2_inputs(torch, dev, bench.BATCH2)
x2 = torch.empty_like(b2)
k = rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN)
f = lambda: rl.dev_randomized_genp_batched(A2, b2, x2, k, rl.MulSide.RIGHT, 0, bench.SEED, sids)  # noqa: E731
ms, _ = bench._timed(torch, f, 3, 20, None)
res = torch.bmm(A2, x2.unsqueeze(2)).squeeze(2) - b2
bwd = float((res.norm(dim=1) / (A2.flatten(1).norm(dim=1) * x2.norm(dim=1))).max())
print(f"config2: {ms:.4f} ms per batch, {bench.BATCH2 / ms * 1e3 / 1e6:.3f} M solves/s, bwd max {bwd:.2e}")

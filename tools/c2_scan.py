"""Config-2 batched kernel time against batch size (dev aid): python tools/c2_scan.py"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402
dev = torch.device("cuda", 0)
A2, b2, sids = bench.make_config2_inputs(torch, dev, bench.BATCH2)
k = rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN)
for nb in (1, 148, 296, 592, 888, 1776, 4096):
    A, b, s = A2[:nb].contiguous(), b2[:nb].contiguous(), sids[:nb].contiguous()
    x = torch.empty_like(b)
    f = lambda: rl.dev_randomized_genp_batched(A, b, x, k, rl.MulSide.RIGHT, 0, bench.SEED, s)  # noqa: E731
    ms, _ = bench._timed(torch, f, 3, 20, None)
    print(f"batch {nb:5d}: {ms * 1e3:8.1f} us  ({nb / ms * 1e3 / 1e6:.3f} M solves/s)", flush=True)

"""One warm config-3 step and one warm config-2 batch, for ncu launch lists / captures."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "both"
dev = torch.device("cuda", 0)
if what in ("c3", "both"):
    A, B = bench.make_config3_inputs(torch, dev)
    X = torch.empty_like(B)
    kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)
    for i in range(2):
        torch.cuda.synchronize()
        t = time.time()
        rep = rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(bench.SEED, 11), skip_raw_arm=True)
        torch.cuda.synchronize()
        print(f"c3 step {i}: {(time.time() - t) * 1e3:.1f} ms attempt {rep.attempt} res {rep.residual:.3e}", flush=True)
if what in ("c2", "both"):
    A2, b2, sids = bench.make_config2_inputs(torch, dev, 4096)
    x2 = torch.empty_like(b2)
    ck = rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN)
    for i in range(3):
        torch.cuda.synchronize()
        t = time.time()
        rl.dev_randomized_genp_batched(A2, b2, x2, ck, rl.MulSide.RIGHT, 0, bench.SEED, sids)
        torch.cuda.synchronize()
        print(f"c2 batch {i}: {(time.time() - t) * 1e3:.2f} ms", flush=True)

"""Per-step times of config 3 (randomized_genp, 16 RHS) to expose step-to-step variability."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402

dev = torch.device("cuda", 0)
A, B = bench.make_config3_inputs(torch, dev)
X = torch.empty_like(B)
kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)
ts = []
for i in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(bench.SEED, 11), skip_raw_arm=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    print(f"step {i}: {ts[-1]:.2f} ms attempts {rep.attempts_drawn} accepted {rep.attempt} res {rep.residual:.3e}",
          flush=True)

"""Config-3 step time with and without the nvidia-smi clock sampler running (bench.py's
ClockSampler), to check the sampler does not perturb the timed region."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402

dev = torch.device("cuda", 0)
A, B = bench.make_config3_inputs(torch, dev)
X = torch.empty_like(B)
kind = rl.MultiplierKind(rl.MultiplierTag.GAUSSIAN)


def step():
    return rl.dev_randomized_genp(A, B, X, kind, rl.MulSide.RIGHT, 0, rl.RngStream(bench.SEED, 11), skip_raw_arm=True)


for _ in range(2):
    rep = step()
torch.cuda.synchronize()
for mode in ("plain", "sampler", "plain"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if mode == "sampler":
        cs = bench.ClockSampler(0).__enter__()
    e0.record()
    for _ in range(5):
        rep = step()
    e1.record()
    torch.cuda.synchronize()
    if mode == "sampler":
        cs.__exit__(None, None, None)
    ms = e0.elapsed_time(e1) / 5
    print(f"{mode}: {ms:.2f} ms/step, attempts {rep.attempts_drawn}, {ms / rep.attempts_drawn:.2f} ms/attempt", flush=True)

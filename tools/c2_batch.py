"""Config-2 kernel at several batch sizes (dev aid: contention vs latency per system).
python tools/c2_batch.py 148 888 4096"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1212_4560_b200 as rl  # noqa: E402
dev = torch.device("cuda", 0)
k = rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN)
for b in [int(x) for x in sys.argv[1:]]:
    A2, b2, sids = bench.make_config2_inputs(torch, dev, b)
    x2 = torch.empty_like(b2)
    f = lambda: rl.dev_randomized_genp_batched(A2, b2, x2, k, rl.MulSide.RIGHT, 0, bench.SEED, sids)  # noqa: E731
    ms, _ = bench._timed(torch, f, 3, 10, None)
    print(f"batch {b}: {ms * 1e3:.1f} us per launch", flush=True)

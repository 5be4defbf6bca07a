"""Table-1 sizes through the batched API (dev aid): 100 systems of n in {64, 256, 1024}, MulSide::Left,
refine 0 / 1, circulant +-1 (bench.cpp:107-140's calls); wall time per batched call."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1212_4560_b200 as rl  # noqa: E402

kind = rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN)
for n in (64, 256, 1024):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((100, n, n))
    h = n // 2
    A[:, :h, :h] = rng.standard_normal((100, h, h - 1)) @ rng.standard_normal((100, h - 1, h))
    b = np.einsum("tij,tj->ti", A, rng.standard_normal((100, n)))
    sids = np.arange(100, dtype=np.uint64)
    for refine in (0, 1):
        rl.randomized_genp_batched(A[:4], b[:4], kind, rl.MulSide.LEFT, refine, 7, sids[:4])  # warm
        t0 = time.perf_counter()
        x, reps = rl.randomized_genp_batched(A, b, kind, rl.MulSide.LEFT, refine, 7, sids)
        dt = time.perf_counter() - t0
        print(f"n={n:5d} refine={refine}: {dt * 1e3:8.2f} ms per 100 systems, worst residual "
              f"{max(r.residual for r in reps):.2e}", flush=True)

"""Table 1 of the paper on the GPU: bench::table1_genp (/root/reference/proj/src/bench.cpp:107-140)
over caller-supplied ill-leading-block systems.

For trial t of size index si the reference draws the system from stream (seed, 0x1000000000000 +
base) with base = (si << 40) + 64 t (rnd::illblock_system, input construction — out of scope here:
the caller passes the systems) and solves it twice with randomized_genp(MulSide::Left, refine 0 and
1) on the multiplier stream (seed, 0x2000000000000 + base). Here all trials of one size run as ONE
batched launch per refine (k_batched_circ64's Left path at n = 64; otherwise the single-system path
with the systems spread over the library's host worker pool, as the reference spreads them over
parallel_trials threads: 100 systems of n = 256 in ~21-29 ms, of n = 1024 in ~160 ms — 2-3.5x the
serial order, bitwise the same results), and the samples (rep0.residual, rep1.residual, rep0.raw_residual) are reduced with the
reference's make_stats (bench.cpp:22-42: population standard deviation)."""
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import MulSide, MultiplierKind, MultiplierTag, randomized_genp_batched


@dataclass
class TrialStats:
    n_trials: int = 0
    min: float = 0.0
    max: float = 0.0
    mean: float = 0.0
    std_dev: float = 0.0
    samples: List[float] = field(default_factory=list)


@dataclass
class GenpRow:
    n: int
    refine: int
    stats: TrialStats
    raw_stats: TrialStats


def make_stats(samples) -> TrialStats:
    """bench::make_stats (bench.cpp:22-42), the same sequential sums."""
    samples = [float(v) for v in samples]
    if not samples:
        raise ValueError("make_stats: empty sample set")
    lo = hi = samples[0]
    total = 0.0
    for v in samples:
        lo = min(lo, v)
        hi = max(hi, v)
        total += v
    mean = total / len(samples)
    ss = 0.0
    for v in samples:
        ss += (v - mean) * (v - mean)
    return TrialStats(len(samples), lo, hi, mean, float(np.sqrt(ss / len(samples))), samples)


def multiplier_streams(si: int, trials: int) -> np.ndarray:
    """stream ids 0x2000000000000 + (si << 40) + 64 t of table1_genp's multiplier draws."""
    return np.array([0x2000000000000 + (si << 40) + 64 * t for t in range(trials)], dtype=np.uint64)


def table1_genp_systems(A, b, seed: int, size_index: int = 0,
                        kind: MultiplierKind = MultiplierKind(MultiplierTag.CIRCULANT_SIGN)) -> List[GenpRow]:
    """The two GenpRows (refine 0, 1) of one size for the systems A (trials x n x n), b (trials x n)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    trials, n = A.shape[0], A.shape[1]
    sids = multiplier_streams(size_index, trials)
    _, rep0 = randomized_genp_batched(A, b, kind, MulSide.LEFT, 0, seed, sids)
    _, rep1 = randomized_genp_batched(A, b, kind, MulSide.LEFT, 1, seed, sids)
    raw = make_stats([r.raw_residual for r in rep0])
    return [GenpRow(n, 0, make_stats([r.residual for r in rep0]), raw),
            GenpRow(n, 1, make_stats([r.residual for r in rep1]), raw)]


def acceptance_criterion1(rows: List[GenpRow]) -> bool:
    """tests/acceptance.cpp:51-73's gates on the rows (the runtime gate excluded)."""
    ok = True
    for r in rows:
        if r.refine == 0:
            ok = ok and r.stats.mean <= 1e-8 and r.stats.max <= 1e-6 and \
                sorted(r.raw_stats.samples)[len(r.raw_stats.samples) // 2] >= 10.0
        else:
            ok = ok and r.stats.mean <= 1e-10
    return ok

"""GPU: the C++ drop-in (include/randla/*.hpp over the C-ABI) passes the reference's own
hot-path test cases, re-hosted in tests/cpp/test_dropin.cpp."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_cpp_dropin_reference_cases():
    exe = os.path.join(ROOT, "paper_1212_4560_b200", "lib", "test_dropin")
    assert os.path.exists(exe), "build() must produce lib/test_dropin"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("offset,count", [(0, 10), (5, 100), (311, 700), (65530, 20), (40000, 70000),
                                          ((1 << 15) - 3, 9), ((1 << 21) + 17, 1000)])
def test_rng_block_offsets(rl, oracle, offset, count):
    lib = rl.lib()
    lib.rl_rng_block.argtypes = [ctypes.c_uint64] * 4 + [np.ctypeslib.ndpointer(np.uint64, flags="C")]
    out = np.empty(count, np.uint64)
    assert lib.rl_rng_block(9, 4, offset, count, out) == 0
    assert np.array_equal(out, oracle.raw_u64(9, 4, offset + count)[offset:])


def test_concurrent_host_threads_bit_identical(rl):
    """The reference drives randomized_genp from parallel_trials worker threads and requires the
    same bits at every thread count (tests/test_bench.cpp:57-73, bench.cpp:63-93). Here 8 host
    threads call the library concurrently (per-thread CUDA streams and workspaces, rl_b200.h) on
    16 illblock-shaped systems of n = 16 .. 256 with mixed multiplier kinds and sides; every
    solution, report and per-column outcome must equal the 1-thread run's bits."""
    from concurrent.futures import ThreadPoolExecutor
    rng = np.random.default_rng(57)
    cases = []
    kinds = [rl.MultiplierTag.CIRCULANT_SIGN, rl.MultiplierTag.GAUSSIAN, rl.MultiplierTag.TOEPLITZ_GAUSSIAN,
             rl.MultiplierTag.UNIFORM_PM1]
    for t in range(16):
        n = [16, 64, 100, 256][t % 4]
        A = rng.standard_normal((n, n))
        h = n // 2
        A[:h, :h] = rng.standard_normal((h, h - 1)) @ rng.standard_normal((h - 1, h))
        b = A @ rng.standard_normal(n)
        side = [rl.MulSide.LEFT, rl.MulSide.RIGHT, rl.MulSide.BOTH][t % 3]
        cases.append((A, b, rl.MultiplierKind(kinds[(t // 4) % 4]), side, t % 2, rl.RngStream(99, t)))

    def run(c):
        A, b, kind, side, refine, st = c
        x, rep = rl.randomized_genp(A, b, kind, side, refine, st)
        return x, (rep.residual, rep.raw_residual, rep.pivot_min, rep.pivot_max, rep.attempt, rep.attempts_drawn)

    serial = [run(c) for c in cases]
    for workers in (4, 8):
        with ThreadPoolExecutor(workers) as ex:
            threaded = list(ex.map(run, cases * 2))
        for i, (x, r) in enumerate(threaded):
            xs, rs = serial[i % len(cases)]
            assert np.array_equal(x, xs) and r == rs, (workers, i)

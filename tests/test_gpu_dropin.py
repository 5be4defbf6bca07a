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

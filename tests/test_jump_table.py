"""CPU: the mt19937_64 jump-ahead table (lib/mt64_jump.bin, built by csrc/mt64_jumpgen.cpp)
really advances the engine: XOR of the polynomial's set-bit windows of the word sequence
equals the sequential state at the jump target."""
import os

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
TABLE = os.path.join(ROOT, "paper_1212_4560_b200", "lib", "mt64_jump.bin")
M64 = (1 << 64) - 1


def seq(seed, count):
    x = [0] * (count + 312)
    x[0] = seed
    for i in range(1, 312):
        x[i] = (6364136223846793005 * (x[i - 1] ^ (x[i - 1] >> 62)) + i) & M64
    for k in range(count):
        y = (x[k] & 0xFFFFFFFF80000000) | (x[k + 1] & 0x7FFFFFFF)
        x[k + 312] = x[k + 156] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
    return np.array(x, dtype=np.uint64)


def load():
    if not os.path.exists(TABLE):
        pytest.skip("jump table not built")
    raw = np.fromfile(TABLE, dtype=np.uint8)
    assert raw[:8].tobytes() == b"RLMT64J1"
    words, log2j, n1, n2 = np.frombuffer(raw[8:24].tobytes(), dtype=np.uint32)
    polys = np.frombuffer(raw[24:].tobytes(), dtype=np.uint64).reshape(-1, 312)
    return int(log2j), polys[:n1], polys[n1:n1 + n2]


def apply(poly, x):
    bits = np.nonzero(np.unpackbits(poly.view(np.uint8), bitorder="little")[:19937])[0]
    return np.array([np.bitwise_xor.reduce(x[bits + j]) for j in range(312)], dtype=np.uint64)


@pytest.mark.parametrize("which,index", [("l2", 1), ("l2", 3), ("l1", 0)])
def test_jump_polynomials_advance_the_engine(which, index):
    log2j, l1, l2 = load()
    J = 1 << log2j
    t = (index * J) if which == "l2" else 8
    poly = (l2 if which == "l2" else l1)[index]
    x = seq(987654321, t + 20000 + 400)
    w = apply(poly, x)
    assert np.array_equal(w[1:], x[t + 1:t + 312])
    assert (int(w[0]) ^ int(x[t])) >> 31 == 0  # low 31 bits of word 0 are not engine state

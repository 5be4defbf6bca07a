"""GPU: the multiplier streams (K1) against the reference's draws (golden fixtures) and the
C restatement.  Signs, uniforms, uniform_int and raw outputs are bit-exact everywhere,
including across jump-ahead chunk (2^15) and level-1 (2^21) boundaries.  Gaussians run
glibc 2.39's own log/sincos operation sequences (csrc/glibc_math.cuh) and are bit-exact too."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _streams(golden, kind):
    for key in golden:
        if key.startswith(f"rng/{kind}/"):
            seed, sid = key.split("/")[-1].split("_")
            yield key, int(seed), int(sid)


def test_signs_uniforms_ints_bit_exact_vs_reference(rl, golden):
    for key, seed, sid in _streams(golden, "sign"):
        assert np.array_equal(rl.rng_draws(rl.RngStream(seed, sid), "sign", len(golden[key])), golden[key])
    for key, seed, sid in _streams(golden, "uniform01"):
        assert np.array_equal(rl.rng_draws(rl.RngStream(seed, sid), "uniform01", 64), golden[key])
    for key, seed, sid in _streams(golden, "uniform_pm1"):
        assert np.array_equal(rl.rng_draws(rl.RngStream(seed, sid), "uniform_pm1", 64), golden[key])
    for key, seed, sid in _streams(golden, "uniform_int"):
        got = rl.rng_draws(rl.RngStream(seed, sid), "uniform_int", 64, 0, 16383)
        assert np.array_equal(got.astype(np.int64), golden[key])
    dice = rl.rng_draws(rl.RngStream(7, 5), "uniform_int", 1000, 1, 6)
    assert np.array_equal(dice.astype(np.int64), golden["rng/uniform_int_dice"])
    assert np.array_equal(rl.uniform_matrix(20, 17, rl.RngStream(11, 1)), golden["uniform_matrix/20x17/11_1"])
    col, _ = rl.random_structured(rl.MultiplierKind(rl.MultiplierTag.CIRCULANT_SIGN), 64, 64, rl.RngStream(9, 1))
    assert np.array_equal(col, golden["circulant_sign/64/9_1"])


@pytest.mark.parametrize("count", [1, 311, 312, 313, 4096, 4097, 65536, 65537, (1 << 15) * 3 + 5, (1 << 21) + 12345])
def test_raw_stream_bit_exact_across_jump_boundaries(rl, oracle, count):
    got = rl.raw_u64(rl.RngStream(5, 9), count)
    assert np.array_equal(got, oracle.raw_u64(5, 9, count))


def test_gaussian_golden_and_rate(rl, golden, oracle):
    g = rl.gaussian_matrix(4, 5, 0.0, 1.0, rl.RngStream(11, 0))
    assert np.array_equal(g, golden["gaussian_matrix/4x5/11_0"])
    g = rl.gaussian_matrix(2, 2, 0.0, 1.0, rl.RngStream(1, 0))
    assert g.ravel().tolist() == [0.49698630815925782, 0.47268287749077509, -0.26078844461327677,
                                  0.27389602589300449]
    got = rl.gaussian_matrix(33, 31, 0.5, 2.0, rl.RngStream(3, 9))
    assert np.array_equal(got, golden["gaussian_matrix/33x31/mu_sigma"])
    for key, seed, sid in _streams(golden, "gaussian"):
        got = rl.rng_draws(rl.RngStream(seed, sid), "gaussian", len(golden[key]))
        assert np.array_equal(got, golden[key]), key


def test_gaussian_matrix_large_bit_exact(rl, oracle):
    m = n = 1536  # 2.36 M entries: crosses level-1 jump windows
    got = rl.gaussian_matrix(m, n, 0.0, 1.0, rl.RngStream(20260825, 99))
    ref = oracle.gaussian_matrix(m, n, 20260825, 99)
    assert np.array_equal(got, ref), int(np.sum(got != ref))


def test_new_multiplier_streams_bit_exact(rl, oracle):
    u1, u2 = rl.householder_pair_signs(16384, rl.RngStream(4, 4))
    o1, o2 = oracle.householder_pair_signs(16384, 4, 4)
    assert np.array_equal(u1, o1) and np.array_equal(u2, o2)
    r1, s1 = rl.sparse_sign(16384, rl.RngStream(3, 4))
    r2, s2 = oracle.sparse_pm1(16384, 3, 4)
    assert np.array_equal(r1, r2) and np.array_equal(s1, s2)
    assert all(len(set(row)) == 4 for row in r1[:1000])


def test_householder_sign_reference_multiplier(rl, golden):
    got = rl.householder_sign(16, rl.RngStream(5, 5))
    assert np.array_equal(got, golden["householder_sign/16/5_5"])


def test_determinism_and_stream_independence(rl):
    a = rl.gaussian_matrix(300, 300, 0.0, 1.0, rl.RngStream(7, 3))
    b = rl.gaussian_matrix(300, 300, 0.0, 1.0, rl.RngStream(7, 3))
    c = rl.gaussian_matrix(300, 300, 0.0, 1.0, rl.RngStream(7, 4))
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def _libm_pair(raw0, raw1):
    """Rng::gaussian (random_gen.cpp:46-52) with this host's libm log and sincos."""
    libm = ctypes.CDLL("libm.so.6")
    libm.log.restype = ctypes.c_double
    libm.log.argtypes = [ctypes.c_double]
    libm.sincos.argtypes = [ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    u1 = 1.0 - float(raw0 >> 11) * 2.0 ** -53
    u2 = float(raw1 >> 11) * 2.0 ** -53
    r = np.sqrt(-2.0 * libm.log(u1))
    s, c = ctypes.c_double(), ctypes.c_double()
    libm.sincos(2.0 * np.pi * u2, ctypes.byref(s), ctypes.byref(c))
    return r * c.value, r * s.value


def test_box_muller_edges_match_host_libm(rl):
    """Box-Muller at the ends of its domain: u1 -> 1 (log near 0, the near-one polynomial),
    u1 -> 2^-53, and angles within a few ulp of k pi/2 (glibc's branch points)."""
    raw = []
    for k in list(range(0, 64)) + [1 << 40, (1 << 45) + 3, (1 << 49) - 1]:
        lo = k << 11                              # u1 = 1 - k 2^-53
        hi = ((1 << 53) - 1 - k) << 11            # u1 = (k + 1) 2^-53
        for q in range(5):                        # u2 near q/4 -> angle near q pi/2
            u2 = ((q * (1 << 51) + k - 32) % (1 << 53)) << 11
            raw += [lo, u2, hi, u2]
    raw = np.array(raw, dtype=np.uint64)
    got = rl.box_muller(raw)
    want = np.array([g for i in range(0, raw.size, 2) for g in _libm_pair(int(raw[i]), int(raw[i + 1]))])
    assert np.array_equal(got, want), int(np.sum(got != want))


def test_box_muller_matches_host_libm_2e24(rl):
    """2^24 random pairs: GPU checksums against the host libm's (tests/cpp/bm_libm_check.cpp).
    tools/bm_full.sh runs the same check on 2^30 pairs (profiles/r02_bm_libm_2e30.txt)."""
    exe = os.path.join(os.path.dirname(rl.LIB_PATH), "bm_libm_check")
    r = subprocess.run([exe, "24"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert '"mismatched_chunks": 0' in r.stdout

"""GPU: the rank-search side of lowrank (csrc/lowrank_search.cu) against the reference's own
lowrank.cpp (compiled into oracle/_ref; fixtures in tests/golden): extremal_sv_estimate by the
power method and by Lanczos, cond_probe, nrank_search (both policies, and the transposed wide
case), power_transform — the reference's test cases (tests/test_lowrank.cpp:116-177).

Tolerances: Lanczos with full reorthogonalization runs to the closed Krylov space, so both sides
return the extreme eigenvalues of A^T A to rounding (1e-9 relative); the power method stops when
successive estimates move by <= 1e-4, so the two implementations may stop one iteration apart
(1e-3 relative, the reference test's own bar); ranks are equal; bases agree to GEMM rounding."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case,iters,seed_sid", [("d51", 200, (41, 15)), ("q8", 200, (41, 17)), ("p32", 5000, (41, 19))])
@pytest.mark.parametrize("method", [0, 1])
def test_extremal_sv_estimate(rl, golden, case, iters, seed_sid, method):
    a = np.diag([5.0, 1.0]) if case == "d51" else golden[f"es/{case}"]
    hi, lo = rl.extremal_sv_estimate(a, method, iters, rl.RngStream(*seed_sid))
    want = golden[f"es/{case}/{method}"]
    tol = 1e-9 if method == 1 else 1e-3
    assert abs(hi - want[0]) <= tol * want[0]
    assert abs(lo - want[1]) <= tol * want[0] + (1e-3 * want[1] if method == 0 else 1e-9 * want[1])
    s = np.linalg.svd(a, compute_uv=False)
    assert abs(hi - s[0]) <= 1e-2 * s[0] and abs(lo - s[-1]) <= 1e-2 * s[-1]


def test_extremal_sv_no_convergence(rl):
    # a rank-deficient matrix and a tiny budget: the power method cannot settle (NoConvergence)
    a = np.diag([1.0, 0.5, 0.25, 0.0])
    with pytest.raises(rl.NoConvergence):
        rl.extremal_sv_estimate(a, 0, 3, rl.RngStream(1, 2))


def test_cond_probe(rl, golden):
    assert rl.cond_probe(np.eye(8), 1e6, 0, 500, rl.RngStream(41, 20))
    sig = np.full(8, 1e-10)
    sig[0] = 1.0
    assert not rl.cond_probe(np.diag(sig), 1e6, 0, 500, rl.RngStream(41, 21))
    assert rl.cond_probe(golden["cp/b8"], 1e6, 1, 56, rl.RngStream(41, 24)) == bool(golden["cp/b8/pass"][0])
    assert rl.cond_probe(golden["cp/b9"], 1e6, 1, 56, rl.RngStream(41, 25)) == bool(golden["cp/b9/pass"][0])
    with pytest.raises(rl.InvalidArgument):
        rl.cond_probe(np.eye(3), 1.0, 1, 10, rl.RngStream(1, 1))


@pytest.mark.parametrize("policy", [0, 1])
def test_nrank_search_profile(rl, golden, policy):
    rho, basis = rl.nrank_search(golden["nr/a"], 0, 16, 1e6, policy, rl.RngStream(41, 27))
    ref = golden[f"nr/{policy}/basis"]
    assert rho == int(golden[f"nr/{policy}/rho"][0]) == 8
    assert basis.shape == ref.shape
    assert np.abs(basis - ref).max() <= 1e-12 * np.abs(ref).max()


def test_nrank_search_zero_identity_wide(rl, golden):
    rho, basis = rl.nrank_search(np.zeros((8, 8)), 0, 8, 1e6, 0, rl.RngStream(41, 28))
    assert rho == 0 and basis.shape == (8, 1) and not basis.any()
    rho, _ = rl.nrank_search(np.eye(16), 0, 16, 1e6, 0, rl.RngStream(41, 29))
    assert rho == 16
    rho, basis = rl.nrank_search(golden["nr/wide/a"], 2, 20, 1e6, 0, rl.RngStream(41, 41))
    ref = golden["nr/wide/basis"]
    assert rho == int(golden["nr/wide/rho"][0]) and basis.shape == ref.shape
    assert np.abs(basis - ref).max() <= 1e-12 * np.abs(ref).max()
    with pytest.raises(rl.InvalidArgument):
        rl.nrank_search(np.eye(4), 3, 3, 1e6, 0, rl.RngStream(1, 1))


def test_power_transform(rl, golden):
    a = golden["pt/a"]
    assert np.array_equal(rl.power_transform(a, 0), a)
    got, want = rl.power_transform(a, 2), golden["pt/h2"]
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()

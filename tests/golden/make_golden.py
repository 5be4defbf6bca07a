"""Generate tests/golden/*.npz from the UNMODIFIED reference compiled by oracle/Makefile
(oracle/_ref/librandla_ref.so, built from /root/reference/proj/src).  Run here, where
/root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures are small (a few MB) and committed; the GPU box never needs the reference.
Inputs for the configuration-shaped cases are built with the reference's own RNG
(gaussian_matrix) and Matrix::multiply, so the bytes are exactly what the reference sees.
"""
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Reference, Restated  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__))
R = Reference()
O = Restated()
g = {}

# --- RNG streams (random_gen.cpp:22-70) -------------------------------------------
streams = [(1, 0), (7, 3), (7, 4), (11, 0), (20260825, 0x2000000000000), (31, 5)]
for seed, sid in streams:
    key = f"{seed}_{sid}"
    g[f"rng/uniform01/{key}"] = R.draws(seed, sid, "uniform01", 64)
    g[f"rng/uniform_pm1/{key}"] = R.draws(seed, sid, "uniform_pm1", 64)
    g[f"rng/gaussian/{key}"] = R.draws(seed, sid, "gaussian", 257)
    g[f"rng/sign/{key}"] = R.draws(seed, sid, "sign", 128)
    g[f"rng/uniform_int/{key}"] = R.uniform_int(seed, sid, 64, 0, 16383).astype(np.int64)
g["rng/uniform_int_dice"] = R.uniform_int(7, 5, 1000, 1, 6)
g["gaussian_matrix/4x5/11_0"] = R.gaussian_matrix(4, 5, 11, 0)
g["gaussian_matrix/33x31/mu_sigma"] = R.gaussian_matrix(33, 31, 3, 9, mu=0.5, sigma=2.0)
g["uniform_matrix/20x17/11_1"] = R.uniform_matrix(20, 17, 11, 1)
g["circulant_sign/64/9_1"] = R.circulant_sign(64, 9, 1)
g["circulant_sign/8/1_0"] = R.circulant_sign(8, 1, 0)
g["householder_sign/16/5_5"] = R.householder_sign(16, 5, 5)

# --- GENP KATs (tests/test_genp.cpp) -----------------------------------------------
dd = R.uniform_matrix(8, 8, 31, 0)
np.fill_diagonal(dd, 9.0)  # diag_dominant(8, {31, 0}) (test_genp.cpp:25-30)
L, U, piv, mm = R.genp_factor(dd)
g["genp/diag_dominant8/A"], g["genp/diag_dominant8/L"], g["genp/diag_dominant8/U"] = dd, L, U
g["genp/diag_dominant8/pivots"] = piv
a = R.gaussian_matrix(150, 150, 5, 5) + 150 * np.eye(150)
L, U, piv, mm = R.genp_factor(a)
g["genp/gauss150/A"], g["genp/gauss150/L"], g["genp/gauss150/U"], g["genp/gauss150/pivots"] = a, L, U, piv
bb = R.gaussian_matrix(150, 1, 5, 6).ravel()
g["genp/gauss150/b"], g["genp/gauss150/y"] = bb, R.genp_solve(L, U, bb)

# --- config 1 (n = 256, Gaussian, Right) ------------------------
n, seed = 256, 20260825
A = R.gaussian_matrix(n, n, seed, 1)
P = R.gaussian_matrix(128, 127, seed, 2)
Q = R.gaussian_matrix(127, 128, seed, 3)
A[:128, :128] = R.matmul(P, Q)
xt = R.gaussian_matrix(n, 1, seed, 4).ravel()
b = R.matvec(A, xt)
g["c1/A"], g["c1/b"], g["c1/x_true"] = A, b, xt
for kind in ("gaussian", "circulant_sign", "uniform_pm1"):
    for refine in (0, 1):
        y, rep = R.randomized_genp(A, b, kind, "right", refine, seed=seed, sid=11)
        g[f"c1/{kind}/r{refine}/y"], g[f"c1/{kind}/r{refine}/report"] = y, rep
y, rep = R.randomized_genp(A, b, "gaussian", "left", 0, seed=seed, sid=11)
g["c1/gaussian/left/y"], g["c1/gaussian/left/report"] = y, rep
y, rep = R.randomized_genp(A, b, "circulant_sign", "both", 1, seed=seed, sid=11)
g["c1/circulant_sign/both/y"], g["c1/circulant_sign/both/report"] = y, rep
# the other reference multiplier kinds of draw_multiplier (genp.cpp:183-203) on every side
for kind in ("toeplitz_gaussian", "householder_sign"):
    for side in ("right", "left", "both"):
        for refine in (0, 1):
            y, rep = R.randomized_genp(A, b, kind, side, refine, seed=seed, sid=11)
            g[f"c1/{kind}/{side}/r{refine}/y"], g[f"c1/{kind}/{side}/r{refine}/report"] = y, rep

# --- config 2 shape (n = 64 systems, circulant sign, Right) --------------------------
batch, n2, seed2 = 48, 64, 4096
As, bs, ys, reps, atts = [], [], [], [], []
for t in range(batch):
    At = R.gaussian_matrix(n2, n2, seed2, 10 * t + 1)
    Pt = R.gaussian_matrix(32, 31, seed2, 10 * t + 2)
    Qt = R.gaussian_matrix(31, 32, seed2, 10 * t + 3)
    At[:32, :32] = R.matmul(Pt, Qt)
    xt = R.gaussian_matrix(n2, 1, seed2, 10 * t + 4).ravel()
    bt = R.matvec(At, xt)
    y, rep = R.randomized_genp(At, bt, "circulant_sign", "right", 0, seed=seed2, sid=1000 + t)
    # the reference's report has no attempt field: take it from the restatement, whose y and report
    # must equal the reference's bit for bit (so it accepted the same draw)
    yo, ro, eo = O.randomized_genp(At, bt, "circulant_sign", "right", 0, seed=seed2, sid=1000 + t)
    assert np.array_equal(y, yo) and np.array_equal(rep, ro), t
    atts.append(int(eo[0]))
    As.append(At), bs.append(bt), ys.append(y), reps.append(rep)
g["c2/A"], g["c2/b"], g["c2/y"], g["c2/report"] = np.array(As), np.array(bs), np.array(ys), np.array(reps)
g["c2/attempt"] = np.array(atts, dtype=np.int32)
g["c2/sids"] = np.arange(1000, 1000 + batch, dtype=np.uint64)
g["c2/seed"] = np.array([seed2], dtype=np.uint64)

# --- Table-1 shaped systems (illblock_system, test_genp.cpp:136-161) -----------------
for t in range(4):
    Ai, bi, yi = R.illblock_system(64, 32, t)
    g[f"illblock64/{t}/A"], g[f"illblock64/{t}/b"] = Ai, bi
    for refine in (0, 1):
        y, rep = R.randomized_genp(Ai, bi, "circulant_sign", "left", refine, seed=33, sid=t)
        g[f"illblock64/{t}/r{refine}/y"], g[f"illblock64/{t}/r{refine}/report"] = y, rep

# --- dense core ------------------------------------------------------------------------
M = R.gaussian_matrix(40, 12, 8, 8)
qq, rr = R.qr_positive(M)
g["qr/40x12/A"], g["qr/40x12/Q"], g["qr/40x12/R"] = M, qq, rr
g["nrank/profile64"] = R.profile_matrix_paper(64, 8, 42, 90)

# proto_lowrank test matrix (tests/test_lowrank.cpp:80-91): paper profile, rank 8 of 64
g["proto/A"] = R.profile_matrix_paper(64, 8, 41, 10)
# --- structured products through the reference's own FFT (structured.cpp:20-189) -------
rs = np.random.default_rng(1212)
for n in (1, 2, 8, 64, 1024, 2048, 4096, 16384):
    z = rs.standard_normal(n) + 1j * rs.standard_normal(n)
    g[f"fft/{n}/x"] = z
    g[f"fft/{n}/fwd"] = R.fft(z, False)
    g[f"fft/{n}/inv"] = R.fft(z, True)
for n in (8, 48, 64, 1000, 4096):
    c, x = rs.standard_normal(n), rs.standard_normal(n)
    g[f"circ_mul/{n}/c"], g[f"circ_mul/{n}/x"] = c, x
    g[f"circ_mul/{n}/y"] = R.circ_mul(c, x)
for m, n in ((5, 3), (64, 64), (100, 37), (1000, 1000), (3, 700)):
    col, row, x = rs.standard_normal(m), rs.standard_normal(n), rs.standard_normal(n)
    row[0] = col[0]
    g[f"toeplitz_mul/{m}x{n}/col"], g[f"toeplitz_mul/{m}x{n}/row"], g[f"toeplitz_mul/{m}x{n}/x"] = col, row, x
    g[f"toeplitz_mul/{m}x{n}/y"] = R.toeplitz_mul(col, row, x)
for n, cols in ((48, 7), (64, 5), (300, 33)):
    c, a = rs.standard_normal(n), rs.standard_normal((n, cols))
    g[f"circ_mm/{n}x{cols}/c"], g[f"circ_mm/{n}x{cols}/a"] = c, a
    g[f"circ_mm/{n}x{cols}/out"] = R.circulant_multiply_matrix(c, a)
col, row, a = rs.standard_normal(30), rs.standard_normal(20), rs.standard_normal((20, 6))
row[0] = col[0]
g["toep_mm/col"], g["toep_mm/row"], g["toep_mm/a"] = col, row, a
g["toep_mm/out"] = R.toeplitz_multiply_matrix(col, row, a)
# take_real's imaginary-residue Error (structured.cpp:39-50) and non-finite propagation: inputs
# found by searching extreme values with the reference; the error cases raise, the others return
# inf/nan patterns
errs = [([-1e154, 1e-300, -1e154, 1e154], [-1e154, -1e154, 1.0, 1e-300]),
        ([1e154, 1e154, -1e154, -1e154], [1e-300, -1e154, 1e300, 1e308]),
        ([1.0, 1e-300, 1e-300, 0.0, 0.0], [-1e154, 0.0, -1e154, -1e308, 1e154]),
        ([1.0, 1e154, 1e154, -1e154], [1.0, 1e300, 1e300, 1e154])]
for k, (c, x) in enumerate(errs):
    try:
        R.circ_mul(np.array(c), np.array(x))
        raise SystemExit("expected the reference to raise")
    except Exception as e:  # OracleError with the Error status
        assert "imaginary residue" in str(e), e
    g[f"circ_err/{k}/c"], g[f"circ_err/{k}/x"] = np.array(c), np.array(x)
nonfinite = [([np.inf, 0, 0, 0], [1, 0, 0, 0]), ([np.inf, 1, 2, 3], [1, 1, 1, 1]),
             ([1e300, 1e300, -1e300, 1e-300], [1e300, 1, 1, 1]), ([1, 2, 3], [np.inf, 1, 1])]
for k, (c, x) in enumerate(nonfinite):
    c, x = np.array(c, float), np.array(x, float)
    g[f"circ_nf/{k}/c"], g[f"circ_nf/{k}/x"], g[f"circ_nf/{k}/y"] = c, x, R.circ_mul(c, x)

# --- the rank-search side of lowrank (lowrank.cpp:179-396; tests/test_lowrank.cpp:116-177) ----
d51 = np.diag([5.0, 1.0])
q8 = R.random_orthogonal(8, 41, 16)
sig32 = np.ones(32)
sig32[31] = 1e-3
p32 = R.profile_matrix(sig32, 41, 18)
g["es/q8"], g["es/p32"] = q8, p32
for meth in (0, 1):
    g[f"es/d51/{meth}"] = np.array(R.extremal_sv_estimate(d51, meth, 200, 41, 15))
    g[f"es/q8/{meth}"] = np.array(R.extremal_sv_estimate(q8, meth, 200, 41, 17))
    g[f"es/p32/{meth}"] = np.array(R.extremal_sv_estimate(p32, meth, 5000, 41, 19))
a64 = R.profile_matrix_paper(64, 8, 41, 22)
g9 = R.gaussian_matrix(64, 9, 41, 23)
g["cp/b8"], g["cp/b9"] = a64.T @ g9[:, :8], a64.T @ g9
g["cp/b8/pass"] = np.array([R.cond_probe(g["cp/b8"], 1e6, 1, 56, 41, 24)])
g["cp/b9/pass"] = np.array([R.cond_probe(g["cp/b9"], 1e6, 1, 56, 41, 25)])
a26 = R.profile_matrix_paper(64, 8, 41, 26)
g["nr/a"] = a26
for pol in (0, 1):
    rho, basis = R.nrank_search(a26, 0, 16, 1e6, pol, 41, 27)
    g[f"nr/{pol}/rho"], g[f"nr/{pol}/basis"] = np.array([rho]), basis
wide = R.gaussian_matrix(24, 80, 41, 40)
wide = wide[:, :80] * 1.0
rho, basis = R.nrank_search(wide, 2, 20, 1e6, 0, 41, 41)  # m < n: the transposed work matrix
g["nr/wide/a"], g["nr/wide/rho"], g["nr/wide/basis"] = wide, np.array([rho]), basis
g["pt/a"] = R.gaussian_matrix(20, 7, 41, 42)
g["pt/h2"] = R.power_transform(g["pt/a"], 2)

# proto_lowrank beyond the one-CTA SVD: a 320 x 320 paper profile (rank 8), rho_plus 12, both kinds
g["proto320/A"] = R.profile_matrix_paper(320, 8, 41, 60)
for kind in ("gaussian", "toeplitz_gaussian"):
    rho, basis, approx, res, ok = R.proto_lowrank(g["proto320/A"], 12, 1e-6, 1e-6, 41, 61, kind=kind)
    g[f"proto320/{kind}/out"] = np.array([rho, res, float(ok)])
    g[f"proto320/{kind}/approx"] = approx

# --- Table 1 (bench.cpp:107-140 table1_genp, acceptance.cpp:51-73 scale): 100 trials at n = 64,
# seed 20260825; systems and the reference's samples (rep0.residual, rep1.residual, raw) per trial,
# each trial exactly table1_genp's run(): illblock_system on (seed, 0x1000000000000 + base),
# randomized_genp Left refine 0/1 on (seed, 0x2000000000000 + base), base = 64 t (size index 0)
T1, s1 = 100, 20260825
As, bs, samp = [], [], []
for t in range(T1):
    base = 64 * t
    At, bt, _ = R.illblock_system(64, s1, 0x1000000000000 + base)
    _, r0 = R.randomized_genp(At, bt, "circulant_sign", "left", 0, seed=s1, sid=0x2000000000000 + base)
    _, r1 = R.randomized_genp(At, bt, "circulant_sign", "left", 1, seed=s1, sid=0x2000000000000 + base)
    As.append(At), bs.append(bt), samp.append([r0[0], r1[0], r0[1]])
g["t1/A"], g["t1/b"], g["t1/samples"] = np.array(As), np.array(bs), np.array(samp)

np.savez_compressed(os.path.join(OUT, "golden.npz"), **g)
print("wrote", os.path.join(OUT, "golden.npz"), len(g), "arrays")

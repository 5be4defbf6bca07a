"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracles.

* ``Restated``  -> oracle/lib/librl_oracle.so   (plain-C restatement, rl_oracle.c)
* ``Reference`` -> oracle/_ref/librandla_ref.so (the unmodified reference sources
  compiled by oracle/Makefile; absent when /root/reference was never available)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this
module.  The product package (paper_1212_4560_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(HERE, "lib", "librl_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "librandla_ref.so")

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u64, i64, dbl, cint = C.c_uint64, C.c_int64, C.c_double, C.c_int

TAGS = {"gaussian": 0, "uniform_pm1": 1, "toeplitz_gaussian": 2, "circulant_gaussian": 3,
        "circulant_sign": 4, "householder_sign": 5, "householder_pair": 6, "sparse_sign": 7}
SIDES = {"left": 0, "right": 1, "both": 2}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: status {code}")
        self.code = code


def _ensure_built(target: str) -> None:
    if target == "restated" and not os.path.exists(RESTATED_SO):
        subprocess.check_call(["make", "-s", "-C", HERE, "restated"])


def _chk(code: int, where: str) -> None:
    if code != 0:
        raise OracleError(code, where)


class Restated:
    """The C restatement (oracle/rl_oracle.c).  threads > 1 enables its row-parallel
    loops (bit-identical results; used by the full-size parity runs)."""

    def __init__(self, threads: int = 1) -> None:
        _ensure_built("restated")
        L = C.CDLL(RESTATED_SO)
        L.rlo_set_threads.argtypes = [cint]
        L.rlo_set_threads(threads)
        self.lib = L
        L.rlo_raw_u64.argtypes = [u64, u64, u64, _u64p]
        L.rlo_gaussian_matrix.argtypes = [u64, u64, dbl, dbl, u64, u64, _d]
        L.rlo_uniform_matrix.argtypes = [u64, u64, u64, u64, _d]
        L.rlo_sign_vector.argtypes = [u64, u64, u64, _d]
        L.rlo_householder_pair_signs.argtypes = [u64, u64, u64, _d, _d]
        L.rlo_sparse_pm1.argtypes = [u64, cint, u64, u64, _i32p, _d]
        L.rlo_matmul.argtypes = [u64, u64, u64, _d, _d, _d]
        L.rlo_matvec.argtypes = [u64, u64, _d, _d, _d]
        L.rlo_genp_factor.argtypes = [u64, _d, dbl, _d]
        L.rlo_genp_solve.argtypes = [u64, _d, _d, _d]
        L.rlo_relative_residual.argtypes = [u64, _d, _d, _d]
        L.rlo_relative_residual.restype = dbl
        L.rlo_circ_mul.argtypes = [u64, _d, _d, _d]
        L.rlo_circ_apply_right.argtypes = [u64, _d, _d, _d]
        L.rlo_circ_apply_left.argtypes = [u64, _d, u64, _d, _d]
        L.rlo_hh2_apply_right.argtypes = [u64, _d, _d, _d, _d]
        L.rlo_hh2_apply_vec.argtypes = [u64, _d, _d, _d, _d]
        L.rlo_sparse_apply_right.argtypes = [u64, cint, _i32p, _d, _d, _d]
        L.rlo_sparse_apply_vec.argtypes = [u64, cint, _i32p, _d, _d, _d]
        L.rlo_randomized_genp.argtypes = [u64, _d, _d, cint, dbl, dbl, cint, cint, u64, u64, _d, _d, _ip]
        L.rlo_randomized_genp_multi.argtypes = [u64, u64, _d, _d, cint, dbl, dbl, cint, cint, u64, u64, cint, _d,
                                                _d, _ip]
        L.rlo_qr_positive.argtypes = [u64, u64, _d, _d, _d]
        L.rlo_singular_values.argtypes = [u64, u64, _d, _d]
        L.rlo_proto_lowrank.argtypes = [u64, u64, _d, u64, dbl, dbl, cint, dbl, dbl, u64, u64, C.POINTER(C.c_uint64), _d, _d,
                                        C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.rlo_numerical_rank.argtypes = [u64, _d, dbl]
        L.rlo_numerical_rank.restype = u64

    def raw_u64(self, seed, sid, count):
        out = np.empty(count, np.uint64)
        self.lib.rlo_raw_u64(seed, sid, count, out)
        return out

    def gaussian_matrix(self, m, n, seed, sid, mu=0.0, sigma=1.0):
        out = np.empty((m, n))
        _chk(self.lib.rlo_gaussian_matrix(m, n, mu, sigma, seed, sid, out), "gaussian_matrix")
        return out

    def uniform_matrix(self, m, n, seed, sid):
        out = np.empty((m, n))
        self.lib.rlo_uniform_matrix(m, n, seed, sid, out)
        return out

    def sign_vector(self, n, seed, sid):
        out = np.empty(n)
        self.lib.rlo_sign_vector(n, seed, sid, out)
        return out

    def householder_pair_signs(self, n, seed, sid):
        u1, u2 = np.empty(n), np.empty(n)
        self.lib.rlo_householder_pair_signs(n, seed, sid, u1, u2)
        return u1, u2

    def sparse_pm1(self, n, seed, sid, nnz=4):
        rows = np.empty((n, nnz), np.int32)
        signs = np.empty((n, nnz))
        _chk(self.lib.rlo_sparse_pm1(n, nnz, seed, sid, rows, signs), "sparse_pm1")
        return rows, signs

    def matmul(self, a, b):
        a, b = np.ascontiguousarray(a, float), np.ascontiguousarray(b, float)
        c = np.empty((a.shape[0], b.shape[1]))
        self.lib.rlo_matmul(a.shape[0], a.shape[1], b.shape[1], a, b, c)
        return c

    def matvec(self, a, x):
        a, x = np.ascontiguousarray(a, float), np.ascontiguousarray(x, float)
        y = np.empty(a.shape[0])
        self.lib.rlo_matvec(a.shape[0], a.shape[1], a, x, y)
        return y

    def genp_factor(self, a, pivot_floor=1e-300):
        """Returns (L, U, pivots) like genp.cpp:11-41 (raises on breakdown)."""
        n = a.shape[0]
        w = np.array(a, dtype=float, order="C")
        piv = np.empty(n)
        st = self.lib.rlo_genp_factor(n, w, pivot_floor, piv)
        if st != 0:
            raise OracleError(3, f"genp_factor: pivot below floor at step {-st - 1}")
        L = np.tril(w, -1) + np.eye(n)
        U = np.triu(w)
        return L, U, piv, w

    def genp_solve_packed(self, lu, b):
        y = np.empty(lu.shape[0])
        self.lib.rlo_genp_solve(lu.shape[0], np.ascontiguousarray(lu), np.ascontiguousarray(b, float), y)
        return y

    def relative_residual(self, a, y, b):
        return self.lib.rlo_relative_residual(a.shape[0], np.ascontiguousarray(a), np.ascontiguousarray(y),
                                              np.ascontiguousarray(b))

    def circ_mul(self, c, x):
        y = np.empty(len(c))
        _chk(self.lib.rlo_circ_mul(len(c), np.ascontiguousarray(c, float), np.ascontiguousarray(x, float), y),
             "circ_mul")
        return y

    def circ_apply_right(self, c, a):
        out = np.empty_like(a)
        _chk(self.lib.rlo_circ_apply_right(len(c), np.ascontiguousarray(c, float), np.ascontiguousarray(a), out),
             "circ_apply_right")
        return out

    def hh2_apply_right(self, u1, u2, a):
        out = np.empty_like(a)
        self.lib.rlo_hh2_apply_right(len(u1), u1, u2, np.ascontiguousarray(a), out)
        return out

    def hh2_apply_vec(self, u1, u2, y):
        x = np.empty(len(u1))
        self.lib.rlo_hh2_apply_vec(len(u1), u1, u2, np.ascontiguousarray(y, float), x)
        return x

    def sparse_apply_right(self, rows, signs, a):
        out = np.empty_like(a)
        self.lib.rlo_sparse_apply_right(a.shape[0], rows.shape[1], np.ascontiguousarray(rows),
                                        np.ascontiguousarray(signs), np.ascontiguousarray(a), out)
        return out

    def sparse_apply_vec(self, rows, signs, y):
        x = np.empty(rows.shape[0])
        self.lib.rlo_sparse_apply_vec(rows.shape[0], rows.shape[1], np.ascontiguousarray(rows),
                                      np.ascontiguousarray(signs), np.ascontiguousarray(y, float), x)
        return x

    def proto_lowrank(self, a, rho_plus, tau, tau_prime, seed, sid, mu=0.0, sigma=1.0, kind="gaussian"):
        """lowrank::proto_lowrank, Gaussian / ToeplitzGaussian: (rho, basis n x rho, approx, residual, ok)."""
        a = np.ascontiguousarray(a, float)
        m, n = a.shape
        basis, approx = np.zeros((n, rho_plus)), np.empty((m, n))
        rho, res, ok = C.c_uint64(0), C.c_double(0.0), C.c_int(0)
        _chk(self.lib.rlo_proto_lowrank(m, n, a, rho_plus, tau, tau_prime, TAGS[kind], mu, sigma, seed, sid, C.byref(rho), basis,
                                        approx, C.byref(res), C.byref(ok)), "proto_lowrank")
        return rho.value, basis[:, :rho.value], approx, res.value, bool(ok.value)

    def randomized_genp(self, a, b, kind="gaussian", side="right", refine=0, seed=0, sid=0, mu=0.0, sigma=1.0):
        n = a.shape[0]
        y, rep, extra = np.empty(n), np.empty(6), np.zeros(2, np.int32)
        _chk(self.lib.rlo_randomized_genp(n, np.ascontiguousarray(a, float), np.ascontiguousarray(b, float),
                                          TAGS[kind], mu, sigma, SIDES[side], refine, seed, sid, y, rep, extra),
             "randomized_genp")
        return y, rep, extra

    def randomized_genp_multi(self, a, B, kind="gaussian", side="right", refine=0, seed=0, sid=0, mu=0.0,
                              sigma=1.0, skip_raw=False):
        """nrhs columns of B as independent randomized_genp calls sharing the stream: Y, reports
        (nrhs x 6), extras (nrhs x 2: accepted attempt, attempts drawn)."""
        n, nrhs = B.shape
        Y, rep, extra = np.empty((n, nrhs)), np.empty((nrhs, 6)), np.zeros((nrhs, 2), np.int32)
        _chk(self.lib.rlo_randomized_genp_multi(n, nrhs, np.ascontiguousarray(a, float), np.ascontiguousarray(B, float),
                                                TAGS[kind], mu, sigma, SIDES[side], refine, seed, sid, int(skip_raw),
                                                Y, rep, extra), "randomized_genp_multi")
        return Y, rep, extra

    def qr_positive(self, a):
        m, n = a.shape
        q, r = np.empty((m, n)), np.empty((n, n))
        _chk(self.lib.rlo_qr_positive(m, n, np.ascontiguousarray(a, float), q, r), "qr_positive")
        return q, r

    def singular_values(self, a):
        m, n = a.shape
        s = np.empty(min(m, n))
        self.lib.rlo_singular_values(m, n, np.ascontiguousarray(a, float), s)
        return s

    def numerical_rank(self, sigma, tol):
        return int(self.lib.rlo_numerical_rank(len(sigma), np.ascontiguousarray(sigma, float), tol))


class Reference:
    """The unmodified reference, compiled from /root/reference by oracle/Makefile."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REFERENCE_SO)

    def __init__(self) -> None:
        L = C.CDLL(REFERENCE_SO)
        self.lib = L
        L.rlref_last_error.restype = C.c_char_p
        L.rlref_draws.argtypes = [u64, u64, cint, u64, i64, i64, _d]
        L.rlref_uniform_int.argtypes = [u64, u64, u64, i64, i64, _i64p]
        L.rlref_gaussian_matrix.argtypes = [u64, u64, dbl, dbl, u64, u64, _d]
        L.rlref_uniform_matrix.argtypes = [u64, u64, u64, u64, _d]
        L.rlref_random_structured.argtypes = [cint, dbl, dbl, u64, u64, u64, u64, _d, C.c_void_p]
        L.rlref_householder_sign.argtypes = [u64, u64, u64, _d]
        L.rlref_matmul.argtypes = [u64, u64, u64, _d, _d, _d]
        L.rlref_matvec.argtypes = [u64, u64, _d, _d, _d]
        L.rlref_circulant_multiply_matrix.argtypes = [u64, _d, u64, _d, _d]
        L.rlref_circ_mul.argtypes = [u64, _d, _d, _d]
        L.rlref_fft.argtypes = [u64, _d, cint, _d]
        L.rlref_toeplitz_mul.argtypes = [u64, u64, _d, _d, _d, _d]
        L.rlref_toeplitz_multiply_matrix.argtypes = [u64, u64, _d, _d, u64, _d, _d]
        L.rlref_genp_factor.argtypes = [u64, _d, dbl, _d, _d, _d, _d]
        L.rlref_block_ge.argtypes = [u64, _d, u64, _d, _d, _d, _d]
        L.rlref_genp_solve.argtypes = [u64, _d, _d, _d, _d]
        L.rlref_randomized_genp.argtypes = [u64, _d, _d, cint, dbl, dbl, cint, cint, u64, u64, _d, _d]
        L.rlref_illblock_system.argtypes = [u64, u64, u64, _d, _d, _d]
        L.rlref_qr_positive.argtypes = [u64, u64, _d, _d, _d]
        L.rlref_singular_values.argtypes = [u64, u64, _d, _d]
        L.rlref_profile_matrix_paper.argtypes = [u64, u64, u64, u64, _d]
        P = C.POINTER
        L.rlref_proto_lowrank.argtypes = [u64, u64, _d, u64, dbl, dbl, cint, dbl, dbl, u64, u64, P(C.c_uint64), _d,
                                          _d, P(C.c_uint64), P(C.c_double), P(C.c_int)]
        L.rlref_nrank_search.argtypes = [u64, u64, _d, u64, u64, dbl, cint, u64, u64, P(C.c_uint64), _d,
                                         P(C.c_uint64), P(C.c_uint64)]
        L.rlref_extremal_sv_estimate.argtypes = [u64, u64, _d, cint, cint, u64, u64, P(C.c_double), P(C.c_double)]
        L.rlref_cond_probe.argtypes = [u64, u64, _d, dbl, cint, cint, u64, u64, P(C.c_int)]
        L.rlref_power_transform.argtypes = [u64, u64, _d, C.c_uint, _d]
        L.rlref_profile_matrix.argtypes = [u64, _d, u64, u64, _d]
        L.rlref_random_orthogonal.argtypes = [u64, u64, u64, _d]
        L.rlref_sampled_residual_check.argtypes = [u64, u64, _d, _d, u64, u64, dbl, u64, u64, P(C.c_int)]

    def _chk(self, code, where):
        if code != 0:
            raise OracleError(code, f"{where}: {self.lib.rlref_last_error().decode()}")

    def draws(self, seed, sid, kind, count, lo=0, hi=1):
        out = np.empty(count)
        k = {"uniform01": 0, "uniform_pm1": 1, "gaussian": 2, "sign": 3, "uniform_int": 4}[kind]
        self._chk(self.lib.rlref_draws(seed, sid, k, count, lo, hi, out), "draws")
        return out

    def uniform_int(self, seed, sid, count, lo, hi):
        out = np.empty(count, np.int64)
        self._chk(self.lib.rlref_uniform_int(seed, sid, count, lo, hi, out), "uniform_int")
        return out

    def gaussian_matrix(self, m, n, seed, sid, mu=0.0, sigma=1.0):
        out = np.empty((m, n))
        self._chk(self.lib.rlref_gaussian_matrix(m, n, mu, sigma, seed, sid, out), "gaussian_matrix")
        return out

    def uniform_matrix(self, m, n, seed, sid):
        out = np.empty((m, n))
        self._chk(self.lib.rlref_uniform_matrix(m, n, seed, sid, out), "uniform_matrix")
        return out

    def circulant_sign(self, n, seed, sid):
        col = np.empty(n)
        self._chk(self.lib.rlref_random_structured(TAGS["circulant_sign"], 0.0, 1.0, n, n, seed, sid, col, None),
                  "random_structured")
        return col

    def householder_sign(self, n, seed, sid):
        out = np.empty((n, n))
        self._chk(self.lib.rlref_householder_sign(n, seed, sid, out), "householder_sign")
        return out

    def matmul(self, a, b):
        a, b = np.ascontiguousarray(a, float), np.ascontiguousarray(b, float)
        c = np.empty((a.shape[0], b.shape[1]))
        self._chk(self.lib.rlref_matmul(a.shape[0], a.shape[1], b.shape[1], a, b, c), "matmul")
        return c

    def matvec(self, a, x):
        a, x = np.ascontiguousarray(a, float), np.ascontiguousarray(x, float)
        y = np.empty(a.shape[0])
        self._chk(self.lib.rlref_matvec(a.shape[0], a.shape[1], a, x, y), "matvec")
        return y

    def circ_mul(self, c, x):
        y = np.empty(len(c))
        self._chk(self.lib.rlref_circ_mul(len(c), np.ascontiguousarray(c, float), np.ascontiguousarray(x, float), y),
                  "circ_mul")
        return y

    def fft(self, x, inverse=False):
        """structured::fft on a complex vector."""
        z = np.ascontiguousarray(np.asarray(x, np.complex128)).view(np.float64)
        out = np.empty_like(z)
        self._chk(self.lib.rlref_fft(len(z) // 2, z, int(inverse), out), "fft")
        return out.view(np.complex128)

    def toeplitz_mul(self, col, row, x):
        y = np.empty(len(col))
        self._chk(self.lib.rlref_toeplitz_mul(len(col), len(row), np.ascontiguousarray(col, float),
                                              np.ascontiguousarray(row, float), np.ascontiguousarray(x, float), y),
                  "toeplitz_mul")
        return y

    def toeplitz_multiply_matrix(self, col, row, a):
        out = np.empty((len(col), a.shape[1]))
        self._chk(self.lib.rlref_toeplitz_multiply_matrix(len(col), len(row), np.ascontiguousarray(col, float),
                                                          np.ascontiguousarray(row, float), a.shape[1],
                                                          np.ascontiguousarray(a, float), out), "multiply_matrix")
        return out

    def circulant_multiply_matrix(self, c, a):
        out = np.empty_like(a)
        self._chk(self.lib.rlref_circulant_multiply_matrix(len(c), np.ascontiguousarray(c, float), a.shape[1],
                                                           np.ascontiguousarray(a), out), "multiply_matrix")
        return out

    def genp_factor(self, a, pivot_floor=1e-300):
        n = a.shape[0]
        L, U, piv, mm = np.empty((n, n)), np.empty((n, n)), np.empty(n), np.empty(2)
        self._chk(self.lib.rlref_genp_factor(n, np.ascontiguousarray(a, float), pivot_floor, L, U, piv, mm),
                  "genp_factor")
        return L, U, piv, mm

    def block_ge(self, a, block):
        n = a.shape[0]
        nb = (n + block - 1) // block
        L, U, pn, pin = np.empty((n, n)), np.empty((n, n)), np.empty(nb), np.empty(nb)
        self._chk(self.lib.rlref_block_ge(n, np.ascontiguousarray(a, float), block, L, U, pn, pin), "block_ge")
        return L, U, pn, pin

    def genp_solve(self, L, U, b):
        y = np.empty(L.shape[0])
        self._chk(self.lib.rlref_genp_solve(L.shape[0], np.ascontiguousarray(L), np.ascontiguousarray(U),
                                            np.ascontiguousarray(b, float), y), "genp_solve")
        return y

    def randomized_genp(self, a, b, kind="gaussian", side="right", refine=0, seed=0, sid=0, mu=0.0, sigma=1.0):
        n = a.shape[0]
        y, rep = np.empty(n), np.empty(6)
        self._chk(self.lib.rlref_randomized_genp(n, np.ascontiguousarray(a, float), np.ascontiguousarray(b, float),
                                                 TAGS[kind], mu, sigma, SIDES[side], refine, seed, sid, y, rep),
                  "randomized_genp")
        return y, rep

    def proto_lowrank(self, a, rho_plus, tau, tau_prime, seed, sid, mu=0.0, sigma=1.0, kind="gaussian"):
        """lowrank::proto_lowrank (lowrank.cpp:108-177): (rho, basis, approx, residual, ok)."""
        a = np.ascontiguousarray(a, float)
        m, n = a.shape
        basis, approx = np.zeros(max(n * rho_plus, n)), np.empty((m, n))
        rho, cols, res, ok = C.c_uint64(0), C.c_uint64(0), C.c_double(0.0), C.c_int(0)
        self._chk(self.lib.rlref_proto_lowrank(m, n, a, rho_plus, tau, tau_prime, TAGS[kind], mu, sigma, seed, sid,
                                               C.byref(rho), approx, basis, C.byref(cols), C.byref(res), C.byref(ok)),
                  "proto_lowrank")
        basis = basis[:n * cols.value].reshape(n, cols.value)
        return rho.value, basis[:, :rho.value], approx, res.value, bool(ok.value)

    def nrank_search(self, a, rho_minus, rho_plus, kappa, policy, seed, sid):
        """lowrank::nrank_search (lowrank.cpp:360-396): (rho, basis) with policy 0 Binary / 1 LinearDown."""
        a = np.ascontiguousarray(a, float)
        m, n = a.shape
        w = max(m, n)
        basis = np.zeros(max(min(m, n) * rho_plus, w))
        rho, br, bc = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        self._chk(self.lib.rlref_nrank_search(m, n, a, rho_minus, rho_plus, kappa, policy, seed, sid, C.byref(rho),
                                              basis, C.byref(br), C.byref(bc)), "nrank_search")
        return rho.value, basis[:br.value * bc.value].reshape(br.value, bc.value)

    def extremal_sv_estimate(self, a, method, iters, seed, sid):
        """lowrank::extremal_sv_estimate: (sv_max, sv_min); method 0 Power / 1 Lanczos."""
        a = np.ascontiguousarray(a, float)
        hi, lo = C.c_double(0.0), C.c_double(0.0)
        self._chk(self.lib.rlref_extremal_sv_estimate(a.shape[0], a.shape[1], a, method, iters, seed, sid,
                                                      C.byref(hi), C.byref(lo)), "extremal_sv_estimate")
        return hi.value, lo.value

    def cond_probe(self, b, kappa, method, iters, seed, sid):
        b = np.ascontiguousarray(b, float)
        ok = C.c_int(0)
        self._chk(self.lib.rlref_cond_probe(b.shape[0], b.shape[1], b, kappa, method, iters, seed, sid, C.byref(ok)),
                  "cond_probe")
        return bool(ok.value)

    def power_transform(self, a, h):
        a = np.ascontiguousarray(a, float)
        out = np.empty_like(a)
        self._chk(self.lib.rlref_power_transform(a.shape[0], a.shape[1], a, h, out), "power_transform")
        return out

    def sampled_residual_check(self, a, ahat, rho1, rho2, tau, seed, sid):
        ok = C.c_int(0)
        a, ahat = np.ascontiguousarray(a, float), np.ascontiguousarray(ahat, float)
        self._chk(self.lib.rlref_sampled_residual_check(a.shape[0], a.shape[1], a, ahat, rho1, rho2, tau, seed, sid,
                                                        C.byref(ok)), "sampled_residual_check")
        return bool(ok.value)

    def profile_matrix(self, sigmas, seed, sid):
        n = len(sigmas)
        out = np.empty((n, n))
        self._chk(self.lib.rlref_profile_matrix(n, np.ascontiguousarray(sigmas, float), seed, sid, out),
                  "profile_matrix")
        return out

    def random_orthogonal(self, n, seed, sid):
        out = np.empty((n, n))
        self._chk(self.lib.rlref_random_orthogonal(n, seed, sid, out), "random_orthogonal")
        return out

    def illblock_system(self, n, seed, sid):
        a, b, y = np.empty((n, n)), np.empty(n), np.empty(n)
        self._chk(self.lib.rlref_illblock_system(n, seed, sid, a, b, y), "illblock_system")
        return a, b, y

    def profile_matrix_paper(self, n, rho, seed, sid):
        out = np.empty((n, n))
        self._chk(self.lib.rlref_profile_matrix_paper(n, rho, seed, sid, out), "profile_matrix")
        return out

    def qr_positive(self, a):
        m, n = a.shape
        q, r = np.empty((m, n)), np.empty((n, n))
        self._chk(self.lib.rlref_qr_positive(m, n, np.ascontiguousarray(a, float), q, r), "qr_positive")
        return q, r

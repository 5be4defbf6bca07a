"""B200-native randomized-multiplier GENP and range finder (arXiv 1212.4560 hot path).

Python mirror of the reference's C++ API (``randla``, /root/reference/proj/include/randla)
over the C-ABI in ``include/rl_b200.h`` (``lib/librl_b200.so``).  Names, argument
meaning and error behaviour follow the reference:

    gaussian_matrix / uniform_matrix / random_structured / householder_sign   random_gen.hpp
    genp_factor / genp_solve / randomized_genp                                genp.hpp
    approx_basis / project_onto_basis / qr_positive / numerical_rank         lowrank.hpp, dense_core.hpp

plus the additive extensions of SURVEY.md §8(b): multi-RHS solves, the batched
randomized_genp, the orthogonal Householder-pair and sparse +-1 multipliers, and the
fused device range finder.  Host (numpy) arguments follow the reference's value
semantics; ``dev_*`` functions take CUDA tensors (torch is plumbing only).

There is no CPU fallback: every compute call runs the CUDA library, and importing a
function whose library is missing raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Error", "DimensionMismatch", "InvalidArgument", "PivotBreakdown", "RankDeficient", "Degenerate",
    "NoConvergence", "TooLarge", "CudaError", "NoDevice", "RngStream", "MultiplierKind", "MultiplierTag",
    "MulSide", "PrecondReport", "GenpFactorization", "lib", "gaussian_matrix", "uniform_matrix",
    "random_structured", "householder_sign", "householder_pair_signs", "sparse_sign", "sparse_apply_right", "rng_draws", "raw_u64",
    "multiply", "circ_mul", "circulant_multiply_matrix", "genp_factor", "genp_solve", "randomized_genp",
    "randomized_genp_batched", "approx_basis", "qr_positive", "project_onto_basis", "numerical_rank",
    "dev_gemm", "dev_gaussian_matrix", "dev_genp_factor", "dev_genp_solve", "dev_randomized_genp",
    "dev_randomized_genp_batched", "dev_range_finder", "dev_sparse_apply_right",
    "dev_householder_pair_apply_right", "dev_circulant_apply_right", "dev_toeplitz_apply_right", "proto_lowrank", "dev_qr_positive", "dev_numerical_rank", "probe_peaks",
    "box_muller", "box_muller_hash", "last_column_reports", "fft", "toeplitz_mul", "toeplitz_multiply_matrix", "SvMethod", "SearchPolicy", "extremal_sv_estimate", "cond_probe", "nrank_search", "power_transform", "launch_count", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "librl_b200.so")


# ------------------------------------------------------------------ errors ----
class Error(RuntimeError):
    """randla::Error (errors.hpp:9-11)."""


class DimensionMismatch(Error):
    pass


class InvalidArgument(Error):
    pass


class PivotBreakdown(Error):
    pass


class RankDeficient(Error):
    pass


class Degenerate(Error):
    pass


class LengthNotPowerOfTwo(Error):
    pass


class IndexOutOfRange(Error):
    pass


class NoConvergence(Error):
    pass


class ZeroMatrix(Error):
    pass


class ConstructionFailed(Error):
    pass


class TooLarge(Error):
    pass


class CudaError(Error):
    pass


class NoDevice(Error):
    pass


_ERRORS = {1: DimensionMismatch, 2: InvalidArgument, 3: PivotBreakdown, 4: RankDeficient, 5: Degenerate,
           6: LengthNotPowerOfTwo, 7: IndexOutOfRange, 8: NoConvergence, 9: ZeroMatrix, 10: ConstructionFailed,
           11: Error, 12: TooLarge, 20: CudaError, 21: NoDevice}


# ------------------------------------------------------------------- types ----
@dataclass(frozen=True)
class RngStream:
    """rnd::RngStream (random_gen.hpp:16-21)."""
    seed: int = 0
    stream_id: int = 0

    def with_stream(self, sid: int) -> "RngStream":
        return RngStream(self.seed, sid)


class MultiplierTag:
    """rnd::MultiplierTag (random_gen.hpp:46-53) + HOUSEHOLDER_PAIR / SPARSE_SIGN."""
    GAUSSIAN = 0
    UNIFORM_PM1 = 1
    TOEPLITZ_GAUSSIAN = 2
    CIRCULANT_GAUSSIAN = 3
    CIRCULANT_SIGN = 4
    HOUSEHOLDER_SIGN = 5
    HOUSEHOLDER_PAIR = 6
    SPARSE_SIGN = 7


@dataclass(frozen=True)
class MultiplierKind:
    """rnd::MultiplierKind (random_gen.hpp:56-60)."""
    tag: int = MultiplierTag.GAUSSIAN
    mu: float = 0.0
    sigma: float = 1.0


class MulSide:
    """genp::MulSide (genp.hpp:49)."""
    LEFT = 0
    RIGHT = 1
    BOTH = 2


class _ColumnReport(C.Structure):
    _fields_ = [("residual", C.c_double), ("pivot_min", C.c_double), ("pivot_max", C.c_double),
                ("attempt", C.c_int32), ("attempts_drawn", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("residual", C.c_double), ("raw_residual", C.c_double), ("pivot_min", C.c_double),
                ("pivot_max", C.c_double), ("raw_pivot_min", C.c_double), ("raw_pivot_max", C.c_double),
                ("attempt", C.c_int32), ("attempts_drawn", C.c_int32)]


@dataclass
class PrecondReport:
    """genp::PrecondReport (genp.hpp:51-60) + attempt bookkeeping."""
    multiplier: MultiplierKind
    refinement_steps: int
    residual: float
    raw_residual: float
    pivot_min: float
    pivot_max: float
    raw_pivot_min: float
    raw_pivot_max: float
    attempt: int
    attempts_drawn: int


@dataclass
class GenpFactorization:
    """genp::GenpFactorization (genp.hpp:14-20)."""
    L: np.ndarray
    U: np.ndarray
    pivot_abs: np.ndarray
    pivot_min: float
    pivot_max: float


# ----------------------------------------------------------------- library ----
_lib = None
_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64a = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i32a = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u64, i64, dbl, cint, vp = C.c_uint64, C.c_int64, C.c_double, C.c_int, C.c_void_p


def lib() -> C.CDLL:
    """Load lib/librl_b200.so (fails loudly: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    L.rl_last_error.restype = C.c_char_p
    L.rl_launch_count.restype = u64
    L.rl_get_stream.restype = vp
    sig = {
        "rl_init": [cint], "rl_set_stream": [vp], "rl_synchronize": [],
        "rl_rng_draws": [u64, u64, cint, u64, i64, i64, _d],
        "rl_raw_u64": [u64, u64, u64, _u64a],
        "rl_gaussian_matrix": [u64, u64, dbl, dbl, u64, u64, _d],
        "rl_dev_gaussian_matrix": [u64, u64, dbl, dbl, u64, u64, vp],
        "rl_uniform_matrix": [u64, u64, u64, u64, _d],
        "rl_random_structured": [cint, dbl, dbl, u64, u64, u64, u64, _d, vp],
        "rl_householder_sign": [u64, u64, u64, _d],
        "rl_householder_pair_signs": [u64, u64, u64, _d, _d],
        "rl_sparse_sign": [u64, cint, u64, u64, _i32a, _d],
        "rl_sparse_apply_right": [u64, cint, _i32a, _d, _d, _d],
        "rl_dev_sparse_apply_right": [u64, cint, vp, vp, vp, vp],
        "rl_dev_householder_pair_apply_right": [u64, vp, vp, vp, vp],
        "rl_dev_circulant_apply_right": [u64, u64, vp, vp, vp],
        "rl_dev_toeplitz_apply_right": [u64, u64, vp, vp, vp],
        "rl_proto_lowrank": [u64, u64, _d, u64, dbl, dbl, cint, dbl, dbl, u64, u64, C.POINTER(C.c_uint64), _d, _d,
                             C.POINTER(C.c_double), C.POINTER(C.c_int)],
        "rl_matmul": [u64, u64, u64, _d, _d, _d],
        "rl_dev_gemm": [cint, cint, u64, u64, u64, dbl, vp, u64, vp, u64, dbl, vp, u64],
        "rl_circ_mul": [u64, _d, _d, _d],
        "rl_circulant_multiply_matrix": [u64, _d, u64, _d, _d],
        "rl_toeplitz_mul": [u64, u64, _d, _d, _d, _d],
        "rl_toeplitz_multiply_matrix": [u64, u64, _d, _d, u64, _d, _d],
        "rl_fft": [u64, vp, cint, vp],
        "rl_genp_factor": [u64, _d, dbl, _d, _d, _d, _d, C.POINTER(C.c_int64)],
        "rl_dev_genp_factor": [u64, vp, u64, dbl, vp, C.POINTER(C.c_int64)],
        "rl_genp_solve": [u64, u64, _d, _d, _d, _d],
        "rl_dev_genp_solve_packed": [u64, u64, vp, u64, vp],
        "rl_randomized_genp": [u64, u64, _d, _d, cint, dbl, dbl, cint, cint, u64, u64, _d, C.POINTER(_Report)],
        "rl_dev_randomized_genp_ex": [u64, u64, vp, vp, cint, dbl, dbl, cint, cint, u64, u64, vp,
                                      C.POINTER(_Report), C.c_uint32],
        "rl_randomized_genp_batched": [u64, u64, _d, _d, cint, dbl, dbl, cint, cint, u64, _u64a, _d, vp],
        "rl_dev_randomized_genp_batched": [u64, u64, vp, vp, cint, dbl, dbl, cint, cint, u64, vp, vp, vp],
        "rl_approx_basis": [u64, u64, _d, u64, dbl, dbl, cint, u64, u64, _d],
        "rl_qr_positive": [u64, u64, _d, _d, _d],
        "rl_project_onto_basis_left": [u64, u64, u64, _d, _d, vp, vp],
        "rl_numerical_rank": [u64, u64, _d, dbl, C.POINTER(u64), _d],
        "rl_dev_range_finder": [u64, u64, vp, u64, u64, u64, dbl, vp, vp, _d, C.POINTER(u64), C.POINTER(dbl)],
        "rl_dev_qr_positive": [u64, u64, vp, vp, vp],
        "rl_dev_numerical_rank": [u64, u64, vp, dbl, C.POINTER(u64), _d],
        "rl_probe_peaks": [C.POINTER(dbl), C.POINTER(dbl)],
        "rl_box_muller": [u64, vp, vp],
        "rl_last_column_reports": [u64, vp],
        "rl_extremal_sv_estimate": [u64, u64, _d, cint, cint, u64, u64, vp, vp],
        "rl_cond_probe": [u64, u64, _d, dbl, cint, cint, u64, u64, vp],
        "rl_nrank_search": [u64, u64, _d, u64, u64, dbl, cint, u64, u64, vp, _d, vp, vp],
        "rl_power_transform": [u64, u64, _d, C.c_uint, _d],
        "rl_box_muller_hash": [u64, u64, u64, vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = cint
    _lib = L
    return L


def _chk(code: int) -> None:
    if code != 0:
        msg = lib().rl_last_error().decode(errors="replace")
        raise _ERRORS.get(code, Error)(msg or f"rl status {code}")


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def launch_count() -> int:
    """Kernel launches made by librl_b200 in this process so far."""
    return int(lib().rl_launch_count())


def _ptr(t) -> int:
    """Device pointer of a CUDA tensor (torch is plumbing only)."""
    if not t.is_cuda or not t.is_contiguous():
        raise InvalidArgument("device arguments must be contiguous CUDA tensors")
    return t.data_ptr()


def _ptr64(t) -> int:
    """Device pointer of a contiguous float64 CUDA tensor."""
    import torch
    if t.dtype != torch.float64:
        raise InvalidArgument("device matrices must be float64")
    return _ptr(t)


def _bind_stream() -> None:
    """Run rl_dev_* calls on torch's current stream so events/timers see them."""
    import torch
    _chk(lib().rl_set_stream(torch.cuda.current_stream().cuda_stream))


# ------------------------------------------------------------- random_gen ----
def rng_draws(stream: RngStream, kind: str, count: int, lo: int = 0, hi: int = 1) -> np.ndarray:
    """Draws of one rnd::Rng method (random_gen.cpp:33-70) from a fresh Rng(stream)."""
    k = {"uniform01": 0, "uniform_pm1": 1, "gaussian": 2, "sign": 3, "uniform_int": 4}[kind]
    out = np.empty(count)
    _chk(lib().rl_rng_draws(stream.seed, stream.stream_id, k, count, lo, hi, out))
    return out


def raw_u64(stream: RngStream, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    _chk(lib().rl_raw_u64(stream.seed, stream.stream_id, count, out))
    return out


def gaussian_matrix(m: int, n: int, mu: float, sigma: float, stream: RngStream) -> np.ndarray:
    """rnd::gaussian_matrix (random_gen.cpp:72-80), bit-exact draws."""
    out = np.empty((m, n))
    _chk(lib().rl_gaussian_matrix(m, n, mu, sigma, stream.seed, stream.stream_id, out))
    return out


def uniform_matrix(m: int, n: int, stream: RngStream) -> np.ndarray:
    """rnd::uniform_matrix (random_gen.cpp:82-88)."""
    out = np.empty((m, n))
    _chk(lib().rl_uniform_matrix(m, n, stream.seed, stream.stream_id, out))
    return out


def random_structured(kind: MultiplierKind, m: int, n: int, stream: RngStream):
    """rnd::random_structured (random_gen.cpp:90-123) -> (first_col, first_row or None)."""
    col = np.empty(m)
    row = np.empty(n) if kind.tag == MultiplierTag.TOEPLITZ_GAUSSIAN else None
    _chk(lib().rl_random_structured(kind.tag, kind.mu, kind.sigma, m, n, stream.seed, stream.stream_id, col,
                                    row.ctypes.data if row is not None else None))
    return col, row


def householder_sign(n: int, stream: RngStream) -> np.ndarray:
    """rnd::householder_sign (random_gen.cpp:125-143): I - u v^T/(u^T v) (singular)."""
    out = np.empty((n, n))
    _chk(lib().rl_householder_sign(n, stream.seed, stream.stream_id, out))
    return out


def householder_pair_signs(n: int, stream: RngStream) -> Tuple[np.ndarray, np.ndarray]:
    u1, u2 = np.empty(n), np.empty(n)
    _chk(lib().rl_householder_pair_signs(n, stream.seed, stream.stream_id, u1, u2))
    return u1, u2


def sparse_sign(n: int, stream: RngStream, nnz: int = 4) -> Tuple[np.ndarray, np.ndarray]:
    rows = np.empty((n, nnz), np.int32)
    signs = np.empty((n, nnz))
    _chk(lib().rl_sparse_sign(n, nnz, stream.seed, stream.stream_id, rows, signs))
    return rows, signs


# ----------------------------------------------------------- matrix/struct ----
def multiply(a, b) -> np.ndarray:
    """Matrix::multiply (matrix.cpp:86-102) on the DMMA GEMM."""
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch("multiply: inner dimensions differ")
    c = np.empty((a.shape[0], b.shape[1]))
    _chk(lib().rl_matmul(a.shape[0], a.shape[1], b.shape[1], a, b, c))
    return c


def circ_mul(first_col, x) -> np.ndarray:
    """structured::circ_mul (structured.cpp:132-154)."""
    c, x = _f64(first_col), _f64(x)
    if len(x) != len(c):
        raise DimensionMismatch("circ_mul: vector length mismatch")
    y = np.empty(len(c))
    _chk(lib().rl_circ_mul(len(c), c, x, y))
    return y


def circulant_multiply_matrix(first_col, a) -> np.ndarray:
    """structured::multiply_matrix for a circulant spec (structured.cpp:178-189)."""
    c, a = _f64(first_col), _f64(a)
    if a.shape[0] != len(c):
        raise DimensionMismatch("multiply_matrix: inner dimensions differ")
    out = np.empty_like(a)
    _chk(lib().rl_circulant_multiply_matrix(len(c), c, a.shape[1], a, out))
    return out


def toeplitz_mul(first_col, first_row, x) -> np.ndarray:
    """structured::toeplitz_mul (structured.cpp:156-176): T x, T m x n."""
    c, r, x = _f64(first_col), _f64(first_row), _f64(x)
    if len(x) != len(r):
        raise DimensionMismatch("toeplitz_mul: vector length mismatch")
    y = np.empty(len(c))
    _chk(lib().rl_toeplitz_mul(len(c), len(r), c, r, x, y))
    return y


def toeplitz_multiply_matrix(first_col, first_row, a) -> np.ndarray:
    """structured::multiply_matrix for a Toeplitz spec: T A."""
    c, r, a = _f64(first_col), _f64(first_row), _f64(a)
    if a.shape[0] != len(r):
        raise DimensionMismatch("multiply_matrix: inner dimensions differ")
    out = np.empty((len(c), a.shape[1]))
    _chk(lib().rl_toeplitz_multiply_matrix(len(c), len(r), c, r, a.shape[1], a, out))
    return out


def fft(x, inverse: bool = False) -> np.ndarray:
    """structured::fft (structured.cpp:96-130), bit-identical to the reference, on the GPU."""
    z = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    out = np.empty_like(z)
    _chk(lib().rl_fft(len(z), z.ctypes.data, int(inverse), out.ctypes.data))
    return out


# ------------------------------------------------------------------- genp ----
def genp_factor(a, pivot_floor: float = 1e-300) -> GenpFactorization:
    """genp::genp_factor (genp.cpp:11-41): blocked no-pivot LU on the GPU."""
    a = _f64(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionMismatch("genp_factor: square matrix required")
    n = a.shape[0]
    L, U, piv, mm = np.empty((n, n)), np.empty((n, n)), np.empty(n), np.empty(2)
    step = C.c_int64(-1)
    _chk(lib().rl_genp_factor(n, a, pivot_floor, L, U, piv, mm, C.byref(step)))
    return GenpFactorization(L, U, piv, float(mm[0]), float(mm[1]))


def genp_solve(f: GenpFactorization, b) -> np.ndarray:
    """genp::genp_solve (genp.cpp:106-124); b may be n or n x nrhs."""
    b = _f64(b)
    n = f.L.shape[0]
    if b.shape[0] != n:
        raise DimensionMismatch("genp_solve: rhs length mismatch")
    nrhs = 1 if b.ndim == 1 else b.shape[1]
    x = np.empty_like(b)
    _chk(lib().rl_genp_solve(n, nrhs, _f64(f.L), _f64(f.U), b, x))
    return x


def _report(r: _Report, kind: MultiplierKind, refine: int) -> PrecondReport:
    return PrecondReport(kind, refine, r.residual, r.raw_residual, r.pivot_min, r.pivot_max, r.raw_pivot_min,
                         r.raw_pivot_max, r.attempt, r.attempts_drawn)


def randomized_genp(a, b, kind: MultiplierKind, side: int, refine: int,
                    stream: RngStream) -> Tuple[np.ndarray, PrecondReport]:
    """genp::randomized_genp (genp.cpp:207-291); b may be n or n x nrhs."""
    a, b = _f64(a), _f64(b)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or b.shape[0] != a.shape[0]:
        raise DimensionMismatch("randomized_genp: shape mismatch")
    n = a.shape[0]
    nrhs = 1 if b.ndim == 1 else b.shape[1]
    x = np.empty_like(b)
    rep = _Report()
    _chk(lib().rl_randomized_genp(n, nrhs, a, b, kind.tag, kind.mu, kind.sigma, side, refine, stream.seed,
                                  stream.stream_id, x, C.byref(rep)))
    return x, _report(rep, kind, refine)


def randomized_genp_batched(a, b, kind: MultiplierKind, side: int, refine: int, seed: int,
                            stream_ids: Sequence[int]):
    """Batched randomized_genp: system t uses RngStream(seed, stream_ids[t])."""
    a, b = _f64(a), _f64(b)
    batch, n = a.shape[0], a.shape[1]
    sids = np.ascontiguousarray(stream_ids, dtype=np.uint64)
    x = np.empty((batch, n))
    reps = (_Report * batch)()
    _chk(lib().rl_randomized_genp_batched(batch, n, a, b, kind.tag, kind.mu, kind.sigma, side, refine, seed,
                                          sids, x, C.cast(reps, vp)))
    return x, [_report(r, kind, refine) for r in reps]


# ---------------------------------------------------------- lowrank/dense ----
def approx_basis(a, rho_plus: int, kind: MultiplierKind, side: int, stream: RngStream) -> np.ndarray:
    """lowrank::approx_basis, Gaussian kind (lowrank.cpp:67-84); side 0 = LeftSpace (A H)."""
    if kind.tag != MultiplierTag.GAUSSIAN:
        raise InvalidArgument("approx_basis: only the Gaussian kind is on the B200 path")
    a = _f64(a)
    m, n = a.shape
    y = np.empty((m if side == 0 else n, rho_plus))
    _chk(lib().rl_approx_basis(m, n, a, rho_plus, kind.mu, kind.sigma, side, stream.seed, stream.stream_id, y))
    return y


def qr_positive(a) -> Tuple[np.ndarray, np.ndarray]:
    """dense::qr_positive (dense_core.cpp:86-115)."""
    a = _f64(a)
    m, n = a.shape
    q, r = np.empty((m, n)), np.empty((n, n))
    _chk(lib().rl_qr_positive(m, n, a, q, r))
    return q, r


def project_onto_basis(a, basis, orthonormal: bool = True, side: str = "left"):
    """lowrank::project_onto_basis, orthonormal Side::Left (lowrank.cpp:61-64) -> (Q Q^T A, Q^T A)."""
    if not orthonormal or side != "left":
        raise InvalidArgument("project_onto_basis: only the orthonormal Side::Left form is on the B200 path")
    a, q = _f64(a), _f64(basis)
    if q.shape[0] != a.shape[0]:
        raise DimensionMismatch("project_onto_basis: basis row count mismatch")
    m, n, k = a.shape[0], a.shape[1], q.shape[1]
    sta, out = np.empty((k, n)), np.empty((m, n))
    _chk(lib().rl_project_onto_basis_left(m, n, k, a, q, sta.ctypes.data, out.ctypes.data))
    return out, sta


def numerical_rank(a, tol: float) -> Tuple[int, np.ndarray]:
    """dense::numerical_rank (dense_core.cpp:171-175) -> (rank, singular values)."""
    a = _f64(a)
    m, n = a.shape
    r = u64(0)
    sg = np.empty(min(m, n))
    _chk(lib().rl_numerical_rank(m, n, a, tol, C.byref(r), sg))
    return int(r.value), sg


# ------------------------------------------------------------------ device ----
def dev_gemm(a, b, c, alpha=1.0, beta=0.0, trans_a=False, trans_b=False) -> None:
    _bind_stream()
    m = a.shape[1] if trans_a else a.shape[0]
    k = a.shape[0] if trans_a else a.shape[1]
    n = b.shape[0] if trans_b else b.shape[1]
    _chk(lib().rl_dev_gemm(int(trans_a), int(trans_b), m, n, k, alpha, _ptr(a), a.shape[1], _ptr(b),
                           b.shape[1], beta, _ptr(c), c.shape[1]))


def dev_gaussian_matrix(out, mu: float, sigma: float, stream: RngStream) -> None:
    _bind_stream()
    _chk(lib().rl_dev_gaussian_matrix(out.shape[0], out.shape[1], mu, sigma, stream.seed, stream.stream_id,
                                      _ptr(out)))


def dev_genp_factor(a, pivot_floor: float = 1e-300, pivots=None):
    """In-place packed blocked GENP on a CUDA tensor; returns the |pivots| tensor."""
    import torch
    _bind_stream()
    n = a.shape[0]
    piv = pivots if pivots is not None else torch.empty(n, dtype=torch.float64, device=a.device)
    step = C.c_int64(-1)
    _chk(lib().rl_dev_genp_factor(n, _ptr(a), a.shape[1], pivot_floor, _ptr(piv), C.byref(step)))
    return piv


def dev_genp_solve(lu, b) -> None:
    """In-place multi-RHS solve with a packed LU (b: n x nrhs CUDA tensor)."""
    _bind_stream()
    nrhs = 1 if b.dim() == 1 else b.shape[1]
    _chk(lib().rl_dev_genp_solve_packed(lu.shape[0], nrhs, _ptr(lu), lu.shape[1], _ptr(b)))


def dev_randomized_genp(a, b, x, kind: MultiplierKind, side: int, refine: int, stream: RngStream,
                        skip_raw_arm: bool = False) -> PrecondReport:
    _bind_stream()
    n = a.shape[0]
    nrhs = 1 if b.dim() == 1 else b.shape[1]
    rep = _Report()
    _chk(lib().rl_dev_randomized_genp_ex(n, nrhs, _ptr(a), _ptr(b), kind.tag, kind.mu, kind.sigma, side, refine,
                                         stream.seed, stream.stream_id, _ptr(x), C.byref(rep),
                                         1 if skip_raw_arm else 0))
    return _report(rep, kind, refine)


def last_column_reports(nrhs: int):
    """Per-column outcome of this thread's last randomized_genp call (rl_last_column_reports):
    a list of (attempt, attempts_drawn, residual, pivot_min, pivot_max)."""
    arr = (_ColumnReport * nrhs)()
    _chk(lib().rl_last_column_reports(nrhs, arr))
    return [(c.attempt, c.attempts_drawn, c.residual, c.pivot_min, c.pivot_max) for c in arr]


def dev_randomized_genp_batched(a, b, x, kind: MultiplierKind, side: int, refine: int, seed: int, sids,
                                reports=None) -> None:
    """a: batch x n x n, b/x: batch x n, sids: uint64-valued int64 CUDA tensor; reports: optional
    CUDA uint8 tensor of batch * 56 bytes (rl_precond_report)."""
    _bind_stream()
    batch, n = a.shape[0], a.shape[1]
    _chk(lib().rl_dev_randomized_genp_batched(batch, n, _ptr(a), _ptr(b), kind.tag, kind.mu, kind.sigma, side,
                                              refine, seed, _ptr(sids), _ptr(x),
                                              _ptr(reports) if reports is not None else None))


def dev_range_finder(a, rho_plus: int, stream: RngStream, rank_tol: float, q, bmat, want_residual=True):
    """Fused range finder on device data -> (sigma(B), rank, ||A - QB||_F/||A||_F or None)."""
    _bind_stream()
    m, n = a.shape
    sg = np.empty(rho_plus)
    r = u64(0)
    res = dbl(0.0)
    _chk(lib().rl_dev_range_finder(m, n, _ptr(a), rho_plus, stream.seed, stream.stream_id, rank_tol, _ptr(q),
                                   _ptr(bmat), sg, C.byref(r), C.byref(res) if want_residual else None))
    return sg, int(r.value), (res.value if want_residual else None)


def sparse_apply_right(rows, signs, a) -> np.ndarray:
    """A S for the sparse +-1 multiplier (rows, signs: n x nnz per column of S)."""
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    signs, a = _f64(signs), _f64(a)
    n, nnz = rows.shape
    if a.shape != (n, n) or signs.shape != rows.shape:
        raise DimensionMismatch("sparse_apply_right: shape mismatch")
    out = np.empty_like(a)
    _chk(lib().rl_sparse_apply_right(n, nnz, rows, signs, a, out))
    return out


def dev_sparse_apply_right(rows, signs, a, out) -> None:
    """out = A S on device tensors (rows int32 n x nnz, signs/a/out float64)."""
    _bind_stream()
    n, nnz = rows.shape
    if a.shape != (n, n) or out.shape != (n, n) or signs.shape != rows.shape:
        raise DimensionMismatch("sparse_apply_right: shape mismatch")
    _chk(lib().rl_dev_sparse_apply_right(n, nnz, _ptr(rows), _ptr(signs), _ptr(a), _ptr(out)))


def dev_householder_pair_apply_right(u1, u2, a, out) -> None:
    """out = A H1 H2 on device tensors, H_i = I - (2/n) u_i u_i^T (u_i +-1 vectors)."""
    _bind_stream()
    n = a.shape[0]
    if a.shape != (n, n) or out.shape != (n, n) or u1.shape[0] != n or u2.shape[0] != n:
        raise DimensionMismatch("householder_pair_apply_right: shape mismatch")
    _chk(lib().rl_dev_householder_pair_apply_right(n, _ptr(u1), _ptr(u2), _ptr(a), _ptr(out)))


def dev_circulant_apply_right(c, a, out) -> None:
    """out = A C on device tensors for the circulant with first column c (FFT for power-of-two
    64 <= n <= 8192)."""
    _bind_stream()
    m, n = a.shape
    if c.shape[0] != n or out.shape != (m, n):
        raise DimensionMismatch("circulant_apply_right: shape mismatch")
    _chk(lib().rl_dev_circulant_apply_right(m, n, _ptr(c), _ptr(a), _ptr(out)))


def dev_toeplitz_apply_right(col, row, a, out) -> None:
    """out = A T on device tensors for the Toeplitz with first column col and first row row
    (row[0] == col[0]); FFT of the circulant embedding when next_pow2(2n - 1) <= 8192."""
    import torch
    _bind_stream()
    m, n = a.shape
    if col.shape[0] != n or row.shape[0] != n or out.shape != (m, n):
        raise DimensionMismatch("toeplitz_apply_right: shape mismatch")
    g = torch.cat([col, row[1:]]).contiguous()
    _chk(lib().rl_dev_toeplitz_apply_right(m, n, _ptr(g), _ptr(a), _ptr(out)))
    torch.cuda.current_stream().synchronize()  # g is a temporary


def proto_lowrank(a, rho_plus: int, tau: float, tau_prime: float, kind: MultiplierKind, stream: RngStream):
    """lowrank::proto_lowrank (lowrank.cpp:108-177), Gaussian / ToeplitzGaussian kinds: (rho,
    basis n x rho, approx, residual, ok)."""
    a = _f64(a)
    m, n = a.shape
    basis, approx = np.empty((n, rho_plus)), np.empty((m, n))
    rho, res, ok = C.c_uint64(0), C.c_double(0.0), C.c_int(0)
    _chk(lib().rl_proto_lowrank(m, n, a, rho_plus, tau, tau_prime, kind.tag, kind.mu, kind.sigma, stream.seed,
                                stream.stream_id, C.byref(rho), basis, approx, C.byref(res), C.byref(ok)))
    return rho.value, basis[:, :rho.value].copy(), approx, res.value, bool(ok.value)


def dev_qr_positive(y, q, r) -> None:
    """dense::qr_positive on device data: q (m x n), r (n x n) with diag(r) > 0 (n <= 128)."""
    _bind_stream()
    m, n = y.shape
    _chk(lib().rl_dev_qr_positive(m, n, _ptr64(y), _ptr64(q), _ptr64(r)))


def dev_numerical_rank(a, tol: float) -> Tuple[int, np.ndarray]:
    """dense::numerical_rank of device data -> (rank, singular values), min(m, n) <= 128."""
    _bind_stream()
    m, n = a.shape
    r = u64(0)
    sg = np.empty(min(m, n))
    _chk(lib().rl_dev_numerical_rank(m, n, _ptr64(a), tol, C.byref(r), sg))
    return int(r.value), sg


class SvMethod:
    POWER = 0
    LANCZOS = 1


class SearchPolicy:
    BINARY = 0
    LINEAR_DOWN = 1


def extremal_sv_estimate(a, method: int, iters: int, stream: RngStream) -> Tuple[float, float]:
    """lowrank::extremal_sv_estimate (lowrank.cpp:204-348) -> (sv_max, sv_min)."""
    a = _f64(a)
    hi, lo = dbl(0.0), dbl(0.0)
    _chk(lib().rl_extremal_sv_estimate(a.shape[0], a.shape[1], a, method, iters, stream.seed, stream.stream_id,
                                       C.byref(hi), C.byref(lo)))
    return hi.value, lo.value


def cond_probe(b, kappa: float, method: int, iters: int, stream: RngStream) -> bool:
    """lowrank::cond_probe (lowrank.cpp:350-358)."""
    b = _f64(b)
    ok = C.c_int(0)
    _chk(lib().rl_cond_probe(b.shape[0], b.shape[1], b, kappa, method, iters, stream.seed, stream.stream_id,
                             C.byref(ok)))
    return bool(ok.value)


def nrank_search(a, rho_minus: int, rho_plus: int, kappa: float, policy: int, stream: RngStream):
    """lowrank::nrank_search (lowrank.cpp:360-396) -> (rho, basis)."""
    a = _f64(a)
    m, n = a.shape
    basis = np.zeros(max(m, n) * max(rho_plus, 1))
    rho, br, bc = u64(0), u64(0), u64(0)
    _chk(lib().rl_nrank_search(m, n, a, rho_minus, rho_plus, kappa, policy, stream.seed, stream.stream_id,
                               C.byref(rho), basis, C.byref(br), C.byref(bc)))
    return int(rho.value), basis[:br.value * bc.value].reshape(br.value, bc.value).copy()


def power_transform(a, h: int) -> np.ndarray:
    """lowrank::power_transform (lowrank.cpp:179-187): (A A^T)^h A."""
    a = _f64(a)
    out = np.empty_like(a)
    _chk(lib().rl_power_transform(a.shape[0], a.shape[1], a, h, out))
    return out


def box_muller(raw) -> np.ndarray:
    """Rng::gaussian's Box-Muller (random_gen.cpp:46-52) of consecutive raw u64 pairs on the GPU:
    out[2q] = r cos a, out[2q + 1] = r sin a."""
    raw = np.ascontiguousarray(raw, dtype=np.uint64)
    out = np.empty(raw.size, dtype=np.float64)
    _chk(lib().rl_box_muller(raw.size // 2, raw.ctypes.data, out.ctypes.data))
    return out


def box_muller_hash(seed: int, npairs: int, chunk: int = 1 << 20) -> np.ndarray:
    """Per-chunk checksums of the GPU Box-Muller over splitmix64 pairs (rl_b200.h)."""
    out = np.zeros((npairs + chunk - 1) // chunk, dtype=np.uint64)
    _chk(lib().rl_box_muller_hash(seed, npairs, chunk, out.ctypes.data))
    return out


def probe_peaks() -> Tuple[float, float]:
    """K12: measured FP64 DMMA TFLOP/s and HBM copy GB/s on the current device."""
    f, h = dbl(0), dbl(0)
    _chk(lib().rl_probe_peaks(C.byref(f), C.byref(h)))
    return f.value, h.value

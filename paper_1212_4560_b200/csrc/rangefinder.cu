// K9/K10/K11: the randomized range finder (config 4) and its dense-core pieces.
//
// Reference calls:
//   lowrank::approx_basis  Y = A H, H = gaussian_matrix(n, rho+)  (lowrank.cpp:67-84)
//   dense::qr_positive     thin Q, R with diag(R) > 0, rank check
//                          min|R_ii| > 1e-13 sigma_1(R)           (dense_core.cpp:86-115)
//   lowrank::project_onto_basis (Left, orthonormal): sta = Q^T A  (lowrank.cpp:61-64)
//   dense::numerical_rank  largest j with sigma_j >= tol sigma_1  (dense_core.cpp:161-175)
//
// B200 design: every contraction is the DMMA GEMM (split-K with a fixed-order
// reduction where one output tile would leave SMs idle: Y^T Y, Q^T A).  QR of the
// tall-skinny Y is shifted CholeskyQR3 (Gram on DMMA, 72x72 Cholesky and triangular
// inverse in one CTA, Q = Y R^-1 on DMMA): Householder-grade orthogonality for
// kappa(Y) up to ~1e15 (plain CholQR2 is borderline at kappa 1.2e7).
// sigma(B) comes from the R factor of B^T (never from the squared Gram B B^T) and a
// one-sided Jacobi SVD of that 72x72 R in one CTA.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rl_internal.cuh"

namespace rl {

void copy2d_dev(uint64_t rows, uint64_t cols, const double* src, uint64_t lds, double* dst, uint64_t ldd);
void gemm_splitk_parts(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, const double* a, uint64_t lda,
                       const double* b, uint64_t ldb, double* parts, int splits, uint64_t kchunk);
uint64_t gemm_tiles(uint64_t m, uint64_t n);

namespace {

constexpr int KMAX = 128; // largest rho+ handled by the single-CTA small kernels

// Small outputs (a Gram): one warp per output element, lane l sums slices l, l+32, ... and a
// fixed shuffle tree combines them (deterministic; enough threads to pull the partials at HBM
// rate where one thread per element left most SMs idle).
__global__ void k_splitk_reduce_warp(uint64_t m, uint64_t n, int splits, const double* parts, double alpha,
                                     double beta, double* c, uint64_t ldc) {
    const uint64_t total = m * n;
    const uint64_t e = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= total) // whole warps exit together (e is warp-uniform)
        return;
    double s = 0.0;
    for (int p = lane; p < splits; p += 32)
        s += parts[p * total + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        const uint64_t i = e / n, j = e % n;
        double v = alpha * s;
        if (beta != 0.0)
            v = fma(beta, c[i * ldc + j], v);
        c[i * ldc + j] = v;
    }
}

__global__ void k_splitk_reduce(uint64_t m, uint64_t n, int splits, const double* parts, double alpha,
                                double beta, double* c, uint64_t ldc) {
    uint64_t total = m * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < splits; ++p)
            s += parts[p * total + e];
        uint64_t i = e / n, j = e % n;
        double v = alpha * s;
        if (beta != 0.0)
            v = fma(beta, c[i * ldc + j], v);
        c[i * ldc + j] = v;
    }
}

// Even n / ldc, < 2^32 outputs: two adjacent outputs per thread (16-byte loads and stores),
// 32-bit index arithmetic (the 64-bit e / n of the general kernel dominated A H's 9.4 MB
// reduction); the same summation order as k_splitk_reduce.
__global__ void k_splitk_reduce2(uint32_t n, uint32_t total, int splits, const double* __restrict__ parts,
                                 double alpha, double beta, double* __restrict__ c, uint32_t ldc) {
    const uint32_t e = 2u * (blockIdx.x * blockDim.x + threadIdx.x);
    if (e >= total)
        return;
    double2 s = make_double2(0.0, 0.0);
    for (int p = 0; p < splits; ++p) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(parts + static_cast<uint64_t>(p) * total + e));
        s.x += v.x;
        s.y += v.y;
    }
    const uint32_t i = e / n, j = e - i * n;
    double2* cp = reinterpret_cast<double2*>(c + static_cast<uint64_t>(i) * ldc + j);
    double2 v = make_double2(alpha * s.x, alpha * s.y);
    if (beta != 0.0) {
        const double2 o = *cp;
        v.x = fma(beta, o.x, v.x);
        v.y = fma(beta, o.y, v.y);
    }
    *cp = v;
}

// Reciprocal and reciprocal square root from the SFU seed plus two Newton steps (a few ulp;
// no IEEE slow path): the Jacobi rotation only needs c^2 + s^2 = 1 to rounding level.
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    return y * fma(-h * y, y, 1.5);
}

// Cholesky G + shift I = R^T R and X = R^-1 for k <= 128 in one 512-thread CTA, in shared
// memory (k padded to KP = 8 ceil(k/8) with an identity corner), 8-column blocks J, three
// barriers per block:
//   A  warp 0 factors the 8 x 8 diagonal block in registers (lane c holds column c, pivot
//      rows by shuffle) and inverts it (X_JJ) — for blocks after the first, inside the
//      previous block's phase C (lookahead: it first applies that block's update to its own
//      8 x 8, then factors, while warps 1-15 do the rest of C);
//   B  one thread per trailing column solves the block's panel row R_J,rest; the others form
//      T = R_0:J,J X_JJ;
//   C  rank-8 update of the trailing upper triangle; X_0:J,J = -X_0:J,0:J T.
// X_ij (i < j) lives in the free lower triangle at W[j][i], its diagonal in rdiag.
//   shift = shift_coef * sum(shift_part[0..nshift))    (pass 0 of CholeskyQR3; else 0)
// g <- R (upper, zeros below), rinv <- R^-1.  *bad is sticky: a kernel whose earlier pass
// failed returns at once; a non-positive pivot sets it.
constexpr int CH_T = 512;
// Warp 0: factor the 8 x 8 diagonal block at (c0, c0) of W in registers (lane c holds column
// c, pivot rows by shuffle) -> R_JJ (upper) and rdiag = 1 / R_tt, then X_JJ = R_JJ^-1 by back
// substitution, stored transposed in the free lower triangle (X_rc at W[c0+c][c0+r]).
__device__ __forceinline__ void chol_diag8(double* W, int P, int c0, double* rdiag, int lane, int* s_bad) {
    const int c = lane & 7;
    double col[8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
        col[r] = W[(c0 + r) * P + c0 + c];
    bool ok = true;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const double d = __shfl_sync(0xffffffffu, col[t], t);
        ok = ok && (d > 0.0);
        const double inv = rsqrt_nr(d); // 1 / R_tt
        const double rtc = (c == t) ? d * inv : col[t] * inv; // R_{t,c} (c >= t)
        col[t] = rtc;
        if (c == t)
            rdiag[c0 + t] = inv;
#pragma unroll
        for (int r = t + 1; r < 8; ++r) {
            const double rtr = __shfl_sync(0xffffffffu, rtc, r); // R_{t,r}
            col[r] = fma(-rtr, rtc, col[r]);
        }
    }
    if (lane < 8) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
            if (r <= c)
                W[(c0 + r) * P + c0 + c] = col[r];
    }
    __syncwarp();
    if (lane < 8) {
        double x[8];
#pragma unroll
        for (int r = 7; r >= 0; --r) {
            double v = 0.0;
#pragma unroll
            for (int l = r + 1; l < 8; ++l)
                if (l <= c)
                    v = fma(W[(c0 + r) * P + c0 + l], x[l], v);
            x[r] = (r == c) ? rdiag[c0 + c] : (r < c ? -v * rdiag[c0 + r] : 0.0);
            if (r < c)
                W[(c0 + c) * P + c0 + r] = x[r];
        }
    }
    if (lane == 0 && !ok)
        *s_bad = 1;
}
// G (k x k, read-only) -> R (upper) and R^-1 in shared memory; writes rinv and the accumulated
// factor racc_out = R (racc_in null) or R racc_in (both upper triangular: CholeskyQR3's
// R_acc = R_pass R_acc, rows over warps, columns over lanes, ascending l).
__global__ void __launch_bounds__(CH_T) k_chol_inv(int k, const double* g, const double* shift_part, int nshift,
                                                   double shift_coef, double* rinv, const double* racc_in,
                                                   double* racc_out, int* bad, int diag_only) {
    extern __shared__ double W[]; // KP x (KP + 1)
    __shared__ double rdiag[KMAX];
    __shared__ double T[8][KMAX + 1]; // T[c][l] = (R_0:J,J X_JJ)[l][c]; padded: 8 c's hit 8 banks
    __shared__ double s_shift;
    __shared__ int s_bad;
    if (*bad)
        return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int KP = (k + 7) & ~7, P = KP + 1;
    if (warp == 0) {
        double p = 0.0;
        if (shift_part)
            for (int i = lane; i < nshift; i += 32)
                p += shift_part[i];
        for (int o = 16; o > 0; o >>= 1)
            p += __shfl_xor_sync(0xffffffffu, p, o);
        if (lane == 0) {
            s_shift = shift_coef * p;
            s_bad = 0;
        }
    }
    __syncthreads();
    const double shift = s_shift;
    for (int e = tid; e < KP * KP; e += CH_T) {
        const int i = e / KP, l = e - i * KP;
        double v;
        if (i < k && l < k)
            v = g[i * k + l] + (i == l ? shift : 0.0);
        else
            v = (i == l) ? 1.0 : 0.0;
        W[i * P + l] = v;
    }
    __syncthreads();
    if (warp == 0)
        chol_diag8(W, P, 0, rdiag, lane, &s_bad);
    __syncthreads();
    if (s_bad) { // uniform
        if (tid == 0)
            *bad = 1;
        return;
    }
    for (int c0 = 0; c0 < KP; c0 += 8) {
        // ---- B: panel row of R; T = R_0:J,J X_JJ   (R_JJ, X_JJ: the previous step's lookahead)
        const int rest = KP - c0 - 8;
        if (tid < rest) { // R_{c0+t, l} = (W_{c0+t, l} - sum_{s<t} R_{c0+s, c0+t} R_{c0+s, l}) / R_tt
            const int l = c0 + 8 + tid;
            double x[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                double v = W[(c0 + t) * P + l];
#pragma unroll
                for (int s2 = 0; s2 < t; ++s2)
                    v = fma(-W[(c0 + s2) * P + c0 + t], x[s2], v);
                x[t] = v * rdiag[c0 + t];
                W[(c0 + t) * P + l] = x[t];
            }
        }
        for (int e = tid - rest; e >= 0 && e < 8 * c0; e += CH_T - rest) { // threads >= rest
            const int l = e >> 3, c = e & 7; // T[l][c] = sum_{m <= c} R_{l, c0+m} X_JJ[m][c]
            double v = 0.0;
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (m <= c) {
                    const double xm = (m == c) ? rdiag[c0 + c] : W[(c0 + c) * P + c0 + m];
                    v = fma(W[l * P + c0 + m], xm, v);
                }
            T[c][l] = v;
        }
        __syncthreads();
        // ---- C: warp 0 brings the next diagonal block up to date and factors it (lookahead);
        // warps 1-15 update the rest of the trailing triangle and form X_0:J,J
        if (warp == 0) {
            if (rest > 0) {
                const int l = c0 + 8 + (lane & 7);
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int i = c0 + 8 + (lane >> 3) + 4 * r;
                    if (i <= l) {
                        double v = W[i * P + l];
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            v = fma(-W[(c0 + t) * P + i], W[(c0 + t) * P + l], v);
                        W[i * P + l] = v;
                    }
                }
                __syncwarp();
                chol_diag8(W, P, c0 + 8, rdiag, lane, &s_bad);
            }
        } else {
            const int nd = c0 + 16; // the next diagonal block [c0 + 8, c0 + 16)^2 is warp 0's
            if (rest > 0) {
                for (int i = c0 + 8 + (warp - 1); i < KP; i += 15) {
                    double pi[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        pi[t] = W[(c0 + t) * P + i];
                    const int lstart = i < nd ? nd : i; // upper triangle, minus warp 0's block
                    for (int l = lstart + ((lane - lstart) & 31); l < KP; l += 32) {
                        double v = W[i * P + l];
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            v = fma(-pi[t], W[(c0 + t) * P + l], v);
                        W[i * P + l] = v;
                    }
                }
            }
            for (int e = tid - 32; e < 8 * c0; e += CH_T - 32) { // X_{i, c0+c} = -sum_{l=i}^{c0-1} X_il T[l][c]
                const int i = e >> 3, c = e & 7;
                double v0 = rdiag[i] * T[c][i], v1 = 0.0, v2 = 0.0, v3 = 0.0;
                int l = i + 1;
                for (; l + 3 < c0; l += 4) { // four chains: the loads pipeline
                    v0 = fma(W[l * P + i], T[c][l], v0);
                    v1 = fma(W[(l + 1) * P + i], T[c][l + 1], v1);
                    v2 = fma(W[(l + 2) * P + i], T[c][l + 2], v2);
                    v3 = fma(W[(l + 3) * P + i], T[c][l + 3], v3);
                }
                for (; l < c0; ++l)
                    v0 = fma(W[l * P + i], T[c][l], v0);
                W[(c0 + c) * P + i] = -((v0 + v1) + (v2 + v3));
            }
        }
        __syncthreads();
        if (s_bad) { // uniform
            if (tid == 0)
                *bad = 1;
            return;
        }
    }
    for (int e = tid; e < k * k; e += CH_T) {
        const int i = e / k, l = e - i * k;
        rinv[e] = (l > i) ? W[l * P + i] : (l == i ? rdiag[i] : 0.0);
        if (!racc_in && !diag_only)
            racc_out[e] = (l >= i) ? W[i * P + l] : 0.0;
    }
    if (diag_only) { // only diag(R_acc) = diag(R_pass) .* diag(R_acc_in) (triangular product)
        for (int i = tid; i < k; i += CH_T)
            racc_out[i] = racc_in ? W[i * P + i] * racc_in[i] : W[i * P + i];
        return;
    }
    if (racc_in) { // R_acc = R_pass R_acc_in: R_acc_in (upper) transposed into W's lower half, now free
        __syncthreads(); // X (lower half) and rdiag consumed by the rinv write
        for (int e = tid; e < k * k; e += CH_T) {
            const int l = e / k, j = e - l * k;
            if (j > l)
                W[j * P + l] = racc_in[e];
            else if (j == l)
                rdiag[l] = racc_in[e];
        }
        __syncthreads();
        for (int i = warp; i < k; i += CH_T / 32) { // warp per row i, lane per column j
            const double* wi = W + i * P;
            for (int j = lane; j < k; j += 32) {
                double v = 0.0;
                if (j >= i) { // sum_{l=i..j} R_il Racc_lj: four chains, the diagonal term last
                    const double* wj = W + j * P;
                    double v1 = 0.0, v2 = 0.0, v3 = 0.0;
                    int l = i;
                    for (; l + 3 < j; l += 4) {
                        v = fma(wi[l], wj[l], v);
                        v1 = fma(wi[l + 1], wj[l + 1], v1);
                        v2 = fma(wi[l + 2], wj[l + 2], v2);
                        v3 = fma(wi[l + 3], wj[l + 3], v3);
                    }
                    for (; l < j; ++l)
                        v = fma(wi[l], wj[l], v);
                    v = fma(wi[j], rdiag[j], (v + v1) + (v2 + v3));
                }
                racc_out[static_cast<size_t>(i) * k + j] = v;
            }
        }
    }
}

// Singular values of a k x k matrix (row-major, ld k, k <= 128) by one-sided Jacobi on the
// columns of its transpose (= its rows: for the triangular factors this is fed, fewer sweeps
// than on its columns).  Four lanes per column pair, eight pairs per warp, all k/2 pairs of a
// round at once (round-robin "circle" pairing computed from the round index: slot kk-1
// fixed, the others rotate), one barrier per round.  The kernel is issue-bound on its one
// SM, so a pair's dot products, reductions and rotation are shared by as few warps as
// possible.  A sweep rotates every pair whose cosine |a_p.a_q| / (|a_p||a_q|) exceeds 1e-15;
// the iteration stops after a sweep with no rotation.  sigma (non-increasing) = final
// column norms; sigma[KMAX] = sweeps used.  NE >= ceil(k / 4) elements per lane.
constexpr int JS_T = 256;
template <int NE>
__global__ void __launch_bounds__(JS_T) k_jacobi_sv(int k, const double* a, double* sigma) {
    extern __shared__ double w[]; // column j (= row j of a) at w + j * k
    __shared__ double nrm[KMAX];
    __shared__ int rotated[3];
    const int tid = threadIdx.x, pg = tid >> 2, pl = tid & 3, warp = tid >> 5;
    const int kk = (k + 1) & ~1; // even slot count (one dummy column when k is odd)
    const int npairs = kk / 2;
    for (int e = tid; e < k * k; e += JS_T)
        w[e] = a[e];
    if (tid < 3)
        rotated[tid] = 0;
    __syncthreads();
    // rotate while |cos| = |a_p . a_q| / (|a_p| |a_q|) exceeds k eps (LAPACK dgesvj's test is
    // sqrt(m) eps; a bar below the dot products' own rounding floor, ~sqrt(k) eps, never settles)
    const double tol = static_cast<double>(k) * 2.220446049250313e-16;
    const bool warp_live = warp * 8 < npairs; // warp-uniform
    int sweep = 0;
    for (; sweep < 60; ++sweep) {
        if (tid == 0)
            rotated[(sweep + 1) % 3] = 0;
        for (int round = 0; round < kk - 1; ++round) {
            if (warp_live) {
                int p = kk - 1, q = round; // pair 0
                if (pg > 0) {
                    p = round + pg;
                    if (p >= kk - 1)
                        p -= kk - 1;
                    q = round - pg;
                    if (q < 0)
                        q += kk - 1;
                }
                const bool live = pg < npairs && p < k && q < k;
                if (p > q) {
                    int t = p;
                    p = q;
                    q = t;
                }
                double* wp = w + (live ? p : 0) * k;
                double* wq = w + (live ? q : 0) * k;
                double xs[NE], ys[NE];
                double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
                for (int r = 0; r < NE; ++r) {
                    const int i = pl + 4 * r;
                    const bool in = live && i < k;
                    xs[r] = in ? wp[i] : 0.0;
                    ys[r] = in ? wq[i] : 0.0;
                    al = fma(xs[r], xs[r], al);
                    be = fma(ys[r], ys[r], be);
                    ga = fma(xs[r], ys[r], ga);
                }
#pragma unroll
                for (int o = 2; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
                    if (pl == 0)
                        rotated[sweep % 3] = 1;
                    const double zeta = (be - al) * 0.5 * rcp_nr(ga);
                    const double v = fma(zeta, zeta, 1.0);
                    const double t = copysign(rcp_nr(fabs(zeta) + v * rsqrt_nr(v)), zeta);
                    const double c = rsqrt_nr(fma(t, t, 1.0)), s = c * t;
#pragma unroll
                    for (int r = 0; r < NE; ++r) {
                        const int i = pl + 4 * r;
                        if (i < k) {
                            wp[i] = c * xs[r] - s * ys[r];
                            wq[i] = s * xs[r] + c * ys[r];
                        }
                    }
                }
            }
            __syncthreads();
        }
        if (!rotated[sweep % 3])
            break;
    }
    for (int j0 = 0; j0 < k; j0 += JS_T / 4) { // trip count uniform: the shuffles span the warp
        const int j = j0 + pg;
        double s = 0.0;
        if (j < k)
            for (int i = pl; i < k; i += 4)
                s = fma(w[j * k + i], w[j * k + i], s);
        for (int o = 2; o > 0; o >>= 1)
            s += __shfl_xor_sync(0xffffffffu, s, o);
        if (pl == 0 && j < k)
            nrm[j] = sqrt(s);
    }
    __syncthreads();
    if (tid < k) { // rank sort, descending, ties by index
        const double v = nrm[tid];
        int rank = 0;
        for (int i = 0; i < k; ++i) {
            const double u = nrm[i];
            rank += (u > v) || (u == v && i < tid);
        }
        sigma[rank] = v;
    }
    if (tid == 0)
        sigma[KMAX] = sweep + 1;
}

// Singular values of a k x k matrix (row-major, ld k, 16 <= k <= 128): Householder
// bidiagonalization then multisection on the Golub-Kahan form, one 512-thread CTA.  This is
// the reference's own split (dense_core.cpp:28-43: BDCSVD from min(rows, cols) >= 16, which
// is backward stable, i.e. absolutely accurate to ~u sigma_1; Jacobi below that).
//   Bidiagonalization, two barriers per column j.  Every warp forms the left reflector of
//   column j itself from the squares the previous phase left in sq[] (no broadcast barrier),
//   then four threads per column c > j apply it to column c and record row j's new squares in
//   sq2[]; every warp forms the right reflector of row j from sq2[], four threads per row r > j
//   apply it and record column j+1's squares in sq[].
//   sigma: the 2k x 2k tridiagonal TGK(d, e) (zero diagonal, off-diagonals d0 e0 d1 ...
//   d_{k-1}) has eigenvalues +-sigma_i, so #{sigma_i < x} = #{negative pivots of TGK - x I}
//   - k.  The pivots are ratios of leading (top) and trailing (bottom) minors; the minors'
//   three-term recurrences need one FMA per step on the dependency chain (the pivot form
//   needs a division), rescaled by powers of two every 8 steps, and the two chains meet at
//   row k (twisted factorization).  d, e are pre-scaled by a power of two to sigma_max ~ 1.
//   Each round every unconverged interval gets G = 3 probe points (one thread each);
//   intervals shrink 4x per round to width 2^-52 sigma_max.
constexpr int BD_SUB = 4; // threads per reflector dot product (8 per column x 1024 threads measured slower)
constexpr int BD_T = 512;  // up to 128 columns x 4 threads
// Row pitch = 4 (mod 16) doubles: a half-warp touching 4 rows x 4 consecutive columns hits
// 16 distinct 8-byte bank pairs (the updates are shared-memory-bandwidth bound).
__host__ __device__ constexpr int bd_pitch(int k) { return k + ((4 - k) & 15); }
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// sum of v[lo .. hi) (hi - lo <= 128), the same value in every lane of every warp
__device__ __forceinline__ double range_sum(const double* v, int lo, int hi, int lane) {
    double t = 0.0;
    for (int i = lo + lane; i < hi; i += 32)
        t += v[i];
    return warp_sum(t);
}
// power-of-two rescale of the pair (a, b) so that max(|a|, |b|) lies in [1, 2)
__device__ __forceinline__ void rescale2(double& a, double& b) {
    const int ea = (__double2hiint(a) >> 20) & 0x7ff, eb = (__double2hiint(b) >> 20) & 0x7ff;
    const int e = max(ea, eb);
    if (e > 0 && e < 2047) {
        const double sc = __hiloint2double((2046 - e) << 20, 0); // 2^(1023 - e)
        a *= sc;
        b *= sc;
    }
}
// #{sigma_i < x} for the bidiagonal with squared off-diagonals bb[0 .. 2k-2] of TGK.
//   top: P_0 = 1, P_1 = -x, P_{i+1} = -x P_i - bb[i-1] P_{i-1}; pivot D+_i = P_{i+1} / P_i
//   bottom: Q_0 = 1, Q_1 = -x, Q_{i+1} = -x Q_i - bb[2k-1-i] Q_{i-1}; D-_{2k-1-i} = Q_{i+1} / Q_i
// A pivot is negative iff consecutive minors differ in sign bit (integer XOR of the high
// words: the count runs on the integer pipe, the FP64 pipe only carries the recurrence).
__device__ __forceinline__ int sbit(double v) { return static_cast<int>(static_cast<unsigned>(__double2hiint(v)) >> 31); }
__device__ __forceinline__ int tgk_count_below(const double* bb, int k, double x) {
    double p0 = 1.0, p1 = -x, q0 = 1.0, q1 = -x;
    int neg = 2 * sbit(-x); // D+_0 = P_1 / P_0 and D-_{2k-1} = Q_1 / Q_0
    const double* bt = bb;             // bb[i - 1] for step i
    const double* bq = bb + 2 * k - 2; // bb[2k - 1 - i] for step i
    int i = 1;
    // steps 1 .. k-2 count both chains; the bottom chain's step k-1 is D-_k (the twist)
    for (; i + 8 <= k - 1; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double p2 = fma(-x, p1, -bt[u] * p0);
            const double q2 = fma(-x, q1, -bq[-u] * q0);
            neg += (sbit(p2) ^ sbit(p1)) + (sbit(q2) ^ sbit(q1));
            p0 = p1;
            p1 = p2;
            q0 = q1;
            q1 = q2;
        }
        bt += 8;
        bq -= 8;
        rescale2(p0, p1);
        rescale2(q0, q1);
    }
    for (; i < k - 1; ++i) {
        const double p2 = fma(-x, p1, -bt[0] * p0);
        const double q2 = fma(-x, q1, -bq[0] * q0);
        neg += (sbit(p2) ^ sbit(p1)) + (sbit(q2) ^ sbit(q1));
        p0 = p1;
        p1 = p2;
        q0 = q1;
        q1 = q2;
        ++bt;
        --bq;
    }
    { // step k-1: top pivot D+_{k-1} counted, bottom minor Q_k feeds the twist
        const double p2 = fma(-x, p1, -bt[0] * p0);
        const double q2 = fma(-x, q1, -bq[0] * q0);
        neg += sbit(p2) ^ sbit(p1);
        p0 = p1;
        p1 = p2;
        q0 = q1;
        q1 = q2;
        ++bt;
    }
    // p1 = P_k, p0 = P_{k-1}, q1 = Q_k, q0 = Q_{k-1}; D+_k = P_{k+1} / P_k, D-_k = Q_k / Q_{k-1}
    const double pk1 = fma(-x, p1, -bt[0] * p0);
    const double dp = (p1 == 0.0) ? 1e300 : pk1 * rcp_nr(p1);
    const double dm = (q0 == 0.0) ? 1e300 : q1 * rcp_nr(q0);
    return neg + ((dp + dm + x) < 0.0) - k;
}
__global__ void __launch_bounds__(BD_T) k_bidiag_sv(int k, const double* a, double* sigma, int gprobe) {
    extern __shared__ double A[]; // k x bd_pitch(k)
    __shared__ double sq[KMAX], sq2[KMAX], d[KMAX], e[KMAX], bb[2 * KMAX], lo[KMAX], up[KMAX];
    __shared__ int cnt[BD_T];
    __shared__ double s_hi;
    constexpr int SUB = BD_SUB; // threads per column (left reflector) / row (right reflector)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = bd_pitch(k);
    const long long t_start = clock64();
    for (int x = tid; x < k * k; x += BD_T) {
        const int i = x / k, l = x - i * k;
        A[i * P + l] = a[x];
        if (l == 0)
            sq[i] = a[x] * a[x];
    }
    __syncthreads();
    for (int j = 0; j < k; ++j) {
        if (j + 1 + warp * (32 / SUB) < k) { // left reflector of column j (rows j .. k-1), formed
                                              // by every warp with a column c > j to update
            const double ts = range_sum(sq, j + 1, k, lane);
            const double x0 = A[j * P + j], ss = fma(x0, x0, ts);
            double alpha = 0.0, tau = 0.0, v0 = x0;
            if (ss > 0.0) {
                alpha = -copysign(sqrt(ss), x0);
                v0 = x0 - alpha;
                const double den = fma(v0, v0, ts);
                tau = den > 0.0 ? 2.0 / den : 0.0;
            }
            if (tid == 0)
                d[j] = alpha;
            const int c = j + 1 + tid / SUB, sub = tid % SUB;
            const bool on = c < k && tau != 0.0;
            // rows: sub 0 takes row j (v_j = v0) then j+SUB, ...; sub s takes j+s, j+s+SUB, ...
            const int i0 = j + sub + (sub == 0 ? SUB : 0);
            double s0 = 0.0, s1 = 0.0, ajc = 0.0;
            if (on) {
                ajc = A[j * P + c];
                if (sub == 0)
                    s0 = v0 * ajc;
                int i = i0;
                for (; i + SUB < k; i += 2 * SUB) {
                    s0 = fma(A[i * P + j], A[i * P + c], s0);
                    s1 = fma(A[(i + SUB) * P + j], A[(i + SUB) * P + c], s1);
                }
                if (i < k)
                    s0 = fma(A[i * P + j], A[i * P + c], s0);
            }
            s0 += s1;
#pragma unroll
            for (int o = 1; o < SUB; o <<= 1)
                s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            if (on) {
                const double w = tau * s0;
                if (sub == 0)
                    A[j * P + c] = fma(-w, v0, ajc);
                int i = i0;
                for (; i + SUB < k; i += 2 * SUB) { // loads ahead of stores: two independent updates
                    const double a0 = A[i * P + c], a1 = A[(i + SUB) * P + c];
                    const double v0i = A[i * P + j], v1 = A[(i + SUB) * P + j];
                    A[i * P + c] = fma(-w, v0i, a0);
                    A[(i + SUB) * P + c] = fma(-w, v1, a1);
                }
                if (i < k)
                    A[i * P + c] = fma(-w, A[i * P + j], A[i * P + c]);
            }
            if (c < k && sub == 0) {
                const double y = A[j * P + c]; // row j's new entry (this thread's i = j update)
                sq2[c] = y * y;
            }
        } else if (j == k - 1 && tid == 0) { // last column: a 1 x 1 reflector
            const double x0 = A[j * P + j];
            d[j] = x0 != 0.0 ? -x0 : 0.0;
        }
        __syncthreads();
        if (j == k - 1)
            break;
        if (j + 1 + warp * (32 / SUB) < k) { // right reflector of row j (columns j+1 .. k-1),
                                              // formed by every warp with a row r > j to update
            const double ts = range_sum(sq2, j + 2, k, lane);
            const double y0 = A[j * P + j + 1], ss = fma(y0, y0, ts);
            double beta = 0.0, tau = 0.0, u0 = y0;
            if (ss > 0.0) {
                beta = -copysign(sqrt(ss), y0);
                u0 = y0 - beta;
                const double den = fma(u0, u0, ts);
                tau = den > 0.0 ? 2.0 / den : 0.0;
            }
            if (tid == 0)
                e[j] = beta;
            const double* urow = A + j * P;
            const int r = j + 1 + tid / SUB, sub = tid % SUB;
            const bool on = r < k && tau != 0.0;
            double* row = A + (r < k ? r : 0) * P;
            // columns: sub 0 takes column j+1 (u = u0) then j+1+SUB, ...; sub s takes j+1+s, ...
            const int c0 = j + 1 + sub + (sub == 0 ? SUB : 0);
            double s0 = 0.0, s1 = 0.0, arj = 0.0;
            if (on) {
                arj = row[j + 1];
                if (sub == 0)
                    s0 = arj * u0;
                int c = c0;
                for (; c + SUB < k; c += 2 * SUB) {
                    s0 = fma(row[c], urow[c], s0);
                    s1 = fma(row[c + SUB], urow[c + SUB], s1);
                }
                if (c < k)
                    s0 = fma(row[c], urow[c], s0);
            }
            s0 += s1;
#pragma unroll
            for (int o = 1; o < SUB; o <<= 1)
                s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            if (on) {
                const double w = tau * s0;
                if (sub == 0)
                    row[j + 1] = fma(-w, u0, arj);
                int c = c0;
                for (; c + SUB < k; c += 2 * SUB) {
                    const double a0 = row[c], a1 = row[c + SUB];
                    const double u0c = urow[c], u1 = urow[c + SUB];
                    row[c] = fma(-w, u0c, a0);
                    row[c + SUB] = fma(-w, u1, a1);
                }
                if (c < k)
                    row[c] = fma(-w, urow[c], row[c]);
            }
            if (r < k && sub == 0) {
                const double y = row[j + 1]; // column j+1's new entry (this thread's c = j+1 update)
                sq[r] = y * y;
            }
        }
        __syncthreads();
    }
    // ---- multisection on TGK(d, e), scaled by a power of two so that sigma_max ~ 1
    const long long t_bidiag = clock64();
    if (warp == 0) {
        double md = 0.0, me = 0.0;
        for (int i = lane; i < k; i += 32) {
            md = fmax(md, fabs(d[i]));
            if (i < k - 1)
                me = fmax(me, fabs(e[i]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
            me = fmax(me, __shfl_xor_sync(0xffffffffu, me, o));
        }
        double hb = md + me, sc = 1.0;
        if (hb > 0.0) {
            const int eh = (__double2hiint(hb) >> 20) & 0x7ff; // hb in [2^(eh-1023), 2^(eh-1022))
            sc = __hiloint2double((2045 - eh) << 20, 0);       // 2^(1022 - eh): hb sc in [0.5, 1)
            if (eh == 0 || eh >= 2046)
                sc = 1.0;
        }
        for (int i = lane; i < k; i += 32) {
            const double di = d[i] * sc;
            bb[2 * i] = di * di;
            if (i < k - 1) {
                const double ei = e[i] * sc;
                bb[2 * i + 1] = ei * ei;
            }
        }
        if (lane == 0) {
            s_hi = hb * sc * (1.0 + 4.4e-16);
            sq[0] = sc; // kept for the unscaling
        }
    }
    __syncthreads();
    const double hi = s_hi, unscale = 1.0 / sq[0], tol = 2.3e-16 * hi;
    if (tid < k) {
        lo[tid] = 0.0;
        up[tid] = hi;
    }
    __syncthreads();
    // probes per interval: 3 (2 bits a round) keeps the count evaluations off the issue limit
    const int G = max(1, min(gprobe, BD_T / k));
    for (int round = 0; round < 200; ++round) {
        const int m = tid / G, g = tid - m * G;
        int c = -1;
        if (m < k) {
            const double l0 = lo[m], w = up[m] - l0;
            if (w > tol)
                c = tgk_count_below(bb, k, l0 + (g + 1) * (w / (G + 1)));
        }
        cnt[tid] = c;
        __syncthreads();
        bool open = false;
        if (tid < k) { // ascending sigma_m lies in [lo, up): #{sigma < x} <= m  <=>  x <= sigma_m
            const double l0 = lo[tid], w = up[tid] - l0;
            if (w > tol) {
                double nl = l0, nu = up[tid];
                for (int g2 = 0; g2 < G; ++g2) {
                    const double x = l0 + (g2 + 1) * (w / (G + 1));
                    if (cnt[tid * G + g2] <= tid)
                        nl = fmax(nl, x);
                    else
                        nu = fmin(nu, x);
                }
                lo[tid] = nl;
                up[tid] = nu;
                open = nu - nl > tol;
            }
        }
        if (!__syncthreads_or(open))
            break;
    }
    if (tid < k)
        sigma[k - 1 - tid] = hi > 0.0 ? 0.5 * (lo[tid] + up[tid]) * unscale : 0.0;
    if (tid == 0) // phase cycles (bidiagonalization, multisection) packed for RL_JACOBI_TRACE
        sigma[KMAX] = static_cast<double>(t_bidiag - t_start) * 1e6 + static_cast<double>(clock64() - t_bidiag);
}

__global__ void k_sumsq_partial(uint64_t count, const double* x, double* partial) {
    double s = 0.0;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        s = fma(x[e], x[e], s);
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1)
        s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (unsigned i = 0; i < blockDim.x / 32; ++i)
            t += red[i];
        partial[blockIdx.x] = t;
    }
}

std::vector<double> to_host(const double* d, uint64_t count) {
    std::vector<double> h(count);
    RL_CUDA(cudaMemcpyAsync(h.data(), d, count * sizeof(double), cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
    return h;
}

} // namespace

// C = alpha op(A) op(B) + beta C with K split into `splits` slices: one split-K GEMM launch
// (slice partials) and one fixed-order reduction, so the result is run-to-run identical.
void gemm_splitk(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, double alpha, const double* a,
                 uint64_t lda, const double* b, uint64_t ldb, double beta, double* c, uint64_t ldc,
                 int splits) {
    if (splits <= 1 || k < static_cast<uint64_t>(splits) * 16) {
        gemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
        return;
    }
    // slices of a multiple of 32 (the TMA kernel's k-tile) so no slice's last tile reaches into the next
    const uint64_t chunk = ((k + splits - 1) / splits + 31) / 32 * 32;
    const int used = static_cast<int>(cdiv(k, chunk));
    double* parts = ws<double>(WS_RF6, static_cast<uint64_t>(used) * m * n);
    gemm_splitk_parts(ta, tb, m, n, k, a, lda, b, ldb, parts, used, chunk);
    if (m * n * 32 <= 4ULL * 1024 * 1024 && used >= 32)
        k_splitk_reduce_warp<<<cdiv(m * n * 32, 256), 256, 0, stream()>>>(m, n, used, parts, alpha, beta, c, ldc);
    else if (n % 2 == 0 && ldc % 2 == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0 && m * n < (1ULL << 32) &&
             ldc < (1ULL << 32))
        k_splitk_reduce2<<<cdiv(m * n / 2, 256), 256, 0, stream()>>>(static_cast<uint32_t>(n),
                                                                     static_cast<uint32_t>(m * n), used, parts,
                                                                     alpha, beta, c, static_cast<uint32_t>(ldc));
    else
        k_splitk_reduce<<<cdiv(m * n, 256), 256, 0, stream()>>>(m, n, used, parts, alpha, beta, c, ldc);
    RL_LAUNCHED();
}

// K slices for an m x n output over K = k, from a small cost model: DMMA time at the
// fraction of two-CTA-per-SM waves the grid fills, ~2 us per wave of fixed CTA cost, and the
// partials' HBM round trip plus the reduction launch when split.
int splits_for(uint64_t m, uint64_t n, uint64_t k) {
    static const int force = getenv("RL_SPLITK_FORCE") ? atoi(getenv("RL_SPLITK_FORCE")) : 0; // dev sweeps
    if (force > 0 && static_cast<uint64_t>(force) * 16 <= k)
        return force;
    const double tiles = static_cast<double>(gemm_tiles(m, n));
    const double slots = 2.0 * ctx().sms;
    const double flops = 2.0 * static_cast<double>(m) * n * k;
    int best = 1;
    double best_t = 1e30;
    for (int s = 1; s <= 256 && k / s >= 16; ++s) {
        const double ctas = tiles * s, waves = std::ceil(ctas / slots);
        const double eff = (ctas / slots) / waves;
        double t = flops / (33e12 * eff) + waves * 2e-6;
        if (s > 1)
            t += 2.0 * s * static_cast<double>(m) * n * 8.0 / 5.5e12 + 2e-6;
        if (t < best_t * 0.98) {
            best = s;
            best_t = t;
        }
    }
    return best;
}

namespace {
using JacobiKernel = void (*)(int, const double*, double*);
template <int NE>
JacobiKernel jacobi_kernel() {
    static bool attr[16] = {};
    if (!attr[ctx().device & 15]) {
        RL_CUDA(cudaFuncSetAttribute(k_jacobi_sv<NE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     KMAX * KMAX * 8));
        attr[ctx().device & 15] = true;
    }
    return k_jacobi_sv<NE>;
}
JacobiKernel jacobi_for(int k) {
    switch ((k + 7) / 8) { // NE = ceil(k / 4) rounded up to even
    case 1: return jacobi_kernel<2>();
    case 2: return jacobi_kernel<4>();
    case 3: return jacobi_kernel<6>();
    case 4: return jacobi_kernel<8>();
    case 5: return jacobi_kernel<10>();
    case 6: return jacobi_kernel<12>();
    case 7: return jacobi_kernel<14>();
    case 8: return jacobi_kernel<16>();
    case 9: return jacobi_kernel<18>();
    case 10: return jacobi_kernel<20>();
    case 11: return jacobi_kernel<22>();
    case 12: return jacobi_kernel<24>();
    case 13: return jacobi_kernel<26>();
    case 14: return jacobi_kernel<28>();
    case 15: return jacobi_kernel<30>();
    default: return jacobi_kernel<32>();
    }
}
void chol_attrs() {
    static bool attr[16] = {};
    if (!attr[ctx().device & 15]) {
        RL_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     KMAX * (KMAX + 1) * 8));

        attr[ctx().device & 15] = true;
    }
}
} // namespace

// Singular values of a k x k device matrix into d_sg (k + 1 doubles: sigma non-increasing,
// then the kernel's diagnostic word), launched on the current stream (no synchronisation).
void small_sv_launch(int k, const double* d_a, double* d_sg) {
    if (k > KMAX)
        fail(RL_TOO_LARGE, "small SVD: k > 128");
    // k >= 16: bidiagonalization + multisection (the reference's BDCSVD range, dense_core.cpp:28);
    // RL_SV_JACOBI=1 selects one-sided Jacobi on the factor's rows (k eps bar) instead
    static const bool bidiag = getenv("RL_SV_JACOBI") == nullptr;
    if (bidiag && k >= 16) {
        static bool attr[16] = {};
        if (!attr[ctx().device & 15]) {
            RL_CUDA(cudaFuncSetAttribute(k_bidiag_sv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         KMAX * bd_pitch(KMAX) * 8));
            attr[ctx().device & 15] = true;
        }
        static const int gprobe = getenv("RL_BD_PROBES") ? atoi(getenv("RL_BD_PROBES")) : 3; // dev sweeps
        k_bidiag_sv<<<1, BD_T, static_cast<size_t>(k) * bd_pitch(k) * 8, stream()>>>(k, d_a, d_sg, gprobe);
    } else {
        JacobiKernel kern = jacobi_for(k);
        kern<<<1, JS_T, static_cast<size_t>(k) * k * 8, stream()>>>(k, d_a, d_sg);
    }
    RL_LAUNCHED();
}

// Singular values of a k x k device matrix -> host vector.
std::vector<double> small_singular_values(int k, const double* d_a) {
    double* sg = ws<double>(WS_RF5, KMAX + 1);
    small_sv_launch(k, d_a, sg);
    std::vector<double> h = to_host(sg, KMAX + 1);
    static const bool trace = getenv("RL_JACOBI_TRACE") != nullptr;
    if (trace)
        fprintf(stderr, "[rl] small svd k=%d: %.0f\n", k, h[KMAX]);
    if (h[KMAX] < 0)
        fail(RL_NO_CONVERGENCE, "small SVD: Jacobi sweeps did not settle");
    h.resize(k);
    return h;
}

namespace {
// qr_positive's rank test min |R_ii| > 1e-13 sigma_1(R) (dense_core.cpp:86-115) bracketed by
// ||R||_F / sqrt(k) <= sigma_1 <= ||R||_F: *flag = 0 passes for sure, 1 fails for sure, 2 needs
// sigma_1 itself (rare). One warp.
__global__ void k_rank_bracket(int k, const double* __restrict__ r, int* flag) {
    __shared__ double s_ss[8], s_mn[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double ss = 0.0, mn = INFINITY;
    for (int e = tid; e < k * k; e += 256) {
        const double v = r[e];
        ss = fma(v, v, ss);
    }
    for (int i = tid; i < k; i += 256)
        mn = fmin(mn, fabs(r[i * k + i]));
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
        s_ss[warp] = ss;
        s_mn[warp] = mn;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, b = INFINITY;
        for (int w = 0; w < 8; ++w) {
            a += s_ss[w];
            b = fmin(b, s_mn[w]);
        }
        const double fro = sqrt(a);
        *flag = (b > 1e-13 * fro) ? 0 : (b <= 1e-13 * fro / sqrt(static_cast<double>(k)) ? 1 : 2);
    }
}
} // namespace

namespace {
// The same bracket from diag(R) and ||Y||_F^2 = ||R||_F^2 (sum of nparts partials).
__global__ void k_rank_bracket_diag(int k, const double* __restrict__ rdiag, const double* __restrict__ part,
                                    int nparts, int* flag) {
    const int lane = threadIdx.x;
    double ss = 0.0, mn = INFINITY;
    for (int e = lane; e < nparts; e += 32)
        ss += part[e];
    for (int i = lane; i < k; i += 32)
        mn = fmin(mn, fabs(rdiag[i]));
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
        const double fro = sqrt(ss);
        *flag = (mn > 1e-13 * fro) ? 0 : (mn <= 1e-13 * fro / sqrt(static_cast<double>(k)) ? 1 : 2);
    }
}
} // namespace

void rank_bracket_diag_launch(int k, const double* d_rdiag, int* d_flag) {
    k_rank_bracket_diag<<<1, 32, 0, stream()>>>(k, d_rdiag, ws<double>(WS_RESID, 256), 256, d_flag);
    RL_LAUNCHED();
}

void rank_bracket_launch(int k, const double* d_r, int* d_flag) {
    k_rank_bracket<<<1, 256, 0, stream()>>>(k, d_r, d_flag);
    RL_LAUNCHED();
}

// Shifted CholeskyQR3 of Y (m x k, row-major, ld k): q (m x k) and r (k x k) with
// diag(r) > 0. Per pass: the Gram (split-K GEMM), k_chol_inv (R and R^-1), Q = src R^-1 on DMMA
// and R_acc = R_pass R_acc. No host round trip: the shift is summed on the device and the failure
// flag d_bad (int, device) is sticky — the caller reads it whenever it next synchronises.
// diag_only: r receives only diag(R) (k values) — the R_acc products are skipped (callers that
// need just the rank test: ||R||_F = ||Y||_F and diag(R) = the product of the passes' diagonals).
void cholqr3_async(uint64_t m, int k, const double* y, double* q, double* r, int* d_bad, bool want_q,
                   bool diag_only) {
    if (k > KMAX)
        fail(RL_TOO_LARGE, "qr_positive: more than 128 columns");
    double* g = ws<double>(WS_RF4, 3 * KMAX * KMAX + 64);
    double* racc0 = g + KMAX * KMAX; // R_acc ping-pong (the last pass writes r)
    double* racc1 = racc0 + KMAX * KMAX;
    double* tmpq = ws<double>(WS_RF5, m * k + KMAX * KMAX + KMAX + 1);
    const int sp = splits_for(k, k, m);
    chol_attrs();
    const int kp = (k + 7) & ~7;
    const size_t chol_smem = static_cast<size_t>(kp) * (kp + 1) * 8;
    // ||Y||_F^2 for the shift (Fukaya et al.: s = 11 (m k + k(k+1)) u ||Y||_2^2, F-norm bound)
    constexpr int kParts = 256;
    double* part = ws<double>(WS_RESID, kParts);
    k_sumsq_partial<<<kParts, 256, 0, stream()>>>(m * k, y, part);
    RL_LAUNCHED();
    const double u = 1.1102230246251565e-16;
    const double coef = 11.0 * (static_cast<double>(m) * k + static_cast<double>(k) * (k + 1)) * u;
    const double* src = y;
    double* rinv = tmpq + m * k; // k x k after the pass-1 Q buffer
    const double* racc_in = nullptr;
    for (int pass = 0; pass < 3; ++pass) {
        // G = src^T src
        gemm_splitk(true, false, k, k, m, 1.0, src, k, src, k, 0.0, g, k, sp);
        // R_pass, R_pass^-1 and R_acc = R_pass R_acc in one kernel
        double* racc_out = pass == 2 ? r : (pass == 0 ? racc0 : racc1);
        k_chol_inv<<<1, CH_T, chol_smem, stream()>>>(k, g, pass == 0 ? part : nullptr, kParts, coef, rinv, racc_in,
                                                     racc_out, d_bad, diag_only ? 1 : 0);
        RL_LAUNCHED();
        racc_in = racc_out;
        // Q_pass = src R_pass^-1 on DMMA (the last pass only when the caller wants Q)
        if (pass == 2 && !want_q)
            break;
        double* dst = (pass == 1) ? tmpq : q;
        gemm(false, false, m, k, k, 1.0, src, k, rinv, k, 0.0, dst, k);
        src = dst;
    }
}

bool cholqr3(uint64_t m, int k, const double* y, double* q, double* r) {
    int* d_bad = ws<int>(WS_FLAGS, 4);
    RL_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), stream()));
    cholqr3_async(m, k, y, q, r, d_bad, true, false);
    int bad = 0;
    RL_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
    return bad == 0;
}

// ||X||_F^2 (deterministic two-level reduction)
double sumsq_dev(uint64_t count, const double* x) {
    double* part = ws<double>(WS_RESID, 512);
    k_sumsq_partial<<<512, 256, 0, stream()>>>(count, x, part);
    RL_LAUNCHED();
    std::vector<double> h = to_host(part, 512);
    double s = 0.0;
    for (double v : h)
        s += v;
    return s;
}

} // namespace rl

// ------------------------------------------------------------- proto_lowrank ----
namespace rl {
void transpose_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda, double* t, uint64_t ldt);
}
// lowrank::proto_lowrank (lowrank.cpp:108-177), small n (the reference's own tests use 64):
// Gaussian RightSpace sketches (approx_basis, lowrank.cpp:67-106), the thin SVD of the sketch
// with left singular vectors (span_basis = its leading s left vectors), the auto-tau rule
// (:132-147), projection A T T^T (project_onto_basis, :45-65) and ||A - A T T^T||_2 / ||A||_2.
namespace rl {
namespace {

constexpr int PJ_T = 512, PJ_MAXC = 64, PJ_MAXR = 256;

// One-sided Jacobi on the R x C matrix W (row-major, ld C, R >= C, C <= 64, R C <= 16384):
// columns orthogonalised by round-robin rotations (C/2 disjoint pairs per step, one warp per
// pair, warp-shuffle reductions in a fixed order), sweeps until every pair is orthogonal to
// 1e-15 relative; sigma_j = ||w_j|| sorted descending (stable), u = normalised columns.
__global__ void __launch_bounds__(PJ_T) k_jacobi_left(int R, int C, const double* __restrict__ w_in,
                                                      double* __restrict__ sigma, double* __restrict__ u) {
    extern __shared__ double W[]; // column-major: W[j * R + i]
    __shared__ int perm[PJ_MAXC], order[PJ_MAXC];
    __shared__ double nrm[PJ_MAXC];
    __shared__ int rotated;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int e = t; e < R * C; e += PJ_T)
        W[(e % C) * R + e / C] = w_in[e];
    const int Ce = C + (C & 1); // even count: a dummy column when C is odd
    if (t < Ce)
        perm[t] = t;
    __syncthreads();
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (t == 0)
            rotated = 0;
        __syncthreads();
        for (int step = 0; step < Ce - 1; ++step) {
            for (int pr = warp; pr < Ce / 2; pr += PJ_T / 32) {
                int p = perm[pr], q = perm[Ce - 1 - pr];
                if (p > q) {
                    const int x = p;
                    p = q;
                    q = x;
                }
                if (q >= C)
                    continue; // the dummy
                double* wp = W + p * R;
                double* wq = W + q * R;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < R; i += 32) {
                    al = fma(wp[i], wp[i], al);
                    be = fma(wq[i], wq[i], be);
                    ga = fma(wp[i], wq[i], ga);
                }
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (ga == 0.0 || !(fabs(ga) > 1e-15 * sqrt(al * be)))
                    continue;
                const double zeta = (be - al) / (2.0 * ga);
                const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
                for (int i = lane; i < R; i += 32) {
                    const double x = wp[i], y = wq[i];
                    wp[i] = c * x - s * y;
                    wq[i] = s * x + c * y;
                }
                if (lane == 0)
                    rotated = 1;
            }
            __syncthreads();
            if (t == 0) { // round-robin: position 0 fixed, the others rotate
                const int last = perm[Ce - 1];
                for (int k = Ce - 1; k > 1; --k)
                    perm[k] = perm[k - 1];
                perm[1] = last;
            }
            __syncthreads();
        }
        if (!rotated)
            break;
        __syncthreads();
    }
    for (int j = warp; j < C; j += PJ_T / 32) {
        double s2 = 0.0;
        for (int i = lane; i < R; i += 32)
            s2 = fma(W[j * R + i], W[j * R + i], s2);
        for (int o = 16; o > 0; o >>= 1)
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0)
            nrm[j] = sqrt(s2);
    }
    __syncthreads();
    if (t == 0) { // stable insertion sort, descending
        for (int j = 0; j < C; ++j)
            order[j] = j;
        for (int i = 1; i < C; ++i)
            for (int k = i; k > 0 && nrm[order[k]] > nrm[order[k - 1]]; --k) {
                const int x = order[k];
                order[k] = order[k - 1];
                order[k - 1] = x;
            }
    }
    __syncthreads();
    for (int e = t; e < R * C; e += PJ_T) {
        const int i = e / C, j = e % C, src = order[j];
        const double sg = nrm[src];
        if (u)
            u[e] = sg > 0.0 ? W[src * R + i] / sg : 0.0;
        if (i == 0)
            sigma[j] = sg;
    }
}

// m x k Toeplitz from g = col[0..m-1], row[1..k-1] (random_structured's draw order,
// random_gen.cpp:94-103; densify, structured.cpp:70-83)
__global__ void k_toeplitz_rect(uint64_t m, uint64_t k, const double* g, double* out) {
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < m * k;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = e / k, j = e % k;
        out[e] = i >= j ? g[i - j] : g[m - 1 + (j - i)];
    }
}

__global__ void k_sub(uint64_t count, const double* a, const double* b, double* c) {
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        c[e] = a[e] - b[e];
}

// sigma (and u) of the m x n device matrix a (row-major): the taller orientation goes in
std::vector<double> jacobi_svd_dev(uint64_t m, uint64_t n, const double* a, double* d_sigma, double* d_u,
                                   double* scratch) {
    const double* src = a;
    uint64_t R = m, C = n;
    if (m < n) {
        transpose_dev(m, n, a, n, scratch, m);
        src = scratch;
        R = n;
        C = m;
    }
    static bool attr[16] = {};
    if (!attr[ctx().device & 15]) {
        RL_CUDA(cudaFuncSetAttribute(k_jacobi_left, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     PJ_MAXR * PJ_MAXC * 8));
        attr[ctx().device & 15] = true;
    }
    k_jacobi_left<<<1, PJ_T, R * C * sizeof(double), stream()>>>(static_cast<int>(R), static_cast<int>(C), src,
                                                                  d_sigma, d_u);
    RL_LAUNCHED();
    std::vector<double> h(C);
    RL_CUDA(cudaMemcpyAsync(h.data(), d_sigma, C * sizeof(double), cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
    return h;
}

} // namespace

bool proto_lowrank_supported(uint64_t m, uint64_t n, uint64_t rho_plus) {
    const uint64_t k = m < n ? m : n, l = m < n ? n : m;
    return k <= PJ_MAXC && l <= PJ_MAXR && rho_plus <= PJ_MAXC && n <= PJ_MAXR;
}

// d_a: m x n on the device.  basis: n x rho_plus (first rho columns valid), approx: m x n.
double norm2_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda);

// proto_lowrank beyond the one-CTA SVD (min(m, n) > 64 or max(m, n) > 256; rho_plus <= 64 <= n):
// ||A||_2 and ||A - approx||_2 by Lanczos (norm2_dev), the n x rho_plus sketch's thin SVD as
// shifted CholeskyQR3 (sketch = Q R) then the one-CTA Jacobi SVD of R with left vectors (the
// sketch's left vectors are Q U_R), everything else as the small path.
void proto_lowrank_large_dev(uint64_t m, uint64_t n, const double* d_a, uint64_t rho_plus, double tau,
                             double tau_prime, int tag, double mu, double sig_g, uint64_t seed, uint64_t sid,
                             uint64_t* rho_out, double* d_basis, double* d_approx, double* residual, int* ok) {
    const uint64_t k = rho_plus;
    double* sc = ws<double>(WS_RF5B, m * k + 3 * n * k + m * n + 3 * k * k + 2 * (m + k) + 64);
    double* g = sc;                 // m x k
    double* sk = g + m * k;         // n x k
    double* qs = sk + n * k;        // n x k
    double* ab = qs + n * k;        // max(m, n) x k
    double* diff = ab + n * k;      // m x n
    double* rs = diff + m * n;      // k x k
    double* ur = rs + k * k;        // k x k
    double* scr = ur + k * k;       // k x k
    double* sg = scr + k * k;       // sigma
    double* gv = sg + k + 8;        // Toeplitz generators (m + k - 1)
    if (m > n) // ab holds A T (m x s) below: grow it
        ab = ws<double>(WS_RF3B, m * k);
    const double norm_a = norm2_dev(m, n, d_a, n);
    *rho_out = 0;
    *residual = 0.0;
    *ok = 0;
    RL_CUDA(cudaMemsetAsync(d_approx, 0, m * n * sizeof(double), stream()));
    RL_CUDA(cudaMemsetAsync(d_basis, 0, n * k * sizeof(double), stream()));
    if (norm_a == 0.0) {
        *ok = 1;
        RL_CUDA(cudaStreamSynchronize(stream()));
        return;
    }
    for (int attempt = 0; attempt <= 3; ++attempt) {
        const uint64_t ds = sid + 104729ULL * static_cast<uint64_t>(attempt);
        if (tag == RL_TOEPLITZ_GAUSSIAN) {
            rng_generate(seed, ds, Draw::Gaussian, m + k - 1, mu, sig_g, gv);
            k_toeplitz_rect<<<cdiv(m * k, 256), 256, 0, stream()>>>(m, k, gv, g);
            RL_LAUNCHED();
        } else {
            rng_generate(seed, ds, Draw::Gaussian, m * k, mu, sig_g, g);
        }
        gemm(true, false, n, k, m, 1.0, d_a, n, g, k, 0.0, sk, k); // A^T G
        if (!cholqr3(n, static_cast<int>(k), sk, qs, rs))
            fail(RL_NO_CONVERGENCE, "proto_lowrank: the sketch's QR broke down (numerically rank-deficient beyond "
                                    "the shifted CholeskyQR3 range)");
        const std::vector<double> ss = jacobi_svd_dev(k, k, rs, sg, ur, scr);
        gemm(false, false, n, k, k, 1.0, qs, k, ur, k, 0.0, d_basis, k); // left vectors of the sketch
        double tau_eff = tau;
        if (tau_eff <= 0.0) { // the auto rule (lowrank.cpp:132-147)
            tau_eff = 1e-6;
            double best_gap = 1.0;
            for (size_t j = 1; j < ss.size(); ++j) {
                if (ss[j] >= 1e-3 * ss[0])
                    continue;
                const double gap = ss[j] / std::max(ss[j - 1], 1e-300);
                if (gap < best_gap) {
                    best_gap = gap;
                    tau_eff = std::sqrt(std::max(ss[j] * ss[j - 1], 1e-300)) / norm_a;
                }
            }
        }
        uint64_t s = ss.size();
        while (s > 0 && ss[s - 1] <= tau_eff * norm_a)
            --s;
        if (s == 0) {
            *rho_out = 0;
            RL_CUDA(cudaMemsetAsync(d_approx, 0, m * n * sizeof(double), stream()));
            *residual = 1.0;
            *ok = 0;
            continue;
        }
        gemm(false, false, m, s, n, 1.0, d_a, n, d_basis, k, 0.0, ab, k);
        gemm(false, true, m, n, s, 1.0, ab, k, d_basis, k, 0.0, d_approx, n);
        k_sub<<<cdiv(m * n, 256), 256, 0, stream()>>>(m * n, d_a, d_approx, diff);
        RL_LAUNCHED();
        *rho_out = s;
        *residual = norm2_dev(m, n, diff, n) / norm_a;
        *ok = *residual <= tau_prime;
        if (*ok)
            break;
    }
    if (*rho_out < k)
        for (uint64_t i = 0; i < n; ++i)
            RL_CUDA(cudaMemsetAsync(d_basis + i * k + *rho_out, 0, (k - *rho_out) * sizeof(double), stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
}

void proto_lowrank_dev(uint64_t m, uint64_t n, const double* d_a, uint64_t rho_plus, double tau, double tau_prime,
                       int tag, double mu, double sig_g, uint64_t seed, uint64_t sid, uint64_t* rho_out,
                       double* d_basis, double* d_approx, double* residual, int* ok) {
    if (!proto_lowrank_supported(m, n, rho_plus)) {
        proto_lowrank_large_dev(m, n, d_a, rho_plus, tau, tau_prime, tag, mu, sig_g, seed, sid, rho_out, d_basis,
                                d_approx, residual, ok);
        return;
    }
    double* sc = ws<double>(WS_RF5, 4 * m * n + 2 * n * rho_plus + 2 * m * rho_plus + 2 * (m + n + rho_plus) + 64);
    double* g = sc;                      // m x rho_plus
    double* sk = g + m * rho_plus;       // n x rho_plus
    double* ab = sk + n * rho_plus;      // m x rho_plus
    double* diff = ab + m * rho_plus;    // m x n
    double* scratch = diff + m * n;      // m x n (transposes)
    double* usv = scratch + m * n;       // m x n (left vectors of A / diff, unused)
    double* sg = usv + m * n;            // sigma scratch
    double* gv = sg + (m + n + rho_plus); // Toeplitz generators (m + rho_plus - 1)
    const std::vector<double> sa = jacobi_svd_dev(m, n, d_a, sg, nullptr, scratch);
    const double norm_a = sa[0];
    *rho_out = 0;
    *residual = 0.0;
    *ok = 0;
    RL_CUDA(cudaMemsetAsync(d_approx, 0, m * n * sizeof(double), stream()));
    RL_CUDA(cudaMemsetAsync(d_basis, 0, n * rho_plus * sizeof(double), stream()));
    if (norm_a == 0.0) {
        *ok = 1;
        RL_CUDA(cudaStreamSynchronize(stream()));
        return;
    }
    for (int attempt = 0; attempt <= 3; ++attempt) {
        const uint64_t ds = sid + 104729ULL * static_cast<uint64_t>(attempt);
        if (tag == RL_TOEPLITZ_GAUSSIAN) { // the m x rho_plus Toeplitz sketching matrix (approx_basis, lowrank.cpp:93-101)
            rng_generate(seed, ds, Draw::Gaussian, m + rho_plus - 1, mu, sig_g, gv);
            k_toeplitz_rect<<<cdiv(m * rho_plus, 256), 256, 0, stream()>>>(m, rho_plus, gv, g);
            RL_LAUNCHED();
        } else {
            rng_generate(seed, ds, Draw::Gaussian, m * rho_plus, mu, sig_g, g);
        }
        gemm(true, false, n, rho_plus, m, 1.0, d_a, n, g, rho_plus, 0.0, sk, rho_plus); // A^T G
        const std::vector<double> ss = jacobi_svd_dev(n, rho_plus, sk, sg, d_basis, scratch);
        double tau_eff = tau;
        if (tau_eff <= 0.0) { // the auto rule (lowrank.cpp:132-147)
            tau_eff = 1e-6;
            double best_gap = 1.0;
            for (size_t j = 1; j < ss.size(); ++j) {
                if (ss[j] >= 1e-3 * ss[0])
                    continue;
                const double gap = ss[j] / std::max(ss[j - 1], 1e-300);
                if (gap < best_gap) {
                    best_gap = gap;
                    tau_eff = std::sqrt(std::max(ss[j] * ss[j - 1], 1e-300)) / norm_a;
                }
            }
        }
        uint64_t s = ss.size();
        while (s > 0 && ss[s - 1] <= tau_eff * norm_a)
            --s;
        if (s == 0) {
            *rho_out = 0;
            RL_CUDA(cudaMemsetAsync(d_approx, 0, m * n * sizeof(double), stream()));
            *residual = 1.0;
            *ok = 0;
            continue;
        }
        // (A T) T^T with T the first s columns of the n x rho_plus basis
        gemm(false, false, m, s, n, 1.0, d_a, n, d_basis, rho_plus, 0.0, ab, rho_plus);
        gemm(false, true, m, n, s, 1.0, ab, rho_plus, d_basis, rho_plus, 0.0, d_approx, n);
        k_sub<<<cdiv(m * n, 256), 256, 0, stream()>>>(m * n, d_a, d_approx, diff);
        RL_LAUNCHED();
        const std::vector<double> sd = jacobi_svd_dev(m, n, diff, sg, nullptr, scratch);
        *rho_out = s;
        *residual = sd[0] / norm_a;
        *ok = *residual <= tau_prime;
        if (*ok)
            break;
    }
    // columns beyond rho are not part of the basis
    if (*rho_out < rho_plus)
        for (uint64_t i = 0; i < n; ++i)
            RL_CUDA(cudaMemsetAsync(d_basis + i * rho_plus + *rho_out, 0, (rho_plus - *rho_out) * sizeof(double),
                                    stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
}

} // namespace rl

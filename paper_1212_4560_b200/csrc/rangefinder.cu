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
#include <vector>

#include "rl_internal.cuh"

namespace rl {

void copy2d_dev(uint64_t rows, uint64_t cols, const double* src, uint64_t lds, double* dst, uint64_t ldd);

namespace {

constexpr int KMAX = 128; // largest rho+ handled by the single-CTA small kernels

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

// In-place Cholesky G = R^T R (k x k, ld k) -> R upper (zeros below) and Rinv (upper).
// shift is added to the diagonal first.  *ok = 0 on a non-positive pivot.
__global__ void __launch_bounds__(1024) k_chol_inv(int k, double* g, double shift, double* rinv, int* ok) {
    extern __shared__ double w[]; // KMAX x (KMAX+1)
    __shared__ double colv[KMAX];
    __shared__ int good;
    constexpr int P = KMAX + 1;
    const int tid = threadIdx.x;
    for (int e = tid; e < k * k; e += blockDim.x) {
        int i = e / k, j = e % k;
        w[i * P + j] = g[e] + (i == j ? shift : 0.0);
    }
    if (tid == 0)
        good = 1;
    __syncthreads();
    // right-looking Cholesky on the upper triangle: R[j][j] = sqrt(w_jj); R[j][l] = w_jl / R_jj;
    // w_il -= R_ji R_jl (i, l > j)
    for (int j = 0; j < k; ++j) {
        double d = w[j * P + j];
        if (!(d > 0.0)) {
            if (tid == 0)
                good = 0;
            break;
        }
        double r = sqrt(d);
        __syncthreads();
        for (int l = j + tid; l < k; l += blockDim.x)
            w[j * P + l] = (l == j) ? r : w[j * P + l] / r;
        __syncthreads();
        const int rem = k - j - 1;
        for (int e = tid; e < rem * rem; e += blockDim.x) {
            int i = j + 1 + e / rem, l = j + 1 + e % rem;
            if (l >= i)
                w[i * P + l] -= w[j * P + i] * w[j * P + l];
        }
        __syncthreads();
    }
    __syncthreads();
    if (!good) {
        if (tid == 0)
            *ok = 0;
        return;
    }
    // write R, then invert in place (Gauss-Jordan on the upper triangle, as genp.cu)
    for (int e = tid; e < k * k; e += blockDim.x) {
        int i = e / k, j = e % k;
        g[e] = (j >= i) ? w[i * P + j] : 0.0;
    }
    for (int kk = k - 1; kk >= 0; --kk) {
        __syncthreads();
        const double d = w[kk * P + kk];
        const double r = 1.0 / d;
        for (int i = tid; i < kk; i += blockDim.x)
            colv[i] = w[i * P + kk];
        __syncthreads();
        for (int j = kk + tid; j < k; j += blockDim.x)
            w[kk * P + j] = (j == kk) ? r : w[kk * P + j] * r;
        __syncthreads();
        const int cols = k - kk;
        for (int e = tid; e < kk * cols; e += blockDim.x) {
            int i = e / cols, j = kk + e % cols;
            double u = colv[i];
            w[i * P + j] = (j == kk) ? -u * w[kk * P + kk] : w[i * P + j] - u * w[kk * P + j];
        }
    }
    __syncthreads();
    for (int e = tid; e < k * k; e += blockDim.x) {
        int i = e / k, j = e % k;
        rinv[e] = (j >= i) ? w[i * P + j] : 0.0;
    }
    if (tid == 0)
        *ok = 1;
}

// Singular values of a k x k matrix (ld k) by one-sided Jacobi with round-robin
// pairing; one warp per column pair.  sigma sorted non-increasing.
__global__ void __launch_bounds__(1024) k_jacobi_sv(int k, const double* a, double* sigma) {
    extern __shared__ double w[]; // KMAX x KMAX column-major: column j at w + j*k
    __shared__ int perm[KMAX + 1];
    __shared__ double off_max;
    __shared__ double nrm[KMAX];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int kk = (k + 1) & ~1; // even number of slots (a dummy column when k is odd)
    for (int e = tid; e < k * k; e += blockDim.x) {
        int i = e / k, j = e % k;
        w[j * k + i] = a[e];
    }
    for (int i = tid; i < kk; i += blockDim.x)
        perm[i] = i;
    __syncthreads();
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (tid == 0)
            off_max = 0.0;
        __syncthreads();
        for (int round = 0; round < kk - 1; ++round) {
            for (int pr = warp; pr < kk / 2; pr += nw) {
                int p = perm[pr], q = perm[kk - 1 - pr];
                if (p >= k || q >= k)
                    continue;
                if (p > q) {
                    int t = p;
                    p = q;
                    q = t;
                }
                double* wp = w + p * k;
                double* wq = w + q * k;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < k; i += 32) {
                    al = fma(wp[i], wp[i], al);
                    be = fma(wq[i], wq[i], be);
                    ga = fma(wp[i], wq[i], ga);
                }
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (ga == 0.0)
                    continue;
                double rel = fabs(ga) / sqrt(al * be);
                if (!(rel > 1e-15))
                    continue;
                if (lane == 0) {
                    // monotone max via atomicMax on the bit pattern (non-negative doubles)
                    atomicMax(reinterpret_cast<unsigned long long*>(&off_max),
                              static_cast<unsigned long long>(__double_as_longlong(rel)));
                }
                double zeta = (be - al) / (2.0 * ga);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int i = lane; i < k; i += 32) {
                    double x = wp[i], y = wq[i];
                    wp[i] = c * x - s * y;
                    wq[i] = s * x + c * y;
                }
            }
            __syncthreads();
            // rotate the round-robin schedule (slot 0 fixed)
            if (tid == 0) {
                int last = perm[kk - 1];
                for (int i = kk - 1; i > 1; --i)
                    perm[i] = perm[i - 1];
                perm[1] = last;
            }
            __syncthreads();
        }
        if (off_max <= 1e-15)
            break;
        __syncthreads();
    }
    for (int j = warp; j < k; j += nw) {
        double s = 0.0;
        for (int i = lane; i < k; i += 32)
            s = fma(w[j * k + i], w[j * k + i], s);
        for (int o = 16; o > 0; o >>= 1)
            s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0)
            nrm[j] = sqrt(s);
    }
    __syncthreads();
    if (tid == 0) { // selection sort, descending
        for (int i = 0; i < k; ++i) {
            int best = i;
            for (int j = i + 1; j < k; ++j)
                if (nrm[j] > nrm[best])
                    best = j;
            double t = nrm[i];
            nrm[i] = nrm[best];
            nrm[best] = t;
            sigma[i] = nrm[i];
        }
    }
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

// C = alpha op(A) op(B) + beta C with K split into `splits` slices (fixed-order sum).
void gemm_splitk(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, double alpha, const double* a,
                 uint64_t lda, const double* b, uint64_t ldb, double beta, double* c, uint64_t ldc,
                 int splits) {
    if (splits <= 1 || k < static_cast<uint64_t>(splits) * 64) {
        gemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
        return;
    }
    uint64_t chunk = ((k + splits - 1) / splits + 15) / 16 * 16;
    double* parts = ws<double>(WS_RF6, static_cast<uint64_t>(splits) * m * n);
    int used = 0;
    for (int s = 0; s < splits; ++s) {
        uint64_t k0 = s * chunk;
        if (k0 >= k)
            break;
        uint64_t kl = std::min<uint64_t>(chunk, k - k0);
        const double* as = ta ? a + k0 * lda : a + k0;
        const double* bs = tb ? b + k0 : b + k0 * ldb;
        gemm(ta, tb, m, n, kl, 1.0, as, lda, bs, ldb, 0.0, parts + used * m * n, n);
        ++used;
    }
    k_splitk_reduce<<<cdiv(m * n, 256), 256, 0, stream()>>>(m, n, used, parts, alpha, beta, c, ldc);
    RL_LAUNCHED();
}

int splits_for(uint64_t m, uint64_t n, uint64_t k) {
    uint64_t tiles = static_cast<uint64_t>(cdiv(m, 64)) * cdiv(n, 64);
    int s = 1;
    while (tiles * s < 2ULL * ctx().sms && k / (s * 2) >= 512 && s < 32)
        s *= 2;
    return s;
}

// Singular values of a k x k device matrix -> host vector.
std::vector<double> small_singular_values(int k, const double* d_a) {
    if (k > KMAX)
        fail(RL_TOO_LARGE, "small SVD: k > 128");
    double* sg = ws<double>(WS_RF5, KMAX);
    static bool attr[16] = {};
    if (!attr[ctx().device & 15]) {
        RL_CUDA(cudaFuncSetAttribute(k_jacobi_sv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     KMAX * KMAX * 8));
        RL_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     KMAX * (KMAX + 1) * 8));
        attr[ctx().device & 15] = true;
    }
    k_jacobi_sv<<<1, 1024, KMAX * KMAX * 8, stream()>>>(k, d_a, sg);
    RL_LAUNCHED();
    return to_host(sg, k);
}

// Shifted CholeskyQR3 of Y (m x k, row-major, ld k): q (m x k) and r (k x k) with
// diag(r) > 0.  Returns false if a Cholesky step broke down.
bool cholqr3(uint64_t m, int k, const double* y, double* q, double* r) {
    if (k > KMAX)
        fail(RL_TOO_LARGE, "qr_positive: more than 128 columns");
    {
        static bool attr[16] = {};
        if (!attr[ctx().device & 15]) {
            RL_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         KMAX * (KMAX + 1) * 8));
            attr[ctx().device & 15] = true;
        }
    }
    double* g = ws<double>(WS_RF4, 3 * KMAX * KMAX + 64);
    double* rinv = g + KMAX * KMAX;
    double* racc = rinv + KMAX * KMAX;
    int* d_ok = reinterpret_cast<int*>(racc + KMAX * KMAX);
    double* tmpq = ws<double>(WS_RF5, m * k + KMAX);
    const int sp = splits_for(k, k, m);
    // ||Y||_F^2 for the shift (Fukaya et al.: s = 11 (m k + k(k+1)) u ||Y||_2^2, F-norm bound)
    double* part = ws<double>(WS_RESID, 256);
    k_sumsq_partial<<<256, 256, 0, stream()>>>(m * k, y, part);
    RL_LAUNCHED();
    std::vector<double> hp = to_host(part, 256);
    double fro2 = 0.0;
    for (double v : hp)
        fro2 += v;
    const double u = 1.1102230246251565e-16;
    const double shift = 11.0 * (static_cast<double>(m) * k + static_cast<double>(k) * (k + 1)) * u * fro2;
    const double* src = y;
    for (int pass = 0; pass < 3; ++pass) {
        // G = src^T src
        gemm_splitk(true, false, k, k, m, 1.0, src, k, src, k, 0.0, g, k, sp);
        RL_CUDA(cudaMemsetAsync(d_ok, 0, sizeof(int), stream()));
        k_chol_inv<<<1, 1024, KMAX * (KMAX + 1) * 8, stream()>>>(k, g, pass == 0 ? shift : 0.0, rinv, d_ok);
        RL_LAUNCHED();
        int ok = 0;
        RL_CUDA(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, stream()));
        RL_CUDA(cudaStreamSynchronize(stream()));
        if (!ok)
            return false;
        // Q_pass = src R^-1
        double* dst = (pass == 1) ? tmpq : q;
        gemm(false, false, m, k, k, 1.0, src, k, rinv, k, 0.0, dst, k);
        // R_acc = R_pass R_acc
        if (pass == 0) {
            copy2d_dev(k, k, g, k, racc, k);
        } else {
            gemm(false, false, k, k, k, 1.0, g, k, racc, k, 0.0, rinv, k);
            copy2d_dev(k, k, rinv, k, racc, k);
        }
        src = dst;
    }
    copy2d_dev(k, k, racc, k, r, k);
    return true;
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

// The rank-search side of lowrank (lowrank.cpp:179-396) on the GPU: extremal_sv_estimate (power
// method on A^T A and its shifted complement, or Lanczos with full reorthogonalization),
// cond_probe, nrank_search (probes A^T G_rho, G drawn once and truncated), power_transform and
// sampled_residual_check.
//
// extremal_sv_estimate is an iteration of matrix-vector products whose every step depends on the
// previous one: one persistent 1024-thread CTA runs the whole iteration (A stays in L2; t = A v
// by warps over rows, w = A^T t by threads over columns, dot products as fixed-order block
// reductions), with the reference's control flow step for step — the same start vectors (the
// stream's Gaussians in Rng::gaussian order), the same convergence tests and NoConvergence rule,
// the Ritz values' extremes of the Lanczos tridiagonal by Sturm bisection (the reference calls
// Eigen's tridiagonal eigensolver, unpinned upstream).
#include <cmath>
#include <vector>

#include "rl_internal.cuh"

namespace rl {

void copy2d_dev(uint64_t rows, uint64_t cols, const double* src, uint64_t lds, double* dst, uint64_t ldd);

namespace {

constexpr int ES_T = 1024;

struct EsOut {
    double sv_max, sv_min;
    int status; // 0 ok, 1 NoConvergence
    int steps;
};

// fixed-order CTA sum, result in every thread
__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0)
        red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll 8
    for (int i = 0; i < ES_T / 32; ++i)
        s += red[i];
    return s;
}

// w = A^T (A v): t (m, scratch) by warps over rows, then w by threads over columns
__device__ void gram_apply(uint64_t m, uint64_t n, const double* __restrict__ a, uint64_t lda,
                           const double* v, double* t, double* w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t i = warp; i < m; i += ES_T / 32) {
        const double* row = a + i * lda;
        double s = 0.0;
        for (uint64_t j = lane; j < n; j += 32)
            s = fma(row[j], v[j], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0)
            t[i] = s;
    }
    __syncthreads();
    for (uint64_t j = threadIdx.x; j < n; j += ES_T) {
        double s = 0.0;
        for (uint64_t i = 0; i < m; ++i)
            s = fma(a[i * lda + j], t[i], s);
        w[j] = s;
    }
    __syncthreads();
}

// #eigenvalues of the symmetric tridiagonal (alpha[0..k), beta[0..k-1)) below x (Sturm count)
__device__ int sturm_below(int k, const double* alpha, const double* beta, double x) {
    int c = 0;
    double d = 1.0;
    for (int i = 0; i < k; ++i) {
        const double b2 = i > 0 ? beta[i - 1] * beta[i - 1] : 0.0;
        d = (alpha[i] - x) - (i > 0 ? b2 / d : 0.0);
        if (d == 0.0)
            d = -1e-300;
        c += d < 0.0;
    }
    return c;
}
// extreme eigenvalues of the tridiagonal by bisection on Gershgorin bounds (thread 0)
__device__ void tridiag_extremes(int k, const double* alpha, const double* beta, double* lo, double* hi) {
    double gl = INFINITY, gu = -INFINITY;
    for (int i = 0; i < k; ++i) {
        const double r = (i > 0 ? fabs(beta[i - 1]) : 0.0) + (i + 1 < k ? fabs(beta[i]) : 0.0);
        gl = fmin(gl, alpha[i] - r);
        gu = fmax(gu, alpha[i] + r);
    }
    const double pad = 1e-300 + 4e-16 * fmax(fabs(gl), fabs(gu));
    gl -= pad;
    gu += pad;
    for (int which = 0; which < 2; ++which) { // 0: smallest (count >= 1), 1: largest (count >= k)
        double a = gl, b = gu;
        const int want = which == 0 ? 1 : k;
        for (int it = 0; it < 200 && b - a > 2.2e-16 * fmax(fabs(a), fabs(b)) + 1e-300; ++it) {
            const double mid = 0.5 * (a + b);
            if (mid <= a || mid >= b)
                break;
            if (sturm_below(k, alpha, beta, mid) >= want)
                b = mid;
            else
                a = mid;
        }
        (which == 0 ? *lo : *hi) = 0.5 * (a + b);
    }
}

// lowrank.cpp:204-348. g0: 2n start draws (Rng::gaussian order). scratch: t (m), v, w (n), and
// for Lanczos the basis (kmax x n). alpha/beta: kmax each (global scratch).
__global__ void __launch_bounds__(ES_T, 1)
    k_extremal_sv(uint64_t m, uint64_t n, const double* __restrict__ a, uint64_t lda, int lanczos, int iters,
                  const double* __restrict__ g0, double* __restrict__ t, double* __restrict__ v, double* __restrict__ w,
                  double* __restrict__ basis, double* __restrict__ alpha, double* __restrict__ beta, EsOut* out,
                  double top_tol) {
    __shared__ double red[ES_T / 32];
    __shared__ double s_lohi[2];
    const int tid = threadIdx.x;
    auto dot = [&](const double* x, const double* y) {
        double s = 0.0;
        for (uint64_t i = tid; i < n; i += ES_T)
            s = fma(x[i], y[i], s);
        return block_sum(s, red);
    };
    // v <- normalised start vector from draws [off, off + n)
    auto start = [&](uint64_t off) {
        for (uint64_t i = tid; i < n; i += ES_T)
            v[i] = g0[off + i];
        __syncthreads();
        const double nv = sqrt(dot(v, v));
        for (uint64_t i = tid; i < n; i += ES_T)
            v[i] = v[i] / nv;
        __syncthreads();
    };
    if (!lanczos) {
        // ---- power iteration for the top eigenvalue of A^T A
        start(0);
        double lambda = 0.0, prev = 0.0, top = 0.0;
        bool conv1 = false, zero = false;
        for (int it = 0; it < iters; ++it) {
            gram_apply(m, n, a, lda, v, t, w);
            const double nw = sqrt(dot(w, w));
            if (nw == 0.0) {
                zero = true;
                conv1 = true;
                break;
            }
            lambda = dot(v, w);
            for (uint64_t i = tid; i < n; i += ES_T)
                v[i] = w[i] / nw;
            __syncthreads();
            if (it > 0 && fabs(lambda - prev) <= 1e-4 * fmax(fabs(lambda), 1e-300)) {
                conv1 = true;
                break;
            }
            prev = lambda;
        }
        top = zero ? 0.0 : lambda;
        top = fmax(top, 0.0);
        if (top == 0.0) {
            if (tid == 0)
                *out = EsOut{0.0, 0.0, 0, 0};
            return;
        }
        const double shift = 1.01 * top;
        start(n); // the next n draws of the same Rng
        const double smax = sqrt(top);
        double est = smax, prev_est = -1.0;
        bool conv2 = false;
        for (int it = 0; it < iters; ++it) {
            gram_apply(m, n, a, lda, v, t, w);
            for (uint64_t i = tid; i < n; i += ES_T)
                w[i] = shift * v[i] - w[i];
            __syncthreads();
            const double nw = sqrt(dot(w, w));
            if (nw == 0.0)
                break;
            const double mu = dot(v, w);
            for (uint64_t i = tid; i < n; i += ES_T)
                v[i] = w[i] / nw;
            __syncthreads();
            est = sqrt(fmax(shift - mu, 0.0));
            if (prev_est >= 0.0 && fabs(est - prev_est) <= 1e-4 * est + 1e-8 * smax) {
                conv2 = true;
                break;
            }
            prev_est = est;
        }
        if (tid == 0)
            *out = EsOut{smax, est, (conv1 && conv2) ? 0 : 1, 0};
        return;
    }
    // ---- Lanczos on A^T A with full reorthogonalization
    start(0);
    double scale = 0.0, prev_lo = -1.0, prev_hi = -1.0;
    bool settled = false, closed = false;
    const int kmax = static_cast<int>(min(static_cast<uint64_t>(iters), n));
    int k = 0;
    for (; k < kmax; ++k) {
        double* qk = basis + static_cast<uint64_t>(k) * n;
        for (uint64_t i = tid; i < n; i += ES_T)
            qk[i] = v[i];
        __syncthreads();
        gram_apply(m, n, a, lda, v, t, w);
        const double ak = dot(v, w);
        if (tid == 0)
            alpha[k] = ak;
        const double bprev = k > 0 ? beta[k - 1] : 0.0;
        const double* qprev = k > 0 ? basis + static_cast<uint64_t>(k - 1) * n : nullptr;
        for (uint64_t i = tid; i < n; i += ES_T) {
            double x = w[i] - ak * v[i];
            if (k > 0)
                x -= bprev * qprev[i];
            w[i] = x;
        }
        __syncthreads();
        for (int b = 0; b <= k; ++b) { // full reorthogonalization, one basis vector at a time
            const double* qq = basis + static_cast<uint64_t>(b) * n;
            const double c = dot(qq, w);
            for (uint64_t i = tid; i < n; i += ES_T)
                w[i] -= c * qq[i];
            __syncthreads();
        }
        scale = fmax(scale, fabs(ak));
        const double bk = sqrt(dot(w, w));
        if (tid == 0)
            tridiag_extremes(k + 1, alpha, beta, &s_lohi[0], &s_lohi[1]);
        __syncthreads();
        const double lo = s_lohi[0], hi = s_lohi[1];
        if (prev_hi >= 0.0) {
            const bool hi_ok = fabs(hi - prev_hi) <= 1e-4 * fmax(fabs(hi), 1e-300);
            const bool lo_ok = fabs(lo - prev_lo) <= 1e-4 * fmax(fabs(hi), 1e-300);
            settled = hi_ok && lo_ok;
            // norm2 mode (top_tol > 0): stop once the largest Ritz value has settled
            if (top_tol > 0.0 && fabs(hi - prev_hi) <= top_tol * fabs(hi)) {
                closed = true;
                ++k;
                break;
            }
        }
        prev_lo = lo;
        prev_hi = hi;
        if (bk <= 1e-14 * fmax(scale, 1e-300)) {
            closed = true; // invariant subspace: the Ritz values are exact
            ++k;
            break;
        }
        if (tid == 0)
            beta[k] = bk;
        for (uint64_t i = tid; i < n; i += ES_T)
            v[i] = w[i] / bk;
        __syncthreads();
    }
    const int steps = k;
    const bool exhausted = static_cast<uint64_t>(steps) >= n;
    if (tid == 0) {
        double lo, hi;
        tridiag_extremes(steps, alpha, beta, &lo, &hi);
        *out = EsOut{sqrt(fmax(hi, 0.0)), sqrt(fmax(lo, 0.0)), (!settled && !closed && !exhausted) ? 1 : 0, steps};
    }
}

} // namespace

// extremal_sv_estimate of the m x n device matrix a (ld lda). method 0 Power, 1 Lanczos.
// Throws NoConvergence as the reference does.
void extremal_sv_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda, int method, int iters, uint64_t seed,
                     uint64_t sid, double* sv_max, double* sv_min) {
    if (iters < 1)
        fail(RL_INVALID_ARGUMENT, "extremal_sv_estimate: iters must be >= 1");
    const uint64_t kmax = std::min<uint64_t>(static_cast<uint64_t>(iters), n);
    double* g0 = ws<double>(WS_ES0, 2 * n + 2);
    rng_generate(seed, sid, Draw::Gaussian, 2 * n, 0.0, 1.0, g0);
    double* sc = ws<double>(WS_ES1, m + 2 * n + 2 * (kmax + 1));
    double* basis = method == 1 ? ws<double>(WS_ES2, kmax * n) : nullptr;
    EsOut* d_out = reinterpret_cast<EsOut*>(ws<double>(WS_ES3, 4));
    double* t = sc;
    double* v = t + m;
    double* w = v + n;
    double* alpha = w + n;
    double* beta = alpha + kmax + 1;
    k_extremal_sv<<<1, ES_T, 0, stream()>>>(m, n, a, lda, method, iters, g0, t, v, w, basis, alpha, beta, d_out,
                                            0.0);
    RL_LAUNCHED();
    EsOut h{};
    RL_CUDA(cudaMemcpyAsync(&h, d_out, sizeof(EsOut), cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
    if (h.status)
        fail(RL_NO_CONVERGENCE, method == 1 ? "extremal_sv_estimate: lanczos did not settle"
                                            : "extremal_sv_estimate: power method did not settle");
    *sv_max = h.sv_max;
    *sv_min = h.sv_min;
}

// ||A||_2 = sigma_1 of the m x n device matrix (dense::norm2 beyond the one-CTA SVD's sizes): Lanczos
// on A^T A with full reorthogonalization from a fixed start vector, stopped when the largest Ritz
// value moves by <= 1e-15 relative (or the Krylov space closes / n steps), then sqrt.
double norm2_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda) {
    const uint64_t kmax = std::min<uint64_t>(n, 96);
    double* g0 = ws<double>(WS_ES0, 2 * n + 2);
    rng_generate(0x6e6f726d32ULL, n, Draw::Gaussian, 2 * n, 0.0, 1.0, g0);
    double* sc = ws<double>(WS_ES1, m + 2 * n + 2 * (kmax + 1));
    double* basis = ws<double>(WS_ES2, kmax * n);
    EsOut* d_out = reinterpret_cast<EsOut*>(ws<double>(WS_ES3, 4));
    double* t = sc;
    double* v = t + m;
    double* w = v + n;
    double* alpha = w + n;
    double* beta = alpha + kmax + 1;
    k_extremal_sv<<<1, ES_T, 0, stream()>>>(m, n, a, lda, 1, static_cast<int>(kmax), g0, t, v, w, basis, alpha, beta,
                                            d_out, 1e-15);
    RL_LAUNCHED();
    EsOut h{};
    RL_CUDA(cudaMemcpyAsync(&h, d_out, sizeof(EsOut), cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
    return h.sv_max;
}

// cond_probe (lowrank.cpp:350-358)
bool cond_probe_dev(uint64_t m, uint64_t n, const double* b, uint64_t ldb, double kappa, int method, int iters,
                    uint64_t seed, uint64_t sid) {
    if (!(kappa > 1.0))
        fail(RL_INVALID_ARGUMENT, "cond_probe: kappa_threshold must exceed 1");
    double hi = 0.0, lo = 0.0;
    extremal_sv_dev(m, n, b, ldb, method, iters, seed, sid, &hi, &lo);
    if (!(lo > 1e-14 * hi) || hi == 0.0)
        return false;
    return hi / lo <= kappa;
}

// nrank_search (lowrank.cpp:360-396) on the m x n device matrix a. Returns rho; basis (device,
// capacity max(m, n) x rho_plus) receives the wide-side work^T G_rho (n_w x rho, ld rho) and
// *basis_rows its row count.
uint64_t nrank_search_dev(uint64_t m, uint64_t n, const double* a, uint64_t rho_minus, uint64_t rho_plus,
                          double kappa, int policy, uint64_t seed, uint64_t sid, double* basis,
                          uint64_t* basis_rows) {
    const bool transpose = m < n; // work on the wide side so rows >= cols
    const uint64_t wm = transpose ? n : m, wn = transpose ? m : n;
    if (!(rho_minus < rho_plus) || rho_plus > wn)
        fail(RL_INVALID_ARGUMENT, "nrank_search: need 0 <= rho_minus < rho_plus <= min(m, n)");
    // G (wm x rho_plus), drawn once; P = work^T G (wn x rho_plus): its leading columns are every
    // probe work^T G_cand (column j of the product depends on column j of G only)
    double* g = ws<double>(WS_ES4, wm * rho_plus);
    rng_generate(seed, sid, Draw::Gaussian, wm * rho_plus, 0.0, 1.0, g);
    double* p = ws<double>(WS_ES5, wn * rho_plus);
    if (!transpose) // work = a (m x n): P = a^T G
        gemm(true, false, wn, rho_plus, wm, 1.0, a, n, g, rho_plus, 0.0, p, rho_plus);
    else // work = a^T: P = a G, a is m x n = wn x wm
        gemm(false, false, wn, rho_plus, wm, 1.0, a, n, g, rho_plus, 0.0, p, rho_plus);
    const int probe_iters = 4 * static_cast<int>(rho_plus) + 20;
    uint64_t lo = rho_minus, hi = rho_plus, probe_idx = 1;
    while (lo < hi) {
        uint64_t cand;
        if (policy == 0) {
            cand = (lo + hi + 1) / 2;
        } else {
            const uint64_t step = std::max<uint64_t>(1, (hi - lo + 3) / 4);
            cand = std::max(lo + 1, hi - step);
        }
        const bool pass = cond_probe_dev(wn, cand, p, rho_plus, kappa, 1, probe_iters, seed,
                                         sid ^ (0x7000000000000000ULL + probe_idx));
        ++probe_idx;
        if (pass)
            lo = cand;
        else
            hi = cand - 1;
    }
    *basis_rows = wn;
    if (lo > 0)
        copy2d_dev(wn, lo, p, rho_plus, basis, lo);
    return lo;
}

} // namespace rl

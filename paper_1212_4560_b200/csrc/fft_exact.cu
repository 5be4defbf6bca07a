// The drop-in structured:: products (structured.cpp:20-189) on the GPU, bit for bit.
//
// structured::fft (structured.cpp:96-130) is an iterative radix-2 DIT transform: bit-reversal
// permutation, then for len = 2, 4, .., n a butterfly pass whose twiddles come from a chain
// w_0 = 1, w_{k+1} = w_k * wlen with wlen = (cos, sin)(+-2 pi / len) — GCC turns the cos/sin pair
// into one libm sincos call. Every step is reproduced exactly:
//   * complex products are GCC's inline complex multiply for finite operands, (ac - bd) +
//     (ad + bc) i with every product rounded (the reference is built without FMA), with the
//     C99 Annex G infinity recovery of libgcc's __muldc3 when both parts come out NaN;
//   * sincos is glibc's own FMA build (glibc_math.cuh), the same one the host calls;
//   * butterflies are u + v, u - v; the inverse divides both parts by n.
// The twiddle chains are inherently sequential (k-th twiddle = k chained products): one thread
// per pass computes its chain once per (n, direction), cached per device; the butterfly passes
// then run in parallel — O(n log n) work. fft_convolve / take_real / circ_mul / toeplitz_mul /
// multiply_matrix (structured.cpp:20-50,132-189) follow on top, batched over matrix columns:
// the spec is transformed once, every column's transform, pointwise product, inverse transform,
// fold (non-power-of-two circulants) and imaginary-residue check run for all columns at once.
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "glibc_math.cuh"
#include "rl_internal.cuh"

namespace rl {

namespace {

unsigned grid_for(uint64_t total, unsigned threads) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(cdiv(total, threads), 8ULL * ctx().sms)));
}

__device__ __forceinline__ double2 cmul_gcc(double2 p, double2 q) {
    double a = p.x, b = p.y, c = q.x, d = q.y;
    const double ac = __dmul_rn(a, c), bd = __dmul_rn(b, d), ad = __dmul_rn(a, d), bc = __dmul_rn(b, c);
    double x = __dsub_rn(ac, bd), y = __dadd_rn(ad, bc);
    if (isnan(x) && isnan(y)) { // libgcc __muldc3 (C99 Annex G.5.1)
        bool recalc = false;
        if (isinf(a) || isinf(b)) {
            a = copysign(isinf(a) ? 1.0 : 0.0, a);
            b = copysign(isinf(b) ? 1.0 : 0.0, b);
            if (isnan(c)) c = copysign(0.0, c);
            if (isnan(d)) d = copysign(0.0, d);
            recalc = true;
        }
        if (isinf(c) || isinf(d)) {
            c = copysign(isinf(c) ? 1.0 : 0.0, c);
            d = copysign(isinf(d) ? 1.0 : 0.0, d);
            if (isnan(a)) a = copysign(0.0, a);
            if (isnan(b)) b = copysign(0.0, b);
            recalc = true;
        }
        if (!recalc && (isinf(ac) || isinf(bd) || isinf(ad) || isinf(bc))) {
            if (isnan(a)) a = copysign(0.0, a);
            if (isnan(b)) b = copysign(0.0, b);
            if (isnan(c)) c = copysign(0.0, c);
            if (isnan(d)) d = copysign(0.0, d);
            recalc = true;
        }
        if (recalc) {
            x = __dmul_rn(INFINITY, __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, d)));
            y = __dmul_rn(INFINITY, __dadd_rn(__dmul_rn(a, d), __dmul_rn(b, c)));
        }
    }
    return make_double2(x, y);
}

// Pass s (len = 2^(s+1), half = 2^s) stores its half twiddles at tw[half - 1 + k].
__global__ void k_fft_twiddles(int lgn, double sign, double2* __restrict__ tw) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= lgn)
        return;
    const uint64_t half = 1ULL << s;
    // ang = sign * 2.0 * pi / len, left to right: (+-2 * pi) / len, both exact
    const double ang = __ddiv_rn(__dmul_rn(__dmul_rn(sign, 2.0), 3.14159265358979323846),
                                 static_cast<double>(2 * half));
    double sn, cs;
    glm::sincos_fma(ang, &sn, &cs);
    const double2 wlen = make_double2(cs, sn);
    double2 w = make_double2(1.0, 0.0);
    double2* out = tw + (half - 1);
    for (uint64_t k = 0; k < half; ++k) {
        out[k] = w;
        w = cmul_gcc(w, wlen);
    }
}

__device__ __forceinline__ uint64_t bitrev(uint64_t i, int lgn) {
    return lgn == 0 ? 0 : (__brevll(i) >> (64 - lgn));
}

// One CTA per vector, n <= 2048: bit-reversed load, all passes in shared memory, store (with the
// inverse's 1/n); src, dst: batch vectors of n complex at stride n.
constexpr int FFT_SMEM_MAX = 2048, FFT_THREADS = 256;
__global__ void __launch_bounds__(FFT_THREADS) k_fft_smem(int lgn, const double2* __restrict__ tw,
                                                          const double2* __restrict__ src, double2* __restrict__ dst,
                                                          int inverse) {
    __shared__ double2 z[FFT_SMEM_MAX];
    const uint64_t n = 1ULL << lgn;
    const double2* in = src + blockIdx.x * n;
    for (uint64_t i = threadIdx.x; i < n; i += FFT_THREADS)
        z[bitrev(i, lgn)] = in[i];
    __syncthreads();
    for (int s = 0; s < lgn; ++s) {
        const uint64_t half = 1ULL << s;
        for (uint64_t b = threadIdx.x; b < n / 2; b += FFT_THREADS) {
            const uint64_t k = b & (half - 1), i = (b >> s) << (s + 1);
            const double2 u = z[i + k];
            const double2 v = cmul_gcc(z[i + k + half], tw[half - 1 + k]);
            z[i + k] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
            z[i + k + half] = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
        }
        __syncthreads();
    }
    double2* out = dst + blockIdx.x * n;
    const double dn = static_cast<double>(n);
    for (uint64_t i = threadIdx.x; i < n; i += FFT_THREADS) {
        const double2 v = z[i];
        out[i] = inverse ? make_double2(__ddiv_rn(v.x, dn), __ddiv_rn(v.y, dn)) : v;
    }
}

// Larger n: bit-reversed copy, then one launch per pass over all vectors' butterflies.
__global__ void k_fft_bitrev(int lgn, uint64_t total, const double2* __restrict__ src, double2* __restrict__ dst) {
    const uint64_t n = 1ULL << lgn;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t v = e >> lgn, i = e & (n - 1);
        dst[v * n + bitrev(i, lgn)] = src[e];
    }
}
__global__ void k_fft_pass(int lgn, int s, uint64_t total_bf, const double2* __restrict__ tw, double2* __restrict__ z) {
    const uint64_t n = 1ULL << lgn, half = 1ULL << s;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total_bf;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t v = e / (n / 2), b = e % (n / 2);
        const uint64_t k = b & (half - 1), i = v * n + ((b >> s) << (s + 1));
        const double2 u = z[i + k];
        const double2 w = cmul_gcc(z[i + k + half], tw[half - 1 + k]);
        z[i + k] = make_double2(__dadd_rn(u.x, w.x), __dadd_rn(u.y, w.y));
        z[i + k + half] = make_double2(__dsub_rn(u.x, w.x), __dsub_rn(u.y, w.y));
    }
}
__global__ void k_fft_scale(uint64_t total, double dn, double2* __restrict__ z) {
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        z[e] = make_double2(__ddiv_rn(z[e].x, dn), __ddiv_rn(z[e].y, dn));
}

// real vectors -> complex, zero-padded: dst[v][i] = (i < len ? src[i * ld + v * vstride] : 0, 0)
__global__ void k_real_to_complex(uint64_t batch, uint64_t n, uint64_t len, const double* __restrict__ src,
                                  uint64_t ld, uint64_t vstride, double2* __restrict__ dst) {
    const uint64_t total = batch * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t v = e / n, i = e % n;
        dst[e] = make_double2(i < len ? src[i * ld + v * vstride] : 0.0, 0.0);
    }
}

// z[v][i] *= conj(ch[i]): FFT of a cross-correlation with the real generator c
__global__ void k_corr_mul(uint64_t batch, uint64_t n, const double2* __restrict__ ch, double2* __restrict__ z) {
    const uint64_t total = batch * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double2 h = ch[e % n];
        z[e] = cmul_gcc(z[e], make_double2(h.x, -h.y));
    }
}

// out[v * ldo + j] = Re z[v][j], j < n_out
__global__ void k_complex_rows_real(uint64_t batch, uint64_t n, uint64_t n_out, const double2* __restrict__ z,
                                    double* __restrict__ out, uint64_t ldo) {
    const uint64_t total = batch * n_out;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t v = e / n_out, j = e % n_out;
        out[v * ldo + j] = z[v * n + j].x;
    }
}

// fa[i] *= fb[i] (structured.cpp:31-32), fa shared by every vector of fb
__global__ void k_pointwise(uint64_t batch, uint64_t n, const double2* __restrict__ fa, double2* __restrict__ fb) {
    const uint64_t total = batch * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        fb[e] = cmul_gcc(fa[e % n], fb[e]);
}

// vector_norm2 (matrix.hpp): sqrt of the sequential sum of squares; one thread per vector.
__global__ void k_norm2_seq(uint64_t batch, uint64_t len, const double* __restrict__ src, uint64_t ld,
                            uint64_t vstride, double* __restrict__ out) {
    const uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (v >= batch)
        return;
    double s = 0.0;
    for (uint64_t i = 0; i < len; ++i) {
        const double x = src[i * ld + v * vstride];
        s = __dadd_rn(s, __dmul_rn(x, x));
    }
    out[v] = __dsqrt_rn(s);
}

// Per vector v: optional fold (circ_mul's general-n path, structured.cpp:146-152), take_real
// (structured.cpp:39-50): max |imag| over the first m (std::max order), the residue test against
// 1e-10 * max(scale, 1e-300) with scale = |c| |x_v|, the real parts to out[i * ldo + v].
// One CTA per vector; flags[v] = 1 when the residue test fails.
__global__ void k_take_real(uint64_t m, uint64_t n_fold, uint64_t len, const double2* __restrict__ conv,
                            double cnorm, const double* __restrict__ xnorm, double* __restrict__ out, uint64_t ldo,
                            int* __restrict__ flags) {
    const uint64_t v = blockIdx.x;
    const double2* z = conv + v * len;
    __shared__ double part[256];
    double mx = 0.0;
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
        double2 w = z[i];
        if (n_fold && i + n_fold < 2 * n_fold - 1) {
            const double2 u = z[i + n_fold];
            w = make_double2(__dadd_rn(w.x, u.x), __dadd_rn(w.y, u.y));
        }
        const double a = fabs(w.y);
        mx = (mx < a) ? a : mx; // std::max(mx, |imag|): NaN never replaces
        out[i * ldo + v] = w.x;
    }
    part[threadIdx.x] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m2 = 0.0;
        for (unsigned t = 0; t < blockDim.x; ++t)
            m2 = (m2 < part[t]) ? part[t] : m2;
        const double scale = __dmul_rn(cnorm, xnorm[v]);
        if (m2 >= __dmul_rn(1e-10, (scale < 1e-300) ? 1e-300 : scale))
            flags[v] = 1;
    }
}

struct TwKey {
    int device, lgn, inverse;
    bool operator<(const TwKey& o) const {
        return device != o.device ? device < o.device : lgn != o.lgn ? lgn < o.lgn : inverse < o.inverse;
    }
};
std::mutex g_tw_mu;
std::map<TwKey, double2*> g_tw;

const double2* twiddles(int lgn, int inverse) {
    std::lock_guard<std::mutex> lk(g_tw_mu);
    const TwKey key{ctx().device, lgn, inverse};
    auto it = g_tw.find(key);
    if (it != g_tw.end())
        return it->second;
    double2* tw = nullptr;
    RL_CUDA(cudaMalloc(&tw, sizeof(double2) * std::max<uint64_t>(1ULL << lgn, 1)));
    if (lgn > 0) {
        k_fft_twiddles<<<cdiv(lgn, 32), 32, 0, stream()>>>(lgn, inverse ? 1.0 : -1.0, tw);
        RL_LAUNCHED();
    }
    RL_CUDA(cudaStreamSynchronize(stream())); // the cache is shared by every thread's stream
    g_tw[key] = tw;
    return tw;
}

int log2_exact(uint64_t n) {
    int l = 0;
    while ((1ULL << l) < n)
        ++l;
    return l;
}

} // namespace

// batch complex vectors of length n (power of two) in `src` -> `dst` (may alias)
void fft_exact_dev(uint64_t n, uint64_t batch, const double2* src, double2* dst, int inverse) {
    if (n == 0 || (n & (n - 1)))
        fail(RL_LENGTH_NOT_POW2, "fft: length must be a power of two");
    if (batch == 0)
        return;
    const int lgn = log2_exact(n);
    const double2* tw = twiddles(lgn, inverse);
    if (n <= static_cast<uint64_t>(FFT_SMEM_MAX)) {
        k_fft_smem<<<static_cast<unsigned>(batch), FFT_THREADS, 0, stream()>>>(lgn, tw, src, dst, inverse);
        RL_LAUNCHED();
        return;
    }
    double2* tmp = dst;
    if (src == dst) { // the bit-reversal permutation needs a second buffer
        tmp = ws<double2>(WS_FFT_TMP, n * batch);
        RL_CUDA(cudaMemcpyAsync(tmp, src, n * batch * sizeof(double2), cudaMemcpyDeviceToDevice, stream()));
        src = tmp;
        tmp = dst;
    }
    k_fft_bitrev<<<grid_for(n * batch, 256), 256, 0, stream()>>>(lgn, n * batch, src, dst);
    RL_LAUNCHED();
    for (int s = 0; s < lgn; ++s) {
        k_fft_pass<<<grid_for(n / 2 * batch, 256), 256, 0, stream()>>>(lgn, s, n / 2 * batch, tw, dst);
        RL_LAUNCHED();
    }
    if (inverse) {
        k_fft_scale<<<grid_for(n * batch, 256), 256, 0, stream()>>>(n * batch, static_cast<double>(n), dst);
        RL_LAUNCHED();
    }
}

// A C for circulants beyond the shared-memory FFT (n > 8192, a power of two): row r of the result
// is the cyclic cross-correlation of row r of A (its first n_in entries, zero-padded to n) with c,
// FFT(row) * conj(FFT(c)) through the global-memory passes of fft_exact_dev, in row batches of at
// most 2^26 complex entries (1 GiB); the first n_out columns are kept (Toeplitz embeddings).
// O(m n log n) and matrix-free: the dense fallback was a 2 n^3 product.
void circ_right_fft_large(uint64_t m, uint64_t n, uint64_t n_in, uint64_t n_out, const double* c, const double* a,
                          uint64_t lda, double* out, uint64_t ldo) {
    cudaStream_t st = stream();
    double2* ch = ws<double2>(WS_FFT_C, n);
    k_real_to_complex<<<grid_for(n, 256), 256, 0, st>>>(1, n, n, c, 1, 0, ch);
    RL_LAUNCHED();
    fft_exact_dev(n, 1, ch, ch, 0);
    const uint64_t batch = std::max<uint64_t>(1, std::min<uint64_t>(m, (1ULL << 26) / n));
    double2* z = ws<double2>(WS_FFT_X, batch * n);
    for (uint64_t r0 = 0; r0 < m; r0 += batch) {
        const uint64_t rows = std::min(batch, m - r0);
        k_real_to_complex<<<grid_for(rows * n, 256), 256, 0, st>>>(rows, n, n_in, a + r0 * lda, 1, lda, z);
        RL_LAUNCHED();
        fft_exact_dev(n, rows, z, z, 0);
        k_corr_mul<<<grid_for(rows * n, 256), 256, 0, st>>>(rows, n, ch, z);
        RL_LAUNCHED();
        fft_exact_dev(n, rows, z, z, 1);
        k_complex_rows_real<<<grid_for(rows * n_out, 256), 256, 0, st>>>(rows, n, n_out, z, out + r0 * ldo, ldo);
        RL_LAUNCHED();
    }
}

// multiply_matrix (structured.cpp:178-189) for `cols` columns of the row-major n_cols x cols
// matrix A (ld = cols): circulant (first_row == nullptr; m = n = n_cols) through circ_mul's pow2 or
// folded path, Toeplitz (m x n_cols) through toeplitz_mul's circulant embedding. out: m x cols.
// Throws Error when a column's imaginary residue fails take_real (structured.cpp:39-50).
void structured_multiply_dev(uint64_t m, uint64_t n, const double* first_col, const double* first_row,
                             uint64_t cols, const double* a, double* out) {
    const bool circ = first_row == nullptr;
    auto next_pow2 = [](uint64_t v) {
        uint64_t p = 1;
        while (p < v)
            p <<= 1;
        return p;
    };
    const bool pow2 = circ && (n & (n - 1)) == 0;
    const uint64_t len = circ ? (pow2 ? n : next_pow2(2 * n - 1)) : next_pow2(m + n - 1);
    // the circulant generator of the product (Toeplitz: its embedding of order len)
    double* gen = ws<double>(WS_FFT_GEN, len + 2 * cols + 1);
    double* xnorm = gen + len;
    double* cnorm_d = xnorm + cols;
    cudaStream_t st = stream();
    if (circ) {
        RL_CUDA(cudaMemcpyAsync(gen, first_col, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else {
        std::vector<double> hc(m), hr(n), emb(len, 0.0);
        RL_CUDA(cudaMemcpyAsync(hc.data(), first_col, m * sizeof(double), cudaMemcpyDeviceToHost, st));
        RL_CUDA(cudaMemcpyAsync(hr.data(), first_row, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        RL_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < m; ++i)
            emb[i] = hc[i];
        for (uint64_t j = 1; j < n; ++j)
            emb[len - j] = hr[j];
        RL_CUDA(cudaMemcpyAsync(gen, emb.data(), len * sizeof(double), cudaMemcpyHostToDevice, st));
        RL_CUDA(cudaStreamSynchronize(st));
    }
    const uint64_t glen = circ ? n : len; // generator entries that carry the spec
    double2* fc = ws<double2>(WS_FFT_C, len);
    double2* fx = ws<double2>(WS_FFT_X, len * cols);
    int* flags = ws<int>(WS_FFT_FLAG, cols);
    k_real_to_complex<<<grid_for(len, 256), 256, 0, st>>>(1, len, glen, gen, 1, 0, fc);
    RL_LAUNCHED();
    k_norm2_seq<<<1, 1, 0, st>>>(1, glen, gen, 1, 0, cnorm_d);
    RL_LAUNCHED();
    // columns of A: element i of column v at a[i * cols + v], zero-padded to len
    k_real_to_complex<<<grid_for(len * cols, 256), 256, 0, st>>>(cols, len, n, a, cols, 1, fx);
    RL_LAUNCHED();
    k_norm2_seq<<<cdiv(cols, 128), 128, 0, st>>>(cols, n, a, cols, 1, xnorm);
    RL_LAUNCHED();
    fft_exact_dev(len, 1, fc, fc, 0);
    fft_exact_dev(len, cols, fx, fx, 0);
    k_pointwise<<<grid_for(len * cols, 256), 256, 0, st>>>(cols, len, fc, fx);
    RL_LAUNCHED();
    fft_exact_dev(len, cols, fx, fx, 1);
    double cnorm = 0.0;
    RL_CUDA(cudaMemcpyAsync(&cnorm, cnorm_d, sizeof(double), cudaMemcpyDeviceToHost, st));
    RL_CUDA(cudaMemsetAsync(flags, 0, cols * sizeof(int), st));
    RL_CUDA(cudaStreamSynchronize(st));
    // circulant: the first n entries (folded when n is not a power of two); Toeplitz: take_real
    // checks all len entries of the embedded product (circ_mul of order len), keeps the first m
    const uint64_t check = circ ? n : len;
    k_take_real<<<static_cast<unsigned>(cols), 256, 0, st>>>(check, (circ && !pow2) ? n : 0, len, fx, cnorm, xnorm,
                                                             circ ? out : ws<double>(WS_FFT_OUT, len * cols), cols,
                                                             flags);
    RL_LAUNCHED();
    if (!circ) {
        const double* full = ws<double>(WS_FFT_OUT, len * cols);
        RL_CUDA(cudaMemcpyAsync(out, full, m * cols * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    std::vector<int> hf(cols);
    RL_CUDA(cudaMemcpyAsync(hf.data(), flags, cols * sizeof(int), cudaMemcpyDeviceToHost, st));
    RL_CUDA(cudaStreamSynchronize(st));
    for (int f : hf)
        if (f)
            fail(RL_ERROR, "structured product: imaginary residue exceeds tolerance");
}

} // namespace rl

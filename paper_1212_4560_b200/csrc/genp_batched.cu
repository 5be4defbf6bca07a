// K6: batched randomized GENP for small systems (config 2: 4096 x n=64, circulant +-1,
// MulSide::Right; Table 1's MulSide::Left + refine) — semantically the loop
// bench::table1_genp runs (bench.cpp:117-133) over genp::randomized_genp (genp.cpp:207-291),
// one stream per system.
//
// One 64-thread CTA (two warps) per system; every FP64 operation runs on the DFMA pipe (on
// sm_100a DMMA and DFMA share one FP64 pipe: tools/micro/pipes.cu measures 37.1 TF/s DMMA alone,
// 34.0 DFMA alone and ~35 mixed, so the design minimises FP64 operations, not DMMA count).
//   * The working matrix lives in registers, distributed 8 x 8 cyclically: thread (tr, tc) =
//     (t / 8, t % 8) owns w(tr + 8r, tc + 8c), r, c < 8 — every thread keeps an equal share of
//     the shrinking trailing matrix until the last block of eight pivots.
//   * No-pivot LU (genp.cpp:20-33): 64 pivot steps, one barrier each. At step k the owners of
//     row k and column k publish them (double-buffered, in the idle staging buffer) and the
//     pivot's owner publishes 1/p; every thread then forms its multipliers m = w(i,k) * (1/p)
//     (1/p := 0 for p = 0) and updates its own entries with one FMA each; rows / columns at
//     or left of the pivot are left untouched (predicated FMAs on the boundary block only).
//   * The multiplier product W = A C (Right) / C A (Left) runs through the FFT, as the
//     reference's own structured::multiply_matrix does (genp.cpp:158-166, structured.cpp:
//     178-189): thread t owns row t of A (Right) or column t (Left), packs it as 32 complex
//     points, runs a register-resident 32-point FFT, the real-FFT split, the pointwise product
//     with the multiplier's spectrum, the inverse split and the inverse 32-point FFT — about
//     1.3 K FP64 operations per row against 8 K FMAs for the dense product.
//   * The packed LU is written once to shared memory for warp 0's substitutions
//     (genp.cpp:106-124); y = C z, refinement and the residual ||A y - b|| / ||b|| run on all
//     64 threads.
// The raw-GENP contrast arm is iteration -1 of the same loop (pivot floor 0, no multiplier).
// The 8-attempt redraw protocol (stream id + 7919 a, accept <= 1e-7, keep best,
// genp.cpp:236-290) runs in-kernel.  Exactly singular circulants (a vanishing 64-point DFT
// coefficient) are pre-screened and skipped; a system that exhausts its
// attempts is re-run with the exact protocol (pass 1) so the returned best attempt is the
// reference's.
#include <cmath>

#include "reg_lu.cuh"
#include "rl_internal.cuh"

namespace rl {

#ifdef RL_B64_PROF // phase timer for one system (tools/micro/b64_prof.cu); compiled out of the library
__device__ long long g_b64_prof[32];
#define B64_MARK(ph)                                                                                \
    do {                                                                                            \
        if (threadIdx.x == 0 && blockIdx.x == 0) {                                                  \
            const long long now_ = clock64();                                                       \
            g_b64_prof[ph] += now_ - prof_t0;                                                       \
            prof_t0 = now_;                                                                         \
        }                                                                                           \
    } while (0)
#else
#define B64_MARK(ph) ((void)0)
#endif

namespace {

constexpr int N = 64;
constexpr int THREADS = 64;
constexpr int P = 66; // staging pitch (528 B rows: 16-byte aligned, conflict-free 128-bit row reads)
// LU publication buffer per parity: the pivot row owner-major at pitch 10 (the eight owners'
// 128-bit reads hit distinct banks), then the pivot column owner-major at pitch 8.
constexpr int PUB = reglu::Pub<8>::SIZE;

struct Smem {
    double X[N * P]; // A staging / W / packed LU (row-major); sign-stream scratch and DFT twiddles
    double rcp[N];   // 1/U_kk
    double pubb[2];  // the forward-substituted right-hand side's pivot entry, per parity
    union {
        double pub[2 * PUB]; // the LU's row / column publications (two parities x (row, column))
        struct {
            double v0[N], v1[N];
            double2 H[33]; // multiplier spectrum (conj for Right) / 128, bins 0..32
        };
    };
    double red[2];
    double pm[2];    // |pivot| min / max of the last LU
    double bsq, best_res;
    uint64_t mask, mask0;
    unsigned bal[2];
    int flag;
    rl_precond_report rp; // the system's report (thread 0), kept out of the register budget
};

// (cos, sin)(2 pi j / 64), j < 32 (exact symmetries between entries)
__constant__ double2 kCS64[32] = {
    {0x1.0000000000000p+0, 0.0},
    {0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4},
    {0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3},
    {0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2},
    {0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2},
    {0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2},
    {0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1},
    {0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1},
    {0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1},
    {0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1},
    {0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1},
    {0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1},
    {0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1},
    {0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1},
    {0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1},
    {0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1},
    {0.0, 0x1.0000000000000p+0},
    {-0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1},
    {-0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1},
    {-0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1},
    {-0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1},
    {-0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1},
    {-0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1},
    {-0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1},
    {-0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1},
    {-0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1},
    {-0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1},
    {-0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2},
    {-0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2},
    {-0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2},
    {-0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3},
    {-0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4},
};

__device__ __forceinline__ double sgn(uint64_t mask, int j) { // bit j set <=> c_j = -1
    return ((mask >> (j & 63)) & 1ULL) ? -1.0 : 1.0;
}

// 64 sign draws of stream (seed, sid) after discard(8) as a bitmask (random_gen.cpp:22-31,
// 55-57).  One thread; only the first phase of the first twist is needed (new[i], i < 72 <
// 156); the 228 seeding words are staged in `scratch` (shared) instead of a local array.
__device__ uint64_t sign_mask_stream(uint64_t seed, uint64_t sid, uint64_t* scratch) {
    auto splitmix = [](uint64_t& st) {
        uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    uint64_t st = seed;
    const uint64_t a = splitmix(st);
    st ^= sid * 0xda942042e4dd58b5ULL + 0x2545f4914f6cdd1dULL;
    const uint64_t b = splitmix(st);
    uint64_t v = a ^ (b << 1);
    scratch[0] = v;
    for (int i = 1; i < 156 + 72; ++i) {
        v = 6364136223846793005ULL * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
        scratch[i] = v;
    }
    uint64_t mask = 0;
    for (int i = 8; i < 72; ++i) {
        const uint64_t y = (scratch[i] & 0xFFFFFFFF80000000ULL) | (scratch[i + 1] & 0x7FFFFFFFULL);
        uint64_t z = scratch[i + 156] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        z ^= z >> 43;
        if (!(z & 1ULL))
            mask |= 1ULL << (i - 8);
    }
    return mask;
}

// ------------------------------------------------------------------ FFT ----
__host__ __device__ constexpr int br5(int m) {
    return ((m & 1) << 4) | ((m & 2) << 2) | (m & 4) | ((m & 8) >> 2) | ((m & 16) >> 4);
}

// (xr + i xi) *= (cos, -sin)(2 pi j / 64) (forward) or (cos, +sin) (inverse); j < 32 constant
template <bool INV>
__device__ __forceinline__ void twiddle(double& xr, double& xi, int j) {
    if (j == 0)
        return;
    if (j == 16) { // -i (forward) / +i (inverse)
        const double t = xr;
        if (!INV) {
            xr = xi;
            xi = -t;
        } else {
            xr = -xi;
            xi = t;
        }
        return;
    }
    const double c = kCS64[j].x, s = INV ? kCS64[j].y : -kCS64[j].y;
    const double r = fma(xr, c, -xi * s);
    const double i = fma(xr, s, xi * c);
    xr = r;
    xi = i;
}

// One radix-2 pass of the in-place 32-point FFT on z_k = x[2k] + i x[2k+1] (LEN = butterfly span).
template <int LEN, bool INV>
__device__ __forceinline__ void fft_pass(double (&x)[N]) {
    constexpr int half = LEN / 2;
#pragma unroll
    for (int g = 0; g < 32; g += LEN)
#pragma unroll
        for (int k = 0; k < half; ++k) {
            const int a = g + k, b = a + half, j = (64 / LEN) * k;
            if (!INV) {
                const double ur = x[2 * a], ui = x[2 * a + 1], vr = x[2 * b], vi = x[2 * b + 1];
                x[2 * a] = ur + vr;
                x[2 * a + 1] = ui + vi;
                double dr = ur - vr, di = ui - vi;
                twiddle<false>(dr, di, j);
                x[2 * b] = dr;
                x[2 * b + 1] = di;
            } else {
                double vr = x[2 * b], vi = x[2 * b + 1];
                twiddle<true>(vr, vi, j);
                const double ur = x[2 * a], ui = x[2 * a + 1];
                x[2 * a] = ur + vr;
                x[2 * a + 1] = ui + vi;
                x[2 * b] = ur - vr;
                x[2 * b + 1] = ui - vi;
            }
        }
}

// Forward: decimation in frequency, natural order in, bit-reversed out.  Inverse (unnormalised,
// +i): decimation in time, bit-reversed in, natural out.
template <bool INV>
__device__ __forceinline__ void fft32(double (&x)[N]) {
    if (!INV) {
        fft_pass<32, false>(x);
        fft_pass<16, false>(x);
        fft_pass<8, false>(x);
        fft_pass<4, false>(x);
        fft_pass<2, false>(x);
    } else {
        fft_pass<2, true>(x);
        fft_pass<4, true>(x);
        fft_pass<8, true>(x);
        fft_pass<16, true>(x);
        fft_pass<32, true>(x);
    }
}

__device__ __forceinline__ double2 cmul(double2 p, double2 q) {
    return make_double2(fma(p.x, q.x, -p.y * q.y), fma(p.x, q.y, p.y * q.x));
}

// x <- the 64-point circular product of the real vector x with the multiplier whose spectrum
// (already conjugated for Right, scaled by 1/128) is H[0..32]: IDFT64(DFT64(x) .* H).
// Packed: Z = FFT32(x_even + i x_odd); X_m = E + W^m O, X_{32-m} = conj(E - W^m O) with
// E = Z_m + conj Z_{32-m}, O = -i (Z_m - conj Z_{32-m}) (both 2x), W = e^{-2 pi i / 64};
// Y = X .* H; inverse Z'_m = E' + i O', E' = Y_m + conj Y_{32-m}, O' = (Y_m - conj Y_{32-m}) W^-m,
// Z'_{32-m} = conj E' + i conj O'; x_even + i x_odd = IFFT32(Z').
__device__ __forceinline__ void circ_fft64(double (&x)[N], const double2* __restrict__ H) {
    fft32<false>(x);
#pragma unroll
    for (int m = 0; m <= 16; ++m) {
        const int p = (32 - m) & 31, im = br5(m), ip = br5(p);
        const double2 zm = make_double2(x[2 * im], x[2 * im + 1]);
        const double2 zp = make_double2(x[2 * ip], x[2 * ip + 1]);
        const double2 E = make_double2(zm.x + zp.x, zm.y - zp.y);
        double2 T = make_double2(zm.y + zp.y, zp.x - zm.x); // O = -i (Z_m - conj Z_p)
        twiddle<false>(T.x, T.y, m);
        const double2 ym = cmul(make_double2(E.x + T.x, E.y + T.y), H[m]);
        const double2 yp = cmul(make_double2(E.x - T.x, T.y - E.y), H[32 - m]);
        const double2 e2 = make_double2(ym.x + yp.x, ym.y - yp.y);
        double2 o2 = make_double2(ym.x - yp.x, ym.y + yp.y);
        twiddle<true>(o2.x, o2.y, m);
        x[2 * im] = e2.x - o2.y;
        x[2 * im + 1] = e2.y + o2.x;
        if (m != 0 && m != 16) {
            x[2 * ip] = e2.x + o2.y;
            x[2 * ip + 1] = o2.x - e2.y;
        }
    }
    fft32<true>(x);
}

// ------------------------------------------------------------------- LU ----
// The factorization itself is reglu::factor<8, true> (reg_lu.cuh): 64 pivot steps, one
// barrier each, the right-hand side forward-substituted alongside.
__device__ __forceinline__ void lu_regs(double (&w)[8][8], double& bcur, Smem& S, int tr, int tc) {
    reglu::factor<8, true>(w, bcur, reglu::Bufs{S.pub, S.rcp, S.pubb}, tr, tc);
}

// The packed LU into X (row-major): U as factored, L_ij = w(i,j) * (1/U_jj) below the diagonal.
__device__ __forceinline__ void lu_store(const double (&w)[8][8], Smem& S, int tr, int tc) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double inv = S.rcp[tc + 8 * c];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            double v = w[r][c];
            if (r > c || (r == c && tr > tc))
                v *= inv;
            S.X[(tr + 8 * r) * P + tc + 8 * c] = v;
        }
    }
}

// Eight substitution steps of warp 0's solve over columns jb .. jb+7 (HI: jb >= 32, the rows
// l + 32 half), branch-free: the block's L / U entries of the lane's two rows (and the eight
// 1/U_jj) are loaded first, so each step's chain is one shuffle, (one multiply) and one FMA.
template <bool HI, bool BACK>
__device__ __forceinline__ void solve_block8(const Smem& S, int jb, int lane, double& x0, double& x1) {
    const double* r0 = S.X + lane * P + jb;
    const double* r1 = S.X + (lane + 32) * P + jb;
    double a0[8], a1[8], rc[8];
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
        const double2 v0 = *reinterpret_cast<const double2*>(r0 + q);
        const double2 v1 = *reinterpret_cast<const double2*>(r1 + q);
        a0[q] = v0.x;
        a0[q + 1] = v0.y;
        a1[q] = v1.x;
        a1[q + 1] = v1.y;
        if (BACK) {
            const double2 vr = *reinterpret_cast<const double2*>(S.rcp + jb + q);
            rc[q] = vr.x;
            rc[q + 1] = vr.y;
        }
    }
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
        const int q = BACK ? 7 - qq : qq, j = jb + q;
        double xj = __shfl_sync(0xffffffffu, HI ? x1 : x0, j & 31);
        if (BACK)
            xj *= rc[q];
        const double f0 = fma(-a0[q], xj, x0), f1 = fma(-a1[q], xj, x1);
        if (!BACK) { // unit L: rows below j
            if (!HI)
                x0 = lane > j ? f0 : x0;
            x1 = lane + 32 > j ? f1 : x1;
        } else { // U: row j takes x_j, rows above it are updated
            if (HI) {
                x1 = lane + 32 == j ? xj : (lane + 32 < j ? f1 : x1);
                x0 = f0;
            } else {
                x0 = lane == j ? xj : (lane < j ? f0 : x0);
            }
        }
    }
}

// warp 0: S.v0 <- U^{-1} L^{-1} S.v0 (FWD) or U^{-1} S.v0 with the packed LU row-major in X
// (L_ij = X[i * P + j] below the diagonal, U on and above; genp.cpp:106-124).  Lane l owns
// rows l and l + 32.  (The factorization's own right-hand side is forward-substituted inside
// the LU; refinement steps run both halves here.)
template <bool FWD>
__device__ __forceinline__ void solve_warp0(Smem& S, int lane) {
    double x0 = S.v0[lane], x1 = S.v0[lane + 32];
    if (FWD) {
#pragma unroll 1
        for (int jb = 0; jb < 32; jb += 8)
            solve_block8<false, false>(S, jb, lane, x0, x1);
#pragma unroll 1
        for (int jb = 32; jb < N; jb += 8)
            solve_block8<true, false>(S, jb, lane, x0, x1);
    }
#pragma unroll 1
    for (int jb = N - 8; jb >= 32; jb -= 8)
        solve_block8<true, true>(S, jb, lane, x0, x1);
#pragma unroll 1
    for (int jb = 24; jb >= 0; jb -= 8)
        solve_block8<false, true>(S, jb, lane, x0, x1);
    S.v0[lane] = x0;
    S.v0[lane + 32] = x1;
}

// (C z)_t, z in S.v0
__device__ __forceinline__ double circ_vec(const Smem& S, int t) {
    const uint64_t mask = S.mask;
    double y = 0.0;
#pragma unroll 16
    for (int j = 0; j < N; ++j)
        y = fma(sgn(mask, t - j), S.v0[j], y);
    return y;
}

// CTA-wide sum, result in every thread
__device__ __forceinline__ double cta_sum(Smem& S, double a, int t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((t & 31) == 0)
        S.red[t >> 5] = a;
    __syncthreads();
    const double s = S.red[0] + S.red[1];
    __syncthreads();
    return s;
}

// (A y)_t - b_t: A's row t (registers, loaded while the solve runs), y in S.v1; four partial
// sums keep the FMA chain short
__device__ __forceinline__ double row_residual(const double (&arow)[N], const Smem& S, double bt) {
    double p[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        const double2 y = *reinterpret_cast<const double2*>(S.v1 + j);
        p[(j >> 1) & 3] = fma(arow[j], y.x, p[(j >> 1) & 3]);
        p[(j >> 1) & 3] = fma(arow[j + 1], y.y, p[(j >> 1) & 3]);
    }
    return ((p[0] + p[1]) + (p[2] + p[3])) - bt;
}

// The multiplier's spectrum: c_hat_m = sum_j c_j e^{-2 pi i jm/64} for m = 0..32 on threads
// 0..32; H_m = (Right ? conj c_hat_m : c_hat_m) / 128.  Returns (CTA-uniform) whether c is
// exactly singular: min_m |c_hat_m| < 1e-9 (m = 0..32 covers all bins by conjugate symmetry).
// The twiddles (cos, sin)(2 pi m / 64) sit in the staging buffer past the sign-stream scratch.
__device__ bool circ_spectrum(Smem& S, int t, bool left) {
    const uint64_t mask = S.mask;
    const double2* tw = reinterpret_cast<const double2*>(S.X + 512);
    bool sing = false;
    if (t <= 32) {
        double re = 0.0, im = 0.0;
#pragma unroll 8
        for (int j = 0; j < N; ++j) {
            const double2 w = tw[(j * t) & 63];
            const double v = sgn(mask, j);
            re = fma(v, w.x, re);
            im = fma(-v, w.y, im);
        }
        sing = sqrt(re * re + im * im) < 1e-9;
        S.H[t] = make_double2(re * 0.0078125, (left ? im : -im) * 0.0078125);
    }
    return __syncthreads_or(sing) != 0;
}

// One CTA per system; the raw arm and the whole redraw protocol (8 attempts on stream
// sid + 7919 a, right multiplier from stream ^ 0x5000000000000000) run in-kernel.
#ifndef RL_B64_MAXREG
#define RL_B64_MAXREG 248
#endif
__global__ void __maxnreg__(RL_B64_MAXREG) k_batched_circ64(
    const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ signs0, uint64_t seed,
    const uint64_t* __restrict__ sids, int refine, int left, double* __restrict__ X,
    rl_precond_report* __restrict__ rep, int* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint64_t sys = blockIdx.x;
#ifdef RL_B64_PROF
    long long prof_t0 = clock64();
#endif
    const double* Ag = A + sys * N * N;
    const double* bg = B + sys * N; // b_t is re-read where needed (keeps it out of the registers)
    {
        const unsigned bal = __ballot_sync(0xffffffffu, signs0[sys * N + t] < 0.0);
        if (lane == 0)
            S.bal[warp] = bal;
    }
    {
        const double bt = bg[t];
        const double bsq = cta_sum(S, bt * bt, t);
        if (t == 0) {
            S.mask0 = (static_cast<uint64_t>(S.bal[1]) << 32) | S.bal[0];
            S.bsq = bsq;
            S.rp = rl_precond_report{};
            S.rp.attempt = -1;
        }
    }
    rl_precond_report& rp = S.rp; // written by thread 0 only
    int st = RL_PIVOT_BREAKDOWN;
    // pass 0: raw arm (a = -1) + pre-screened protocol; pass 1 (rare): exact protocol
    for (int pass = 0; pass < 2; ++pass) {
        bool have_best = false, skipped = false, accepted = false;
        for (int a = (pass == 0 ? -1 : 0); a < 8; ++a) {
            double w[8][8];
            const int tr = t >> 3, tc = t & 7;
            if (a >= 0) {
                __syncthreads(); // X, H and the vectors are free
                if (t == 0)
                    S.mask = a == 0 ? S.mask0
                                    : sign_mask_stream(seed, (sids[sys] + 7919ULL * static_cast<uint64_t>(a)) ^
                                                                 (left ? 0ULL : 0x5000000000000000ULL),
                                                       reinterpret_cast<uint64_t*>(S.X));
                {
                    double sn, cs;
                    sincospi(static_cast<double>(t) / 32.0, &sn, &cs);
                    reinterpret_cast<double2*>(S.X + 512)[t] = make_double2(cs, sn);
                }
                __syncthreads();
                B64_MARK(1);
                const bool sing = circ_spectrum(S, t, left != 0);
                B64_MARK(2);
                if (pass == 0 && sing) {
                    skipped = true;
                    continue;
                }
                // stage A, then W = A C (row t) / C A (column t) through the FFT
#pragma unroll 4
                for (int e = t; e < N * N / 2; e += THREADS) {
                    const double2 v = reinterpret_cast<const double2*>(Ag)[e];
                    *reinterpret_cast<double2*>(S.X + ((2 * e) >> 6) * P + ((2 * e) & 63)) = v;
                }
                __syncthreads();
                double xr[N];
                if (!left) {
#pragma unroll
                    for (int j = 0; j < N; j += 2) {
                        const double2 v = *reinterpret_cast<const double2*>(S.X + t * P + j);
                        xr[j] = v.x;
                        xr[j + 1] = v.y;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < N; ++k)
                        xr[k] = S.X[k * P + t];
                }
                B64_MARK(3);
                circ_fft64(xr, S.H);
                B64_MARK(4);
                __syncthreads(); // every row / column read
                if (!left) {
#pragma unroll
                    for (int j = 0; j < N; j += 2)
                        *reinterpret_cast<double2*>(S.X + t * P + j) = make_double2(xr[j], xr[j + 1]);
                } else {
#pragma unroll
                    for (int k = 0; k < N; ++k)
                        S.X[k * P + t] = xr[k];
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        w[r][c] = S.X[(tr + 8 * r) * P + tc + 8 * c];
            } else {
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        w[r][c] = Ag[(tr + 8 * r) * N + tc + 8 * c];
            }
            const bool lft = left && a >= 0;
            double bcur = bg[t]; // the right-hand side, forward-substituted inside the LU
            if (lft) {           // rhs = C b (genp.cpp:252-255)
                S.v0[t] = bcur;
                __syncthreads();
                bcur = circ_vec(S, t);
            }
            __syncthreads(); // the spectrum, X's and v0's reads are done before the LU publishes
            B64_MARK(5);
            lu_regs(w, bcur, S, tr, tc);
            B64_MARK(6);
            __syncthreads(); // publications consumed
            lu_store(w, S, tr, tc);
            __syncthreads();
            double arow[N]; // A's row t for the residuals (L2), in flight during the fold and solve
#pragma unroll
            for (int j = 0; j < N; j += 2) {
                const double2 v = reinterpret_cast<const double2*>(Ag + t * N)[j >> 1];
                arow[j] = v.x;
                arow[j + 1] = v.y;
            }
            if (warp == 0) { // |pivot| min / max (genp.cpp:34-40) and the breakdown test
                const double p0 = fabs(S.X[lane * (P + 1)]), p1 = fabs(S.X[(lane + 32) * (P + 1)]);
                const double fl = a < 0 ? 0.0 : 1e-300;
                const bool brk = __any_sync(0xffffffffu, p0 < fl || p1 < fl);
                double mn = fmin(p0, p1), mx = fmax(p0, p1);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
                if (lane == 0) {
                    const double first = fabs(S.X[0]); // std::min/max keep a NaN first pivot
                    S.pm[0] = isnan(first) ? first : mn;
                    S.pm[1] = isnan(first) ? first : mx;
                    S.flag = brk ? 1 : 0;
                }
            }
            S.v0[t] = bcur; // L^-1 rhs
            __syncthreads();
            B64_MARK(7);
            if (S.flag && a >= 0)
                continue; // PivotBreakdown: next attempt (genp.cpp:285-288)
            B64_MARK(8);
            if (warp == 0)
                solve_warp0<false>(S, lane);
            __syncthreads();
            B64_MARK(9);
            double y = (a < 0 || lft) ? S.v0[t] : circ_vec(S, t); // y = z (Left) or C z (Right)
            __syncthreads();
            S.v1[t] = y;
            __syncthreads();
            B64_MARK(10);
            for (int s = 0; a >= 0 && s < refine; ++s) { // genp.cpp:263-274
                S.v0[t] = -row_residual(arow, S, bg[t]); // r = b - A y
                __syncthreads();
                if (lft) { // rr = C r
                    const double cr = circ_vec(S, t);
                    __syncthreads();
                    S.v0[t] = cr;
                    __syncthreads();
                }
                if (warp == 0)
                    solve_warp0<true>(S, lane);
                __syncthreads();
                y += lft ? S.v0[t] : circ_vec(S, t);
                S.v1[t] = y;
                __syncthreads();
            }
            B64_MARK(11);
            const double e = row_residual(arow, S, bg[t]);
            const double res = sqrt(cta_sum(S, e * e, t)) / sqrt(S.bsq);
            B64_MARK(12);
            if (a < 0) { // contrast arm: non-finite solution -> +inf (genp.cpp:226-231)
                const int fin = __syncthreads_and(isfinite(y));
                if (t == 0) {
                    rp.raw_residual = fin ? res : INFINITY;
                    rp.raw_pivot_min = S.pm[0];
                    rp.raw_pivot_max = S.pm[1];
                }
                continue;
            }
            const bool acc = res <= 1e-7;
            if (acc || !have_best || res < S.best_res) {
                X[sys * N + t] = y;
                __syncthreads(); // every thread has read S.best_res
                if (t == 0) {
                    rp.residual = res;
                    rp.pivot_min = S.pm[0];
                    rp.pivot_max = S.pm[1];
                    rp.attempt = a;
                    S.best_res = res;
                }
                have_best = true;
            }
            if (t == 0)
                rp.attempts_drawn = a + 1;
            if (acc) {
                accepted = true;
                break;
            }
        }
        if (accepted || have_best)
            st = 0;
        if (accepted || !skipped)
            break;
    }
    B64_MARK(13);
    if (t == 0) {
        if (rp.attempts_drawn == 0)
            rp.attempts_drawn = 8;
        rep[sys] = rp;
        if (st != 0)
            atomicExch(status, st);
    }
}

} // namespace

// Returns RL_OK or RL_PIVOT_BREAKDOWN (some system broke down on every attempt).
rl_status batched_circ64(uint64_t batch, const double* dA, const double* dB, int refine, int left, uint64_t seed,
                         const uint64_t* d_sids, double* dX, rl_precond_report* d_rep) {
    cudaStream_t st = stream();
    constexpr size_t kSmem = sizeof(Smem);
    static bool attr[16] = {};
    if (!attr[ctx().device & 15]) {
        RL_CUDA(cudaFuncSetAttribute(k_batched_circ64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kSmem)));
        attr[ctx().device & 15] = true;
    }
    double* signs = ws<double>(WS_TMP1, batch * N + 1);
    int* d_status = reinterpret_cast<int*>(signs + batch * N);
    rng_sign_vectors_batched(seed, d_sids, 0, left ? 0ULL : 0x5000000000000000ULL, batch, N, signs);
    RL_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int), st));
    k_batched_circ64<<<static_cast<unsigned>(batch), THREADS, kSmem, st>>>(dA, dB, signs, seed, d_sids, refine,
                                                                            left, dX, d_rep, d_status);
    RL_LAUNCHED();
    int h = 0;
    RL_CUDA(cudaMemcpyAsync(&h, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
    RL_CUDA(cudaStreamSynchronize(st));
    return h == 0 ? RL_OK : RL_PIVOT_BREAKDOWN;
}

} // namespace rl

// K6: batched randomized GENP for small systems (config 2: 4096 x n=64, circulant +-1,
// MulSide::Right) — semantically the loop bench::table1_genp runs (bench.cpp:117-133) over
// genp::randomized_genp (genp.cpp:207-291), one stream per system.
//
// One 128-thread CTA per system.  The working matrix lives in registers: thread t (warp
// wp = t/32, lane l) owns row r = 4 (l/2) + wp and, of that row, the columns c = 2 jj + h
// (h = l & 1, jj = 0..31) — 32 doubles, fully unrolled so every index is static.  Rows are
// dealt cyclically over the four warps so every warp has work at every pivot step.
// Per attempt:
//   * A (64 x 64, L2-resident after the first touch) is staged in shared memory and
//     W = A C runs on DMMA (warp wp computes rows 16 wp..16 wp+15); the +-1 B fragment
//     C[k][j] = c[(k - j) mod 64] is synthesised from a 64-bit sign mask.
//   * No-pivot LU (genp.cpp:20-33): per step the pivot row goes through a double-buffered
//     shared row (one barrier per step), the multiplier m = w(i,k) * (1/p) (1/p := 0 for
//     p = 0) is exchanged between the two half-row owners with one shuffle.
//   * The packed LU is spilled transposed to shared memory and warp 0 runs the forward /
//     backward substitution (two rows per lane, shuffle chain; genp.cpp:106-124), then
//     y = C z, refinement and the residual ||A y - b|| / ||b|| on threads 0..63.
// The raw-GENP contrast arm is iteration -1 of the same loop (pivot floor 0, no multiplier),
// so the unrolled LU exists once.  The 8-attempt redraw protocol (stream id + 7919 a, accept
// <= 1e-7, keep best, genp.cpp:236-290) runs in-kernel.  Exactly singular circulants (a
// vanishing 64-point DFT coefficient) are pre-screened and skipped; a
// system that exhausts its attempts is re-run with the exact protocol (pass 1) so the
// returned best attempt is the reference's.
#include <cmath>

#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int N = 64;
constexpr int THREADS = 128;
constexpr int XP = N + 4; // shared pitch: 544 B = 32 mod 128 -> conflict-free DMMA fragments
constexpr int RBH = 36;   // half-row stride inside a pivot-row buffer (16 B aligned)

struct Smem {
    double X[N * XP];      // A / W staging, transposed packed LU, LCG scratch
    double rb[2][2 * RBH]; // pivot row, double-buffered: [h * RBH + jj] = row[2 jj + h]; 1/p at [RBH - 1]
    double v0[N], v1[N];
    double2 tw[N];         // DFT twiddles (cos, sin)(2 pi m / 64)
    double red[4];
    double rcp[N];         // 1/U_kk
    uint64_t mask, mask0;
    unsigned bal[2];
    int flag;
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double sgn(uint64_t mask, int j) { // bit j set <=> c_j = -1
    return ((mask >> (j & 63)) & 1ULL) ? -1.0 : 1.0;
}

__device__ __forceinline__ double min_fold(double a, double v) { return (v < a) ? v : a; }
__device__ __forceinline__ double max_fold(double b, double v) { return (b < v) ? v : b; }

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

__device__ __forceinline__ void load_A(Smem& S, const double* __restrict__ Ag, int t) {
#pragma unroll 4
    for (int e = t; e < N * N / 2; e += THREADS) {
        const double2 v = reinterpret_cast<const double2*>(Ag)[e];
        const int i = (2 * e) >> 6, j = (2 * e) & 63;
        *reinterpret_cast<double2*>(S.X + i * XP + j) = v;
    }
}

// X holds A on entry; on exit X holds W = A C (row-major).
__device__ __forceinline__ void circ_product(Smem& S, uint64_t mask, int t) {
    const int lane = t & 31, warp = t >> 5, g = lane >> 2, q = lane & 3;
    double acc[2][8][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jb = 0; jb < 8; ++jb)
            acc[i][jb][0] = acc[i][jb][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < N; kk += 4) {
        const int k = kk + q;
        const double a0 = S.X[(16 * warp + g) * XP + k];
        const double a1 = S.X[(16 * warp + 8 + g) * XP + k];
#pragma unroll
        for (int jb = 0; jb < 8; ++jb) {
            const double bf = sgn(mask, k - (8 * jb + g)); // C[k][8 jb + g]
            dmma(acc[0][jb], a0, bf);
            dmma(acc[1][jb], a1, bf);
        }
    }
    __syncthreads(); // every read of A is done
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jb = 0; jb < 8; ++jb)
            *reinterpret_cast<double2*>(S.X + (16 * warp + 8 * i + g) * XP + 8 * jb + 2 * q) =
                make_double2(acc[i][jb][0], acc[i][jb][1]);
}

// One pivot step K (static).  Thread owns row r, half h; w[jj] = W(r, 2 jj + h).
template <int K>
__device__ __forceinline__ void lu_step(double (&w)[32], Smem& S, int r, int h, int lane, double floor, bool& brk,
                                        double& pmn, double& pmx) {
    constexpr int KJ = K >> 1, KH = K & 1;
    double* rb = S.rb[K & 1];
    if (r == K) { // publish the pivot row (entries with column >= K suffice)
        double* dst = rb + h * RBH;
#pragma unroll
        for (int jj = (KJ & ~1); jj < 32; jj += 2)
            *reinterpret_cast<double2*>(dst + jj) = make_double2(w[jj], w[jj + 1]);
        if (h == KH) {
            const double p = w[KJ];
            const double rc = (p == 0.0) ? 0.0 : 1.0 / p;
            rb[RBH - 1] = rc;
            S.rcp[K] = rc;
        }
    }
    __syncthreads();
    const double p = rb[KH * RBH + KJ], rc = rb[RBH - 1];
    const double ap = fabs(p);
    pmn = (K == 0) ? ap : min_fold(pmn, ap);
    pmx = (K == 0) ? ap : max_fold(pmx, ap);
    brk |= ap < floor;
    const double m = __shfl_sync(0xffffffffu, w[KJ] * rc, (lane & ~1) | KH);
    if (r > K) {
        if (h == KH)
            w[KJ] = m;
        if (m != 0.0) {
            const double* src = rb + h * RBH;
            if (2 * KJ == K && h == 1) // column K + 1 when K is even
                w[KJ] = fma(-m, src[KJ], w[KJ]);
#pragma unroll
            for (int jj = KJ + 1; jj < 32; ++jj)
                w[jj] = fma(-m, src[jj], w[jj]);
        }
    }
}

template <int K0, int K1>
struct LU {
    __device__ __forceinline__ static void run(double (&w)[32], Smem& S, int r, int h, int lane, double floor,
                                               bool& brk, double& pmn, double& pmx) {
        lu_step<K0>(w, S, r, h, lane, floor, brk, pmn, pmx);
        LU<K0 + 1, K1>::run(w, S, r, h, lane, floor, brk, pmn, pmx);
    }
};
template <int K1>
struct LU<K1, K1> {
    __device__ __forceinline__ static void run(double (&)[32], Smem&, int, int, int, double, bool&, double&,
                                               double&) {}
};

// warp 0: S.v0 <- U^{-1} L^{-1} S.v0 with the packed LU transposed in X (X[c * XP + r]).
__device__ __forceinline__ void solve_warp0(Smem& S, int lane) {
    double x0 = S.v0[lane], x1 = S.v0[lane + 32];
#pragma unroll
    for (int j = 0; j < N; ++j) { // forward, unit L
        const double yj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
        if (j < 32 && lane > j)
            x0 = fma(-S.X[j * XP + lane], yj, x0);
        if (lane + 32 > j)
            x1 = fma(-S.X[j * XP + lane + 32], yj, x1);
    }
#pragma unroll
    for (int j = N - 1; j >= 0; --j) { // backward, U
        const double xj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31) * S.rcp[j];
        if (j < 32) {
            if (lane == j)
                x0 = xj;
            else if (lane < j)
                x0 = fma(-S.X[j * XP + lane], xj, x0);
        } else {
            if (lane + 32 == j)
                x1 = xj;
            else if (lane + 32 < j)
                x1 = fma(-S.X[j * XP + lane + 32], xj, x1);
            x0 = fma(-S.X[j * XP + lane], xj, x0);
        }
    }
    S.v0[lane] = x0;
    S.v0[lane + 32] = x1;
}

// (C z)_t, z in S.v0 (t < 64)
__device__ __forceinline__ double circ_vec(const Smem& S, uint64_t mask, int t) {
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
    const double s = (S.red[0] + S.red[1]) + (S.red[2] + S.red[3]);
    __syncthreads();
    return s;
}

// (A y)_t - b_t (t < 64), A's row t from global (L2), y in S.v1
__device__ __forceinline__ double row_residual(const double* __restrict__ Ag, const Smem& S, double bt, int t) {
    const double2* row = reinterpret_cast<const double2*>(Ag + t * N);
    double s = 0.0;
#pragma unroll 8
    for (int j = 0; j < N / 2; ++j) {
        const double2 a = row[j];
        s = fma(a.x, S.v1[2 * j], s);
        s = fma(a.y, S.v1[2 * j + 1], s);
    }
    return s - bt;
}

// exact singularity pre-screen: min_k |DFT(c)_k| < 1e-9 (k = 0..32 by conjugate symmetry)
__device__ bool circ_singular(Smem& S, uint64_t mask, int t) {
    bool sing = false;
    if (t <= 32) {
        double re = 0.0, im = 0.0;
#pragma unroll 8
        for (int j = 0; j < N; ++j) {
            const double2 w = S.tw[(j * t) & 63];
            const double v = sgn(mask, j);
            re = fma(v, w.x, re);
            im = fma(-v, w.y, im);
        }
        sing = sqrt(re * re + im * im) < 1e-9;
    }
    return __syncthreads_or(sing) != 0;
}

// One CTA per system; the raw arm and the whole redraw protocol (8 attempts on stream
// sid + 7919 a, right multiplier from stream ^ 0x5000000000000000) run in-kernel.
__global__ void __launch_bounds__(THREADS, 5) k_batched_circ64(
    const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ signs0, uint64_t seed,
    const uint64_t* __restrict__ sids, int refine, double* __restrict__ X, rl_precond_report* __restrict__ rep,
    int* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int r = 4 * (lane >> 1) + warp, h = lane & 1; // LU ownership
    const bool vt = t < N;                              // vector-row owner (row t)
    const uint64_t sys = blockIdx.x;
    const double* Ag = A + sys * N * N;
    const double bt = vt ? B[sys * N + t] : 0.0;
    if (vt) {
        const unsigned bal = __ballot_sync(0xffffffffu, signs0[sys * N + t] < 0.0);
        if (lane == 0)
            S.bal[warp] = bal;
        double s, c;
        sincospi(static_cast<double>(t) / 32.0, &s, &c);
        S.tw[t] = make_double2(c, s);
    }
    __syncthreads();
    if (t == 0)
        S.mask0 = (static_cast<uint64_t>(S.bal[1]) << 32) | S.bal[0];
    const double bsq = cta_sum(S, bt * bt, t);
    const uint64_t sid = sids[sys];
    double* xg = X + sys * N;
    rl_precond_report rp{};
    rp.attempt = -1;
    int st = RL_PIVOT_BREAKDOWN;
    double w[32];
    // pass 0: raw arm (a = -1) + pre-screened protocol; pass 1 (rare): exact protocol
    for (int pass = 0; pass < 2; ++pass) {
        bool have_best = false, skipped = false, accepted = false;
        double best_res = 0.0;
        for (int a = (pass == 0 ? -1 : 0); a < 8; ++a) {
            uint64_t mask = 0;
            if (a >= 0) {
                __syncthreads(); // X is free
                if (a == 0) {
                    mask = S.mask0;
                } else {
                    if (t == 0)
                        S.mask = sign_mask_stream(seed, (sid + 7919ULL * static_cast<uint64_t>(a)) ^
                                                            0x5000000000000000ULL,
                                                  reinterpret_cast<uint64_t*>(S.X));
                    __syncthreads();
                    mask = S.mask;
                }
                if (pass == 0 && circ_singular(S, mask, t)) {
                    skipped = true;
                    continue;
                }
            }
            __syncthreads();
            load_A(S, Ag, t);
            __syncthreads();
            if (a >= 0) {
                circ_product(S, mask, t);
                __syncthreads();
            }
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
                w[jj] = S.X[r * XP + 2 * jj + h];
            bool brk = false;
            double pmn = 0.0, pmx = 0.0;
            LU<0, N>::run(w, S, r, h, lane, a < 0 ? 0.0 : 1e-300, brk, pmn, pmx);
            if (__syncthreads_or(brk) && a >= 0)
                continue; // PivotBreakdown: next attempt (genp.cpp:285-288)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
                S.X[(2 * jj + h) * XP + r] = w[jj];
            if (vt)
                S.v0[t] = bt;
            __syncthreads();
            if (warp == 0)
                solve_warp0(S, lane);
            __syncthreads();
            double y = 0.0;
            if (vt)
                y = (a < 0) ? S.v0[t] : circ_vec(S, mask, t);
            __syncthreads();
            if (vt)
                S.v1[t] = y;
            __syncthreads();
            for (int s = 0; a >= 0 && s < refine; ++s) { // genp.cpp:263-274
                if (vt)
                    S.v0[t] = -row_residual(Ag, S, bt, t); // b - A y
                __syncthreads();
                if (warp == 0)
                    solve_warp0(S, lane);
                __syncthreads();
                if (vt) {
                    y += circ_vec(S, mask, t);
                    S.v1[t] = y;
                }
                __syncthreads();
            }
            const double e = vt ? row_residual(Ag, S, bt, t) : 0.0;
            const double res = sqrt(cta_sum(S, e * e, t)) / sqrt(bsq);
            if (a < 0) { // contrast arm: non-finite solution -> +inf (genp.cpp:226-231)
                const int fin = __syncthreads_and(!vt || isfinite(y));
                rp.raw_residual = fin ? res : INFINITY;
                rp.raw_pivot_min = pmn;
                rp.raw_pivot_max = pmx;
                continue;
            }
            const bool acc = res <= 1e-7;
            if (acc || !have_best || res < best_res) {
                if (vt)
                    xg[t] = y;
                rp.residual = res;
                rp.pivot_min = pmn;
                rp.pivot_max = pmx;
                rp.attempt = a;
                best_res = res;
                have_best = true;
            }
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
rl_status batched_circ64(uint64_t batch, const double* dA, const double* dB, int refine, uint64_t seed,
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
    rng_sign_vectors_batched(seed, d_sids, 0, 0x5000000000000000ULL, batch, N, signs);
    RL_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int), st));
    k_batched_circ64<<<static_cast<unsigned>(batch), THREADS, kSmem, st>>>(dA, dB, signs, seed, d_sids, refine,
                                                                            dX, d_rep, d_status);
    RL_LAUNCHED();
    int h = 0;
    RL_CUDA(cudaMemcpyAsync(&h, d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
    RL_CUDA(cudaStreamSynchronize(st));
    return h == 0 ? RL_OK : RL_PIVOT_BREAKDOWN;
}

} // namespace rl

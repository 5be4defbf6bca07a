// K6: batched randomized GENP for small systems (config 2: 4096 x n=64, circulant +-1,
// MulSide::Right) — semantically the loop bench::table1_genp runs (bench.cpp:117-133) over
// genp::randomized_genp (genp.cpp:207-291), one stream per system.
//
// One 128-thread CTA per system, the 64 x 64 working matrix in shared memory (pitch 68 doubles:
// conflict-free DMMA fragments).  Per attempt:
//   * A (64 x 64, L2-resident after the first touch) is staged in shared memory and
//     W = A C runs on DMMA (warp wp computes rows 16 wp..16 wp+15); the +-1 B fragment
//     C[k][j] = c[(k - j) mod 64] is synthesised from a 64-bit sign mask.
//   * No-pivot LU (genp.cpp:20-33) blocked in four 16-column panels: warp 0 factors the
//     panel in registers (pivot row by shuffles, m = w(i,k) * (1/p), 1/p := 0 for p = 0),
//     one thread per column solves U12 against the unit L11, all warps update the trailing
//     square on DMMA — three barriers per panel instead of one per pivot.
//   * Warp 0 runs the forward / backward substitution on the packed LU (two rows per lane,
//     shuffle chain; genp.cpp:106-124), then y = C z,
//     refinement and the residual ||A y - b|| / ||b|| on threads 0..63.
// The raw-GENP contrast arm is iteration -1 of the same loop (pivot floor 0, no multiplier).  The 8-attempt redraw protocol (stream id + 7919 a, accept
// <= 1e-7, keep best, genp.cpp:236-290) runs in-kernel.  Exactly singular circulants (a
// vanishing 64-point DFT coefficient) are pre-screened and skipped; a
// system that exhausts its attempts is re-run with the exact protocol (pass 1) so the
// returned best attempt is the reference's.
#include <cmath>

#include "panel.cuh"
#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int N = 64;
constexpr int THREADS = 128;
constexpr int XP = N + 4; // shared pitch: 544 B = 32 mod 128 -> conflict-free DMMA fragments

struct Smem {
    double X[N * XP];      // A / W staging, transposed packed LU, LCG scratch
    double pm[2];          // running |pivot| min / max of the LU
    double v0[N], v1[N];
    double2 tw[N];         // DFT twiddles (cos, sin)(2 pi m / 64)
    double red[4];
    double rcp[N];         // 1/U_kk
    uint64_t mask, mask0;
    unsigned bal[2];
    int flag;
    rl_precond_report rp; // the system's report (thread 0), kept out of the register budget
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

// 1/p on the pivot chain: the hardware estimate plus two Newton steps (a few cycles instead of
// __drcp_rn's correctly rounded sequence); p is warp-uniform, so the rare tiny-|p| fallback
// does not diverge. 0 -> 0 (the reference's m = 0 for a zero pivot).
__device__ __forceinline__ double pivot_rcp(double p) {
    if (p == 0.0)
        return 0.0;
    if (!(fabs(p) > 1e-300 && fabs(p) < 1e300))
        return __drcp_rn(p);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
    double e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    e = fma(-p, r, 1.0);
    return fma(r, e, r);
}
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

// X holds A on entry; on exit X holds W = A C (row-major).  Two passes over the output's
// column halves (16 accumulators each instead of 32: the kernel's register peak, which sets
// how many systems share an SM); W goes to registers first, then over A after a barrier.
__device__ __forceinline__ void circ_product(Smem& S, uint64_t mask, int t, bool left) {
    const int lane = t & 31, warp = t >> 5, g = lane >> 2, q = lane & 3;
    double keep[2][4][2];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        double acc[2][4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jb = 0; jb < 4; ++jb)
                acc[i][jb][0] = acc[i][jb][1] = 0.0;
#pragma unroll 4
        for (int kk = 0; kk < N; kk += 4) {
            const int k = kk + q;
            if (!left) { // W = A C: A rows from shared memory, C[k][8 jb' + g] = c[k - col]
                const double a0 = S.X[(16 * warp + g) * XP + k];
                const double a1 = S.X[(16 * warp + 8 + g) * XP + k];
#pragma unroll
                for (int jb = 0; jb < 4; ++jb) {
                    const double bf = sgn(mask, k - (8 * (4 * half + jb) + g));
                    dmma(acc[0][jb], a0, bf);
                    dmma(acc[1][jb], a1, bf);
                }
            } else { // W = C A: C[row][k] = c[row - k] synthesised, A[k][col] from shared memory
                const double c0 = sgn(mask, (16 * warp + g) - k);
                const double c1 = sgn(mask, (16 * warp + 8 + g) - k);
#pragma unroll
                for (int jb = 0; jb < 4; ++jb) {
                    const double bf = S.X[k * XP + 8 * (4 * half + jb) + g];
                    dmma(acc[0][jb], c0, bf);
                    dmma(acc[1][jb], c1, bf);
                }
            }
        }
        if (half == 0) {
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int jb = 0; jb < 4; ++jb) {
                    keep[i][jb][0] = acc[i][jb][0];
                    keep[i][jb][1] = acc[i][jb][1];
                }
        } else {
            __syncthreads(); // every read of A is done
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int jb = 0; jb < 4; ++jb) {
                    double* row = S.X + (16 * warp + 8 * i + g) * XP + 2 * q;
                    *reinterpret_cast<double2*>(row + 8 * jb) = make_double2(keep[i][jb][0], keep[i][jb][1]);
                    *reinterpret_cast<double2*>(row + 8 * (4 + jb)) = make_double2(acc[i][jb][0], acc[i][jb][1]);
                }
        }
    }
}

// Blocked no-pivot LU of the 64 x 64 working matrix in S.X (row-major, genp.cpp:20-33 per
// column step): four 16-column panels.  (a) warp 0 factors the panel rows c0..63 x 16 in
// registers (two rows per lane, pivot row by shuffles, 1/p := 0 for p = 0), (b) every column
// right of the panel solves its 16 U entries against the unit L11 (one thread per column),
// (c) the trailing square is updated on DMMA (K = 16) by all warps.  Three barriers per panel
// instead of one per pivot.  Returns breakdown (some |p| < floor); pmin/pmax of |pivots|
// (in pivot order) for every thread; S.rcp = 1/U_kk.
__device__ __forceinline__ bool lu_blocked(Smem& S, double floor, int t, double& pmin, double& pmax) {
    const int lane = t & 31, warp = t >> 5;
#pragma unroll 1
    for (int c0 = 0; c0 < N; c0 += 16) {
        if (warp == 0) { // (a) the 16 x 16 diagonal block: lane l < 16 holds row c0 + l
            const bool v = lane < 16;
            const int r = c0 + (lane & 15);
            double a[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
                a[j] = v ? S.X[r * XP + c0 + j] : 0.0;
            double mn = S.pm[0], mx = S.pm[1];
            bool brk = S.flag != 0;
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                const double piv = __shfl_sync(0xffffffffu, a[kk], kk);
                const double inv = pivot_rcp(piv);
                if (lane == 0)
                    S.rcp[c0 + kk] = inv;
                const double ap = fabs(piv);
                mn = (c0 + kk == 0) ? ap : min_fold(mn, ap);
                mx = (c0 + kk == 0) ? ap : max_fold(mx, ap);
                brk |= ap < floor;
                const bool below = v && lane > kk;
                const double m = below ? a[kk] * inv : 0.0;
                a[kk] = below ? m : a[kk];
#pragma unroll
                for (int l = kk + 1; l < 16; ++l)
                    a[l] = fma(-m, __shfl_sync(0xffffffffu, a[l], kk), a[l]);
            }
            if (v)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    S.X[r * XP + c0 + j] = a[j];
            if (lane == 0) {
                S.pm[0] = mn;
                S.pm[1] = mx;
                if (brk)
                    S.flag = 1;
            }
        }
        __syncthreads();
        const int nc = N - c0 - 16;
        if (nc == 0)
            break;
        // (b) one thread per row below the block (L21 = A21 U11^-1: the same multipliers and
        // updates, in the same order, as eliminating the rows inside the pivot loop) and one
        // per column right of it (U12 = L11^-1 A12), warps 0-1 and 2-3
        if (t < nc) {
            const int i = c0 + 16 + t;
            double y[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
                y[j] = S.X[i * XP + c0 + j];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const double m = y[k] * S.rcp[c0 + k];
                y[k] = m;
#pragma unroll
                for (int l = k + 1; l < 16; ++l)
                    y[l] = fma(-m, S.X[(c0 + k) * XP + c0 + l], y[l]);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j)
                S.X[i * XP + c0 + j] = y[j];
        } else if (t >= 64 && t - 64 < nc) {
            const int c = c0 + 16 + (t - 64);
            double y[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
                y[i] = S.X[(c0 + i) * XP + c];
#pragma unroll
            for (int i = 1; i < 16; ++i)
#pragma unroll
                for (int k = 0; k < i; ++k)
                    y[i] = fma(-S.X[(c0 + i) * XP + c0 + k], y[k], y[i]);
#pragma unroll
            for (int i = 1; i < 16; ++i)
                S.X[(c0 + i) * XP + c] = y[i];
        }
        __syncthreads();
        panel::smem_update16(S.X + (c0 + 16) * XP + c0 + 16, XP, S.X + (c0 + 16) * XP + c0, XP,
                             S.X + c0 * XP + c0 + 16, XP, nc, nc, warp, THREADS / 32, lane);
        __syncthreads();
    }
    pmin = S.pm[0];
    pmax = S.pm[1];
    return S.flag != 0;
}

// warp 0: S.v0 <- U^{-1} L^{-1} S.v0 with the packed LU row-major in X (L_ij = X[i * XP + j]
// below the diagonal, U on and above). Lane l owns rows l and l + 32; step j reads column j of
// L or U down the lanes (a 4-way bank conflict at pitch 68, far cheaper than transposing X).
__device__ __forceinline__ void solve_warp0(Smem& S, int lane) {
    double x0 = S.v0[lane], x1 = S.v0[lane + 32];
    const double* r0 = S.X + lane * XP;
    const double* r1 = S.X + (lane + 32) * XP;
#pragma unroll
    for (int j = 0; j < N; ++j) { // forward, unit L
        const double yj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
        if (j < 32 && lane > j)
            x0 = fma(-r0[j], yj, x0);
        if (lane + 32 > j)
            x1 = fma(-r1[j], yj, x1);
    }
#pragma unroll
    for (int j = N - 1; j >= 0; --j) { // backward, U
        const double xj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31) * S.rcp[j];
        if (j < 32) {
            if (lane == j)
                x0 = xj;
            else if (lane < j)
                x0 = fma(-r0[j], xj, x0);
        } else {
            if (lane + 32 == j)
                x1 = xj;
            else if (lane + 32 < j)
                x1 = fma(-r1[j], xj, x1);
            x0 = fma(-r0[j], xj, x0);
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
__global__ void __launch_bounds__(THREADS, 6) k_batched_circ64(
    const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ signs0, uint64_t seed,
    const uint64_t* __restrict__ sids, int refine, int left, double* __restrict__ X,
    rl_precond_report* __restrict__ rep, int* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
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
    rl_precond_report& rp = S.rp; // written by thread 0 only
    if (t == 0) {
        rp = rl_precond_report{};
        rp.attempt = -1;
    }
    int st = RL_PIVOT_BREAKDOWN;
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
                                                            (left ? 0ULL : 0x5000000000000000ULL),
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
                circ_product(S, mask, t, left != 0);
                __syncthreads();
            }
            if (t == 0) {
                S.flag = 0;
                S.pm[0] = S.pm[1] = 0.0;
            }
            __syncthreads();
            double pmn = 0.0, pmx = 0.0;
            const bool brk = lu_blocked(S, a < 0 ? 0.0 : 1e-300, t, pmn, pmx);
            if (brk && a >= 0)
                continue; // PivotBreakdown: next attempt (genp.cpp:285-288)
            const bool lft = left && a >= 0;
            if (vt)
                S.v0[t] = bt;
            __syncthreads();
            if (lft) { // rhs = C b (genp.cpp:252-255)
                const double cb = vt ? circ_vec(S, mask, t) : 0.0;
                __syncthreads();
                if (vt)
                    S.v0[t] = cb;
                __syncthreads();
            }
            if (warp == 0)
                solve_warp0(S, lane);
            __syncthreads();
            double y = 0.0;
            if (vt)
                y = (a < 0 || lft) ? S.v0[t] : circ_vec(S, mask, t); // y = z (Left) or C z (Right)
            __syncthreads();
            if (vt)
                S.v1[t] = y;
            __syncthreads();
            for (int s = 0; a >= 0 && s < refine; ++s) { // genp.cpp:263-274
                if (vt)
                    S.v0[t] = -row_residual(Ag, S, bt, t); // r = b - A y
                __syncthreads();
                if (lft) { // rr = C r
                    const double cr = vt ? circ_vec(S, mask, t) : 0.0;
                    __syncthreads();
                    if (vt)
                        S.v0[t] = cr;
                    __syncthreads();
                }
                if (warp == 0)
                    solve_warp0(S, lane);
                __syncthreads();
                if (vt) {
                    y += lft ? S.v0[t] : circ_vec(S, mask, t);
                    S.v1[t] = y;
                }
                __syncthreads();
            }
            const double e = vt ? row_residual(Ag, S, bt, t) : 0.0;
            const double res = sqrt(cta_sum(S, e * e, t)) / sqrt(bsq);
            if (a < 0) { // contrast arm: non-finite solution -> +inf (genp.cpp:226-231)
                const int fin = __syncthreads_and(!vt || isfinite(y));
                if (t == 0) {
                    rp.raw_residual = fin ? res : INFINITY;
                    rp.raw_pivot_min = pmn;
                    rp.raw_pivot_max = pmx;
                }
                continue;
            }
            const bool acc = res <= 1e-7;
            if (acc || !have_best || res < best_res) {
                if (vt)
                    xg[t] = y;
                if (t == 0) {
                    rp.residual = res;
                    rp.pivot_min = pmn;
                    rp.pivot_max = pmx;
                    rp.attempt = a;
                }
                best_res = res;
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

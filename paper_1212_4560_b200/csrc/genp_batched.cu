// K6: batched randomized GENP for small systems (config 2: 4096 x n=64, circulant +-1,
// MulSide::Right) — semantically the loop bench::table1_genp runs (bench.cpp:117-133)
// over genp::randomized_genp (genp.cpp:207-291), one stream per system.
//
// One CTA (8 warps) per system, everything on-chip:
//   * A (64 x 64) read from HBM once into shared memory (kept for the residuals).
//   * W = A C on DMMA: warp w owns rows 8w..8w+7; the B-operand fragment
//     C[k][j] = c[(k - j) mod 64] is synthesised from the 64-bit sign mask in a
//     register (no smem traffic for C).  The accumulators stay in registers and ARE
//     the LU's data layout: lane (g, t) of warp w owns row 8w+g, columns 8jb+2t, +1.
//   * No-pivot LU with the rows in registers: per step the pivot row goes through a
//     double-buffered shared row (one __syncthreads per step) and the multiplier
//     w(i,k)/p is broadcast inside the row's 4-lane group with __shfl_sync.
//   * Solves, y = C z, refinement and the residual ||A y - b|| / ||b|| on-chip.
// The redraw protocol (8 attempts on stream id + 7919 a, accept <= 1e-7, keep best,
// genp.cpp:236-290) runs as one launch per attempt over the still-unaccepted systems.
// A circulant +-1 C is exactly singular iff a DFT coefficient of c vanishes
// (SURVEY.md §0 item 4): such attempts are pre-screened and skipped; if a system
// ever exhausts its attempts, it is recomputed without the pre-screen so the
// returned "best" attempt is exactly the reference's choice.
#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int N = 64;
constexpr int P = N + 1;   // smem pitch
constexpr int THREADS = 256;

struct SysState {          // per system, persistent across attempt launches
    double best_res;
    int have_best;
    int accepted;          // attempt index accepted, -1 none
    int skipped;           // attempts skipped by the singularity pre-screen
    int status;            // 0 ok, RL_PIVOT_BREAKDOWN if every attempt broke down
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// element (row, col) of the register layout: row = 8w+g, cols 8jb+2t+e
struct Regs {
    double v[8][2];
};

// signs bit j = 1 <=> c_j = -1
__device__ __forceinline__ double sgn(uint64_t mask, int j) {
    return ((mask >> (j & 63)) & 1ULL) ? -1.0 : 1.0;
}

// W = A C (A in smem), result in the register layout
__device__ void circ_right_dmma(const double* As, uint64_t mask, int warp, int g, int t, Regs& W) {
#pragma unroll
    for (int jb = 0; jb < 8; ++jb)
        W.v[jb][0] = W.v[jb][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < N; kk += 4) {
        double a = As[(8 * warp + g) * P + kk + t];
        const int k = kk + t;
#pragma unroll
        for (int jb = 0; jb < 8; ++jb) {
            // B fragment element: row k, col 8jb+g -> C[k][j] = c[(k - j) mod 64]
            double b = sgn(mask, k - (8 * jb + g));
            dmma(W.v[jb], a, b);
        }
    }
}

// No-pivot LU in registers; returns breakdown flag; pmin/pmax of |pivots|.
__device__ bool lu_regs(Regs& W, double floor, double* rowbuf, int warp, int g, int t, int lane,
                        double* pmin, double* pmax) {
    const int row = 8 * warp + g;
    bool brk = false;
    double mn = 0.0, mx = 0.0;
    for (int k = 0; k < N; ++k) {
        double* rb = rowbuf + (k & 1) * N;
        if (row == k) {
#pragma unroll
            for (int jb = 0; jb < 8; ++jb)
                *reinterpret_cast<double2*>(rb + 8 * jb + 2 * t) = make_double2(W.v[jb][0], W.v[jb][1]);
        }
        __syncthreads();
        const double p = rb[k];
        const double ap = fabs(p);
        if (k == 0) {
            mn = mx = ap;
        } else {
            mn = (ap < mn) ? ap : mn;
            mx = (mx < ap) ? ap : mx;
        }
        brk |= (ap < floor);
        // multiplier for my row from the lane owning column k
        const int jbk = k >> 3, tk = (k & 7) >> 1, ek = k & 1;
        double mine = 0.0;
#pragma unroll
        for (int jb = 0; jb < 8; ++jb)
            if (jb == jbk)
                mine = ek ? W.v[jb][1] : W.v[jb][0];
        double m = (p == 0.0) ? 0.0 : mine / p;
        m = __shfl_sync(0xffffffffu, m, (lane & ~3) | tk);
        if (row > k) {
            if (t == tk) {
#pragma unroll
                for (int jb = 0; jb < 8; ++jb)
                    if (jb == jbk) {
                        if (ek)
                            W.v[jb][1] = m;
                        else
                            W.v[jb][0] = m;
                    }
            }
            if (m != 0.0) {
#pragma unroll
                for (int jb = 0; jb < 8; ++jb) {
                    const int j0 = 8 * jb + 2 * t;
                    double2 r = *reinterpret_cast<const double2*>(rb + j0);
                    if (j0 > k)
                        W.v[jb][0] = fma(-m, r.x, W.v[jb][0]);
                    if (j0 + 1 > k)
                        W.v[jb][1] = fma(-m, r.y, W.v[jb][1]);
                }
            }
        }
    }
    *pmin = mn;
    *pmax = mx;
    return brk;
}

// spill the packed LU to smem (pitch P)
__device__ void regs_to_smem(const Regs& W, double* Ws, int warp, int g, int t) {
    const int row = 8 * warp + g;
#pragma unroll
    for (int jb = 0; jb < 8; ++jb) {
        Ws[row * P + 8 * jb + 2 * t] = W.v[jb][0];
        Ws[row * P + 8 * jb + 2 * t + 1] = W.v[jb][1];
    }
}

// warp 0: x <- LU^{-1} x  (forward unit-L, backward U; genp.cpp:106-124 order of terms)
__device__ void lu_solve_warp(const double* Ws, double* x, int lane) {
    double x0 = x[lane], x1 = x[lane + 32];
    for (int j = 0; j < N; ++j) {
        double zj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
        if (lane > j)
            x0 = fma(-Ws[lane * P + j], zj, x0);
        if (lane + 32 > j)
            x1 = fma(-Ws[(lane + 32) * P + j], zj, x1);
    }
    for (int j = N - 1; j >= 0; --j) {
        double xj = __shfl_sync(0xffffffffu, j < 32 ? x0 : x1, j & 31);
        xj = xj / Ws[j * P + j];
        if (lane == (j & 31)) {
            if (j < 32)
                x0 = xj;
            else
                x1 = xj;
        }
        if (lane < j)
            x0 = fma(-Ws[lane * P + j], xj, x0);
        if (lane + 32 < j)
            x1 = fma(-Ws[(lane + 32) * P + j], xj, x1);
    }
    x[lane] = x0;
    x[lane + 32] = x1;
}

// y = C z (warp 0): y_i = sum_j c[(i - j) mod 64] z_j
__device__ void circ_vec_warp(uint64_t mask, const double* z, double* y, int lane) {
    double y0 = 0.0, y1 = 0.0;
    for (int j = 0; j < N; ++j) {
        double zj = z[j];
        y0 = fma(sgn(mask, lane - j), zj, y0);
        y1 = fma(sgn(mask, lane + 32 - j), zj, y1);
    }
    __syncwarp();
    y[lane] = y0;
    y[lane + 32] = y1;
}

// ||A y - b|| / ||b|| (all threads; result broadcast through red[])
__device__ double rel_residual(const double* As, const double* y, const double* b, double* red,
                               double* rvec, int tid) {
    // 4 threads per row
    const int i = tid >> 2, q = tid & 3;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j)
        s = fma(As[i * P + q * 16 + j], y[q * 16 + j], s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q == 0)
        rvec[i] = s - b[i];
    __syncthreads();
    if (tid < 32) {
        double d0 = rvec[tid], d1 = rvec[tid + 32];
        double num = d0 * d0 + d1 * d1;
        double den = b[tid] * b[tid] + b[tid + 32] * b[tid + 32];
        for (int off = 16; off > 0; off >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, off);
            den += __shfl_xor_sync(0xffffffffu, den, off);
        }
        if (tid == 0)
            red[0] = sqrt(num) / sqrt(den);
    }
    __syncthreads();
    return red[0];
}

__device__ bool all_finite64(const double* v, int tid, int* flag) {
    if (tid == 0)
        *flag = 1;
    __syncthreads();
    if (tid < N && !isfinite(v[tid]))
        *flag = 0;
    __syncthreads();
    return *flag != 0;
}

// exact singularity pre-screen: min_k |DFT(c)_k| < 1e-9
__device__ bool circ_singular(uint64_t mask, int tid, int* flag) {
    if (tid == 0)
        *flag = 0;
    __syncthreads();
    if (tid <= 32) { // k = 0..32 (conjugate symmetry)
        const int k = tid;
        double re = 0.0, im = 0.0;
        for (int j = 0; j < N; ++j) {
            double s, c;
            sincospi(static_cast<double>((j * k) & 63) / 32.0, &s, &c);
            double v = sgn(mask, j);
            re = fma(v, c, re);
            im = fma(-v, s, im);
        }
        if (sqrt(re * re + im * im) < 1e-9)
            atomicOr(flag, 1);
    }
    __syncthreads();
    return *flag != 0;
}

__global__ void __launch_bounds__(THREADS) k_batched_circ64(
    const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ signs,
    const int* __restrict__ active, int nactive, int attempt, int refine, int prescreen, int do_raw,
    double* __restrict__ X, rl_precond_report* __restrict__ rep, SysState* __restrict__ state,
    int* __restrict__ pending) {
    extern __shared__ double dsm[];
    double* As = dsm;          // N x P
    double* Ws = dsm + N * P;  // N x P
    __shared__ double rowbuf[2 * N];
    __shared__ double bv[N], yv[N], zv[N], rv[N], red[2];
    __shared__ int flag;
    if (static_cast<int>(blockIdx.x) >= nactive)
        return;
    const int sys = active ? active[blockIdx.x] : blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const double* Ag = A + static_cast<size_t>(sys) * N * N;
    for (int e = tid; e < N * N / 2; e += THREADS) {
        double2 v = reinterpret_cast<const double2*>(Ag)[e];
        int i = (2 * e) / N, j = (2 * e) % N;
        As[i * P + j] = v.x;
        As[i * P + j + 1] = v.y;
    }
    if (tid < N)
        bv[tid] = B[static_cast<size_t>(sys) * N + tid];
    uint64_t mask = 0;
    {
        // sign vector of this attempt -> bitmask (bit j set <=> c_j = -1)
        const double* sg = signs + static_cast<size_t>(blockIdx.x) * N;
        double v0 = sg[lane], v1 = sg[lane + 32];
        unsigned lo = __ballot_sync(0xffffffffu, v0 < 0.0), hi = __ballot_sync(0xffffffffu, v1 < 0.0);
        mask = (static_cast<uint64_t>(hi) << 32) | lo;
    }
    __syncthreads();
    rl_precond_report* r = rep + sys;
    SysState* stt = state + sys;
    Regs W;

    if (do_raw) {
        // raw-GENP contrast arm on A (genp.cpp:222-234), pivot floor 0
#pragma unroll
        for (int jb = 0; jb < 8; ++jb) {
            W.v[jb][0] = As[(8 * warp + g) * P + 8 * jb + 2 * t];
            W.v[jb][1] = As[(8 * warp + g) * P + 8 * jb + 2 * t + 1];
        }
        double pmn, pmx;
        lu_regs(W, 0.0, rowbuf, warp, g, t, lane, &pmn, &pmx);
        regs_to_smem(W, Ws, warp, g, t);
        if (tid < N)
            zv[tid] = bv[tid];
        __syncthreads();
        if (warp == 0)
            lu_solve_warp(Ws, zv, lane);
        __syncthreads();
        bool fin = all_finite64(zv, tid, &flag);
        double rr = fin ? rel_residual(As, zv, bv, red, rv, tid) : INFINITY;
        if (tid == 0) {
            r->raw_residual = rr;
            r->raw_pivot_min = pmn;
            r->raw_pivot_max = pmx;
            r->residual = 0.0;
            r->pivot_min = 0.0;
            r->pivot_max = 0.0;
            r->attempt = -1;
            r->attempts_drawn = 0;
            stt->best_res = 0.0;
            stt->have_best = 0;
            stt->accepted = -1;
            stt->skipped = 0;
            stt->status = 0;
        }
        __syncthreads();
    }
    if (tid == 0)
        r->attempts_drawn = attempt + 1;
    if (prescreen && circ_singular(mask, tid, &flag)) {
        if (tid == 0) {
            stt->skipped += 1;
            if (attempt < 7)
                atomicAdd(pending, 1);
        }
        return;
    }
    circ_right_dmma(As, mask, warp, g, t, W);
    double pmn, pmx;
    bool brk = lu_regs(W, 1e-300, rowbuf, warp, g, t, lane, &pmn, &pmx);
    if (brk) { // PivotBreakdown: next attempt (genp.cpp:285-288)
        if (tid == 0) {
            if (attempt < 7)
                atomicAdd(pending, 1);
            else if (!stt->have_best)
                stt->status = RL_PIVOT_BREAKDOWN;
        }
        return;
    }
    regs_to_smem(W, Ws, warp, g, t);
    if (tid < N)
        zv[tid] = bv[tid];
    __syncthreads();
    if (warp == 0) {
        lu_solve_warp(Ws, zv, lane);
        __syncwarp();
        circ_vec_warp(mask, zv, yv, lane);
    }
    __syncthreads();
    for (int s = 0; s < refine; ++s) {
        // r = b - A y ; w = solve(r) ; d = C w ; y += d   (genp.cpp:263-274)
        {
            const int i = tid >> 2, q = tid & 3;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                acc = fma(As[i * P + q * 16 + j], yv[q * 16 + j], acc);
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if (q == 0)
                zv[i] = bv[i] - acc;
        }
        __syncthreads();
        if (warp == 0) {
            lu_solve_warp(Ws, zv, lane);
            __syncwarp();
            circ_vec_warp(mask, zv, rv, lane);
            __syncwarp();
            yv[lane] += rv[lane];
            yv[lane + 32] += rv[lane + 32];
        }
        __syncthreads();
    }
    double res = rel_residual(As, yv, bv, red, rv, tid);
    bool accept = res <= 1e-7;
    bool better = !stt->have_best || res < stt->best_res;
    __syncthreads();
    if (accept || better) {
        if (tid < N)
            X[static_cast<size_t>(sys) * N + tid] = yv[tid];
        if (tid == 0) {
            r->residual = res;
            r->pivot_min = pmn;
            r->pivot_max = pmx;
            r->attempt = attempt;
            stt->best_res = res;
            stt->have_best = 1;
        }
    }
    if (tid == 0) {
        if (accept)
            stt->accepted = attempt;
        else if (attempt < 7)
            atomicAdd(pending, 1);
    }
}

__global__ void k_collect_pending(const SysState* state, uint64_t batch, int* active, int* count) {
    uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (s < batch && state[s].accepted < 0 && state[s].status == 0) {
        int pos = atomicAdd(count, 1);
        active[pos] = static_cast<int>(s);
    }
}

// systems that never accepted but skipped attempts: need the full protocol rerun
__global__ void k_collect_exhausted(const SysState* state, uint64_t batch, int* active, int* count) {
    uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (s < batch && state[s].accepted < 0 && state[s].skipped > 0) {
        int pos = atomicAdd(count, 1);
        active[pos] = static_cast<int>(s);
    }
}

__global__ void k_gather_sids(const uint64_t* sids, const int* active, int n, uint64_t* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        out[i] = sids[active[i]];
}

} // namespace

// Returns RL_OK or RL_PIVOT_BREAKDOWN (some system broke down on every attempt).
rl_status batched_circ64(uint64_t batch, const double* dA, const double* dB, int refine, uint64_t seed,
                         const uint64_t* d_sids, double* dX, rl_precond_report* d_rep) {
    cudaStream_t st = stream();
    constexpr size_t kDynSmem = 2 * N * P * sizeof(double);
    static bool attr[16] = {};
    if (!attr[ctx().device & 15]) {
        RL_CUDA(cudaFuncSetAttribute(k_batched_circ64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kDynSmem)));
        attr[ctx().device & 15] = true;
    }
    SysState* state = ws<SysState>(WS_BATCH, batch);
    double* signs = ws<double>(WS_TMP1, batch * N);
    int* active = ws<int>(WS_TMP2, batch + 4);
    int* counter = active + batch;
    uint64_t* sids_act = ws<uint64_t>(WS_SMALL, batch);
    int h_count = 0;
    auto run_protocol = [&](int prescreen, int nact, bool first) {
        for (int attempt = 0; attempt < 8 && nact > 0; ++attempt) {
            const uint64_t* sid_src = d_sids;
            if (!first || attempt > 0) {
                k_gather_sids<<<cdiv(nact, 256), 256, 0, st>>>(d_sids, active, nact, sids_act);
                RL_LAUNCHED();
                sid_src = sids_act;
            }
            rng_sign_vectors_batched(seed, sid_src, 7919ULL * attempt, 0x5000000000000000ULL, nact, N,
                                     signs);
            RL_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
            const int* act = (first && attempt == 0) ? nullptr : active;
            k_batched_circ64<<<nact, THREADS, kDynSmem, st>>>(dA, dB, signs, act, nact, attempt, refine,
                                                       prescreen, attempt == 0 ? 1 : 0, dX, d_rep,
                                                       state, counter);
            RL_LAUNCHED();
            RL_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
            k_collect_pending<<<cdiv(batch, 256), 256, 0, st>>>(state, batch, active, counter);
            RL_LAUNCHED();
            RL_CUDA(cudaMemcpyAsync(&h_count, counter, sizeof(int), cudaMemcpyDeviceToHost, st));
            RL_CUDA(cudaStreamSynchronize(st));
            nact = (attempt < 7) ? h_count : 0;
            first = false;
        }
    };
    run_protocol(1, static_cast<int>(batch), true);
    // exhausted systems with pre-screened attempts: rerun the exact protocol
    RL_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
    k_collect_exhausted<<<cdiv(batch, 256), 256, 0, st>>>(state, batch, active, counter);
    RL_LAUNCHED();
    RL_CUDA(cudaMemcpyAsync(&h_count, counter, sizeof(int), cudaMemcpyDeviceToHost, st));
    RL_CUDA(cudaStreamSynchronize(st));
    if (h_count > 0)
        run_protocol(0, h_count, false);
    // any system still with status != 0?
    std::vector<SysState> hs(batch);
    RL_CUDA(cudaMemcpyAsync(hs.data(), state, batch * sizeof(SysState), cudaMemcpyDeviceToHost, st));
    RL_CUDA(cudaStreamSynchronize(st));
    for (auto& s : hs)
        if (s.status != 0)
            return RL_PIVOT_BREAKDOWN;
    return RL_OK;
}

} // namespace rl

// K3/K4/K5: blocked Gaussian elimination with no pivoting + multi-RHS solves.
//
// Reference: genp::genp_factor (proj/src/genp.cpp:11-41, unblocked right-looking,
// no interchange, |pivot| telemetry, PivotBreakdown when |p| < floor, multiplier 0
// when p == 0), genp::block_ge (genp.cpp:43-104, the same L/U through pivot blocks,
// L21 = A21 U11^-1, U12 = L11^-1 A12, Schur update), genp::genp_solve
// (genp.cpp:106-124, forward unit-L then backward U).
//
// B200 design (n = 8192, block 128 -> 64 steps):
//   k_diag_lu   one CTA factors the 128x128 pivot block in shared memory (the
//               reference's scalar loop order: m = w(i,k)/p, w(i,j) -= m w(k,j)),
//               records |pivots|, and inverts L11 and U11 in place (Gauss-Jordan
//               on the triangles), so both TRSMs become DMMA GEMMs.
//   TRSM        L21 = A21 U11^-1 and U12 = L11^-1 A12 as GEMMs (K = 128).
//   Schur       A22 -= L21 U12, the (n-o)^2 x 128 DMMA GEMM that carries ~2n^3/3.
// Without pivoting the panel is embarrassingly parallel: there is no tall
// sequential panel factorisation on the critical path.
#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int NB = 128;        // block size (config 3's "Block size 128")
constexpr int DIAG_THREADS = 1024;

// One CTA per diagonal block.  mode 1: factor the bs x bs block at (o, o) in place
// (reference loop order, genp.cpp:20-33), write |pivots|, flag breakdown; then (both
// modes) invert L11 (unit lower) and U11 in place in shared memory and store them to
// aux as [Linv NB x NB][Uinv NB x NB].  mode 0: the block is already factored; CTA b
// handles the diagonal block at o = b*NB (all blocks of a packed LU at once).
__global__ void __launch_bounds__(DIAG_THREADS) k_diag_lu(double* a, uint64_t lda, uint64_t n,
                                                          uint64_t o_first, double floor,
                                                          double* pivots,
                                                          unsigned long long* breakdown,
                                                          double* aux, int mode) {
    extern __shared__ double w[]; // NB x (NB+1)
    __shared__ double col[NB];
    constexpr int P = NB + 1;
    const int tid = threadIdx.x;
    const uint64_t o = o_first + static_cast<uint64_t>(blockIdx.x) * NB;
    const int bs = static_cast<int>((n - o) < NB ? (n - o) : NB);
    double* ablk = a + o * lda + o;
    for (int e = tid; e < bs * bs; e += DIAG_THREADS) {
        int i = e / bs, j = e % bs;
        w[i * P + j] = ablk[static_cast<uint64_t>(i) * lda + j];
    }
    __syncthreads();
    if (mode == 1) {
        for (int k = 0; k < bs; ++k) {
            const double p = w[k * P + k];
            if (tid == 0) {
                pivots[o + k] = fabs(p);
                if (fabs(p) < floor)
                    atomicMin(breakdown, static_cast<unsigned long long>(o + k));
            }
            // multipliers m = w(i,k)/p, 0 when p == 0 (genp.cpp:26-28)
            for (int i = k + 1 + tid; i < bs; i += DIAG_THREADS)
                w[i * P + k] = (p == 0.0) ? 0.0 : w[i * P + k] / p;
            __syncthreads();
            const int rem = bs - k - 1;
            for (int e = tid; e < rem * rem; e += DIAG_THREADS) {
                int i = k + 1 + e / rem, j = k + 1 + e % rem;
                double m = w[i * P + k];
                if (m != 0.0)
                    w[i * P + j] -= m * w[k * P + j];
            }
            __syncthreads();
        }
        for (int e = tid; e < bs * bs; e += DIAG_THREADS) {
            int i = e / bs, j = e % bs;
            ablk[static_cast<uint64_t>(i) * lda + j] = w[i * P + j];
        }
    }
    if (!aux)
        return;
    double* linv = aux + (o / NB) * 2 * NB * NB;
    double* uinv = linv + NB * NB;
    // inv(L) in place (strict lower; unit diagonal implicit), steps k ascending:
    //   Y[i][k] = -L[i][k],  Y[i][j] -= L[i][k] Y[k][j]  (i > k, j < k)
    for (int k = 0; k < bs; ++k) {
        __syncthreads();
        for (int i = k + 1 + tid; i < bs; i += DIAG_THREADS)
            col[i] = w[i * P + k];
        __syncthreads();
        const int rows = bs - k - 1;
        for (int e = tid; e < rows * (k + 1); e += DIAG_THREADS) {
            int i = k + 1 + e / (k + 1), j = e % (k + 1);
            double l = col[i];
            w[i * P + j] = (j == k) ? -l : w[i * P + j] - l * w[k * P + j];
        }
    }
    // inv(U) in place (upper incl. diagonal), steps k descending:
    //   X[k][k] = 1/U[k][k], X[k][j] *= X[k][k] (j > k); X[i][k] = -U[i][k] X[k][k],
    //   X[i][j] -= U[i][k] X[k][j]  (i < k, j > k).  1/0 := 0 (genp.cpp:27 convention).
    for (int k = bs - 1; k >= 0; --k) {
        __syncthreads();
        const double d = w[k * P + k];
        const double r = (d == 0.0) ? 0.0 : 1.0 / d;
        for (int i = tid; i < k; i += DIAG_THREADS)
            col[i] = w[i * P + k];
        __syncthreads();
        for (int j = k + tid; j < bs; j += DIAG_THREADS)
            w[k * P + j] = (j == k) ? r : w[k * P + j] * r;
        __syncthreads();
        const int cols = bs - k;
        for (int e = tid; e < k * cols; e += DIAG_THREADS) {
            int i = e / cols, j = k + e % cols;
            double u = col[i];
            w[i * P + j] = (j == k) ? -u * w[k * P + k] : w[i * P + j] - u * w[k * P + j];
        }
    }
    __syncthreads();
    for (int e = tid; e < NB * NB; e += DIAG_THREADS) {
        int i = e / NB, j = e % NB;
        bool in = i < bs && j < bs;
        linv[e] = !in ? 0.0 : (i == j ? 1.0 : (i > j ? w[i * P + j] : 0.0));
        uinv[e] = !in ? 0.0 : (j >= i ? w[i * P + j] : 0.0);
    }
}


// ---------------------------------------------------------------- TRSM ----
// Substitution-based triangular solves on 128-wide panels (backward stable, like the
// reference's block_ge L21/U12 loops, genp.cpp:77-92).  The triangle sits in shared
// memory; every warp owns independent rows (right solve) or columns (left solve) in
// registers, so after the initial load there is no CTA-wide synchronisation: the
// sequential chain is per warp, broadcasts are __shfl_sync.
constexpr int TR_WARPS = 16;            // 512 threads
constexpr int TR_TILE = 64;             // rows (right) or columns (left) per CTA
constexpr int TR_PER_WARP = TR_TILE / TR_WARPS; // 4
constexpr int TP = NB + 1;              // smem pitch of the triangle

// Right solve with U11 (upper, non-unit): rows x of A21 satisfy x U11 = a,
//   x_j = (a_j - sum_{l<j} x_l U_lj) / U_jj      (L21 = A21 U11^-1)
// Left solve with L11 (unit lower): columns y of A12 satisfy L11 y = a,
//   y_i = a_i - sum_{l<i} L_il y_l              (U12 = L11^-1 A12)
// One launch does both: CTAs [0, nrb) take 64-row blocks of A21, the rest take
// 64-column blocks of A12.  rest = n - o - bs rows/cols, bs = NB here.
__global__ void __launch_bounds__(TR_WARPS * 32, 1) k_panel_trsm(double* a, uint64_t lda, uint64_t o,
                                                                 uint64_t rest, int nrb) {
    extern __shared__ double smt[];
    double* T = smt;                 // NB x TP triangle
    double* tile = smt + NB * TP;    // right: 64 x TP ; left: NB x (64+1)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool right = static_cast<int>(blockIdx.x) < nrb;
    const double* diag = a + o * lda + o;
    for (int e = tid; e < NB * NB; e += blockDim.x) {
        int i = e / NB, j = e % NB;
        bool want = right ? (j >= i) : (i > j);
        T[i * TP + j] = want ? diag[static_cast<uint64_t>(i) * lda + j] : 0.0;
    }
    if (right) {
        const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * TR_TILE;
        const int nr = static_cast<int>(rest - r0 < TR_TILE ? rest - r0 : TR_TILE);
        double* src = a + (o + NB + r0) * lda + o;
        for (int e = tid; e < nr * NB; e += blockDim.x) {
            int i = e / NB, j = e % NB;
            tile[i * TP + j] = src[static_cast<uint64_t>(i) * lda + j];
        }
        __syncthreads();
        // warp owns rows warp*4 .. +3 ; lane owns columns lane + 32c
        double w[TR_PER_WARP][4];
#pragma unroll
        for (int r = 0; r < TR_PER_WARP; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                int row = warp * TR_PER_WARP + r;
                w[r][c] = row < nr ? tile[row * TP + lane + 32 * c] : 0.0;
            }
        for (int j = 0; j < NB; ++j) {
            const double d = T[j * TP + j];
            const double rcp = (d == 0.0) ? 0.0 : 1.0 / d; // multiplier 0 when p == 0 (genp.cpp:27)
            const int cj = j >> 5, lj = j & 31;
            double x[TR_PER_WARP];
#pragma unroll
            for (int r = 0; r < TR_PER_WARP; ++r) {
                double mine = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c == cj)
                        mine = w[r][c];
                x[r] = __shfl_sync(0xffffffffu, mine, lj) * rcp;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int col = lane + 32 * c;
                if (col == j) {
#pragma unroll
                    for (int r = 0; r < TR_PER_WARP; ++r)
                        w[r][c] = x[r];
                } else if (col > j) {
                    const double u = T[j * TP + col];
#pragma unroll
                    for (int r = 0; r < TR_PER_WARP; ++r)
                        if (x[r] != 0.0)
                            w[r][c] = fma(-x[r], u, w[r][c]);
                }
            }
        }
        double* dst = a + (o + NB + r0) * lda + o;
#pragma unroll
        for (int r = 0; r < TR_PER_WARP; ++r) {
            int row = warp * TR_PER_WARP + r;
            if (row < nr)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    dst[static_cast<uint64_t>(row) * lda + lane + 32 * c] = w[r][c];
        }
    } else {
        constexpr int CP = TR_TILE + 1;
        const uint64_t c0 = static_cast<uint64_t>(blockIdx.x - nrb) * TR_TILE;
        const int nc = static_cast<int>(rest - c0 < TR_TILE ? rest - c0 : TR_TILE);
        double* src = a + o * lda + o + NB + c0;
        for (int e = tid; e < NB * TR_TILE; e += blockDim.x) {
            int i = e / TR_TILE, j = e % TR_TILE;
            tile[i * CP + j] = j < nc ? src[static_cast<uint64_t>(i) * lda + j] : 0.0;
        }
        __syncthreads();
        // warp owns columns warp*4 .. +3 ; lane owns rows lane + 32c
        double w[TR_PER_WARP][4];
#pragma unroll
        for (int q = 0; q < TR_PER_WARP; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                w[q][c] = tile[(lane + 32 * c) * CP + warp * TR_PER_WARP + q];
        for (int i = 0; i < NB; ++i) {
            const int ci = i >> 5, li = i & 31;
            double y[TR_PER_WARP];
#pragma unroll
            for (int q = 0; q < TR_PER_WARP; ++q) {
                double mine = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c == ci)
                        mine = w[q][c];
                y[q] = __shfl_sync(0xffffffffu, mine, li);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int row = lane + 32 * c;
                if (row > i) {
                    const double l = T[row * TP + i];
                    if (l != 0.0)
#pragma unroll
                        for (int q = 0; q < TR_PER_WARP; ++q)
                            w[q][c] = fma(-l, y[q], w[q][c]);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < TR_PER_WARP; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                tile[(lane + 32 * c) * CP + warp * TR_PER_WARP + q] = w[q][c];
        __syncthreads();
        for (int e = tid; e < NB * TR_TILE; e += blockDim.x) {
            int i = e / TR_TILE, j = e % TR_TILE;
            if (j < nc)
                src[static_cast<uint64_t>(i) * lda + j] = tile[i * CP + j];
        }
    }
}

// Solve with one diagonal block of a packed LU on a bs x nrhs panel of B (ld ldb):
// lower = unit-lower forward substitution, else upper backward substitution with
// division by U_ii (genp.cpp:110-122).  One CTA; warps own RHS columns.
__global__ void __launch_bounds__(TR_WARPS * 32, 1) k_block_solve(const double* lu, uint64_t lda, uint64_t o,
                                                                  int bs, double* b, uint64_t ldb,
                                                                  uint64_t nrhs, int lower) {
    extern __shared__ double smt[];
    double* T = smt; // bs x TP
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* diag = lu + o * lda + o;
    for (int e = tid; e < bs * bs; e += blockDim.x) {
        int i = e / bs, j = e % bs;
        T[i * TP + j] = diag[static_cast<uint64_t>(i) * lda + j];
    }
    __syncthreads();
    for (uint64_t col = warp; col < nrhs; col += TR_WARPS) {
        double w[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int row = lane + 32 * c;
            w[c] = row < bs ? b[(o + row) * ldb + col] : 0.0;
        }
        if (lower) {
            for (int i = 0; i < bs; ++i) {
                double mine = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c == (i >> 5))
                        mine = w[c];
                const double yi = __shfl_sync(0xffffffffu, mine, i & 31);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    int row = lane + 32 * c;
                    if (row > i && row < bs)
                        w[c] = fma(-T[row * TP + i], yi, w[c]);
                }
            }
        } else {
            for (int i = bs - 1; i >= 0; --i) {
                double mine = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c == (i >> 5))
                        mine = w[c];
                const double xi = __shfl_sync(0xffffffffu, mine, i & 31) / T[i * TP + i];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    int row = lane + 32 * c;
                    if (row == i)
                        w[c] = xi;
                    else if (row < i)
                        w[c] = fma(-T[row * TP + i], xi, w[c]);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int row = lane + 32 * c;
            if (row < bs)
                b[(o + row) * ldb + col] = w[c];
        }
    }
}

__global__ void k_copy2d(uint64_t rows, uint64_t cols, const double* src, uint64_t lds, double* dst,
                         uint64_t ldd) {
    uint64_t total = rows * cols;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = e / cols, j = e % cols;
        dst[i * ldd + j] = src[i * lds + j];
    }
}

__global__ void k_axpy(uint64_t count, double alpha, const double* x, double* y) {
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[e] = fma(alpha, x[e], y[e]);
}

__global__ void k_transpose(uint64_t m, uint64_t n, const double* a, uint64_t lda, double* t,
                            uint64_t ldt) {
    __shared__ double tile[32][33];
    uint64_t bx = blockIdx.x * 32ULL, by = blockIdx.y * 32ULL;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        uint64_t i = by + r, j = bx + threadIdx.x;
        if (i < m && j < n)
            tile[r][threadIdx.x] = a[i * lda + j];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        uint64_t j = bx + r, i = by + threadIdx.x;
        if (i < m && j < n)
            t[j * ldt + i] = tile[threadIdx.x][r];
    }
}

// per-column residual: out[j] = ||R[:,j]|| / ||B[:,j]|| with R = A X - B precomputed
__global__ void k_colnorm_ratio(uint64_t n, uint64_t nrhs, const double* r, const double* b,
                                double* out) {
    const uint64_t j = blockIdx.x;
    double num = 0.0, den = 0.0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double d = r[i * nrhs + j], bb = b[i * nrhs + j];
        num += d * d;
        den += bb * bb;
    }
    __shared__ double sn[32], sd[32];
    for (int off = 16; off > 0; off >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, off);
        den += __shfl_xor_sync(0xffffffffu, den, off);
    }
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        sn[wid] = num;
        sd[wid] = den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, c = 0.0;
        for (int k = 0; k < static_cast<int>(blockDim.x / 32); ++k) {
            a += sn[k];
            c += sd[k];
        }
        out[j] = sqrt(a) / sqrt(c);
    }
}

size_t diag_smem() { return static_cast<size_t>(NB) * (NB + 1) * sizeof(double); }

void prep_diag_attr() {
    static bool done[16] = {};
    int dev = ctx().device & 15;
    if (!done[dev]) {
        RL_CUDA(cudaFuncSetAttribute(k_diag_lu, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(diag_smem())));
        done[dev] = true;
    }
}

} // namespace

void copy2d_dev(uint64_t rows, uint64_t cols, const double* src, uint64_t lds, double* dst, uint64_t ldd) {
    if (rows == 0 || cols == 0)
        return;
    uint64_t total = rows * cols;
    unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ULL * 16));
    k_copy2d<<<blocks, 256, 0, stream()>>>(rows, cols, src, lds, dst, ldd);
    RL_LAUNCHED();
}

void axpy_dev(uint64_t count, double alpha, const double* x, double* y) {
    if (count == 0)
        return;
    unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((count + 255) / 256, 148ULL * 16));
    k_axpy<<<blocks, 256, 0, stream()>>>(count, alpha, x, y);
    RL_LAUNCHED();
}

void transpose_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda, double* t, uint64_t ldt) {
    dim3 grid(cdiv(n, 32), cdiv(m, 32));
    k_transpose<<<grid, dim3(32, 8), 0, stream()>>>(m, n, a, lda, t, ldt);
    RL_LAUNCHED();
}

size_t trsm_smem() { return (static_cast<size_t>(NB) * TP + static_cast<size_t>(NB) * (TR_TILE + 1)) * sizeof(double); }

void prep_trsm_attr() {
    static bool done[16] = {};
    int dev = ctx().device & 15;
    if (!done[dev]) {
        RL_CUDA(cudaFuncSetAttribute(k_panel_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(trsm_smem())));
        RL_CUDA(cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(NB * TP * sizeof(double))));
        done[dev] = true;
    }
}

// Blocked right-looking GENP in place (packed LU).  aux is unused (kept for the
// signature); pivots / first breakdown step go to d_pivots / d_breakdown.
void genp_factor_blocked(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                         unsigned long long* d_breakdown, double* aux) {
    (void)aux;
    prep_diag_attr();
    prep_trsm_attr();
    cudaStream_t st = stream();
    for (uint64_t o = 0; o < n; o += NB) {
        const int bs = static_cast<int>(std::min<uint64_t>(NB, n - o));
        k_diag_lu<<<1, DIAG_THREADS, diag_smem(), st>>>(a, lda, n, o, pivot_floor, d_pivots, d_breakdown,
                                                        nullptr, 1);
        RL_LAUNCHED();
        const uint64_t rest = n - o - bs;
        if (rest == 0)
            break;
        // L21 = A21 U11^-1 and U12 = L11^-1 A12 by substitution, in place (bs == NB here)
        const int nrb = static_cast<int>((rest + TR_TILE - 1) / TR_TILE);
        k_panel_trsm<<<2 * nrb, TR_WARPS * 32, trsm_smem(), st>>>(a, lda, o, rest, nrb);
        RL_LAUNCHED();
        // Schur: A22 -= L21 U12  (the DMMA GEMM carrying ~2n^3/3)
        gemm(false, false, rest, rest, bs, -1.0, a + (o + bs) * lda + o, lda, a + o * lda + o + bs, lda, 1.0,
             a + (o + bs) * lda + o + bs, lda);
    }
}

void genp_factor_dev(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                     int64_t* d_breakdown) {
    RL_CUDA(cudaMemsetAsync(d_breakdown, 0xff, sizeof(int64_t), stream())); // -1 == none
    genp_factor_blocked(n, a, lda, pivot_floor, d_pivots,
                        reinterpret_cast<unsigned long long*>(d_breakdown), nullptr);
}

// Kept for the C-ABI signature (block inverses are no longer needed by the solves).
void genp_block_inverses(uint64_t n, const double* lu, uint64_t lda, double* aux) {
    (void)n;
    (void)lu;
    (void)lda;
    (void)aux;
}

// Forward (unit L) then backward (U) substitution, blocked, nrhs columns; b (n x nrhs,
// ldb) is overwritten by the solution (genp.cpp:106-124).
void genp_solve_blocked(uint64_t n, uint64_t nrhs, const double* lu, uint64_t lda, const double* aux,
                        double* b, uint64_t ldb) {
    (void)aux;
    prep_trsm_attr();
    cudaStream_t st = stream();
    const size_t sm = NB * TP * sizeof(double);
    for (uint64_t o = 0; o < n; o += NB) {
        const int bs = static_cast<int>(std::min<uint64_t>(NB, n - o));
        k_block_solve<<<1, TR_WARPS * 32, sm, st>>>(lu, lda, o, bs, b, ldb, nrhs, 1);
        RL_LAUNCHED();
        const uint64_t rest = n - o - bs;
        if (rest)
            gemm(false, false, rest, nrhs, bs, -1.0, lu + (o + bs) * lda + o, lda, b + o * ldb, ldb, 1.0,
                 b + (o + bs) * ldb, ldb);
    }
    const uint64_t nblk = (n + NB - 1) / NB;
    for (uint64_t bi = nblk; bi-- > 0;) {
        const uint64_t o = bi * NB;
        const int bs = static_cast<int>(std::min<uint64_t>(NB, n - o));
        k_block_solve<<<1, TR_WARPS * 32, sm, st>>>(lu, lda, o, bs, b, ldb, nrhs, 0);
        RL_LAUNCHED();
        if (o)
            gemm(false, false, o, nrhs, bs, -1.0, lu + o, lda, b + o * ldb, ldb, 1.0, b, ldb);
    }
}

void genp_solve_dev(uint64_t n, uint64_t nrhs, const double* lu, uint64_t lda, double* b, uint64_t ldb) {
    genp_solve_blocked(n, nrhs, lu, lda, nullptr, b, ldb);
}

// r_j = ||A x_j - b_j|| / ||b_j||  (genp.cpp:146-155), one value per column
void residuals_dev(uint64_t n, uint64_t nrhs, const double* a, const double* x, const double* b,
                   double* d_tmp, double* d_out) {
    copy2d_dev(n, nrhs, b, nrhs, d_tmp, nrhs);
    gemm(false, false, n, nrhs, n, 1.0, a, n, x, nrhs, -1.0, d_tmp, nrhs);
    k_colnorm_ratio<<<static_cast<unsigned>(nrhs), 256, 0, stream()>>>(n, nrhs, d_tmp, b, d_out);
    RL_LAUNCHED();
}

} // namespace rl

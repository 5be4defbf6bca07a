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
#include "panel.cuh"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int NB = 128;        // block size (config 3's "Block size 128")

// ------------------------------------------------------------ panel kernels ----
// All three use the two-level scheme of panel.cuh: 16-wide sub-panels, per-thread
// 16-step substitutions out of registers, DMMA updates between shared-memory tiles.
using panel::PT;
using panel::SB;
constexpr int PK_THREADS = 256; // 8 warps
constexpr int PK_WARPS = PK_THREADS / 32;

// Diagonal-block LU of the bs x bs block at (o, o), in place (genp.cpp:20-33 order
// within each 16-column sub-panel; the sub-panel's effect on the rest is a DMMA update).
// Rows/columns beyond bs are padded with the identity so every tile is 128 x 128.
//   per sub-panel c0:  (1) warp 0 factors the 16x16 diagonal sub-block (lanes own rows,
//   pivot rows broadcast through shared memory, __syncwarp only); (2) every row below
//   solves its 16 L entries against that U (independent rows, no sync); (3) every column
//   right of it solves its 16 U entries against that unit L; (4) DMMA trailing update.
// |pivots| and the first step with |p| < floor are recorded; 1/p := 0 when p == 0 gives
// the reference's multiplier 0 (genp.cpp:27).
__global__ void __launch_bounds__(PK_THREADS, 1) k_diag_lu(double* a, uint64_t lda, uint64_t n, uint64_t o,
                                                           double floor, double* pivots,
                                                           unsigned long long* breakdown) {
    extern __shared__ double W[]; // NB x PT
    __shared__ double rcp[NB];
    __shared__ double prow[SB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bs = static_cast<int>((n - o) < NB ? (n - o) : NB);
    double* blk = a + o * lda + o;
    panel::load_tile<NB, NB, PK_THREADS>(W, PT, blk, lda, bs, bs, [](int, int) { return true; },
                                         [](int i, int j) { return i == j ? 1.0 : 0.0; });
    __syncthreads();
    for (int c0 = 0; c0 < NB; c0 += SB) {
        // (1) 16x16 diagonal sub-block, warp 0, lanes 0..15 own its rows
        if (warp == 0) {
            double p[SB];
            const int r = c0 + (lane & (SB - 1));
#pragma unroll
            for (int l = 0; l < SB; ++l)
                p[l] = W[r * PT + c0 + l];
#pragma unroll
            for (int kk = 0; kk < SB; ++kk) {
                if (lane == kk) {
#pragma unroll
                    for (int l = 0; l < SB; ++l)
                        prow[l] = p[l];
                }
                __syncwarp();
                const double piv = prow[kk];
                const double inv = (piv == 0.0) ? 0.0 : 1.0 / piv;
                if (lane == 0) {
                    const int k = c0 + kk;
                    if (k < bs) {
                        pivots[o + k] = fabs(piv);
                        if (fabs(piv) < floor)
                            atomicMin(breakdown, static_cast<unsigned long long>(o + k));
                    }
                    rcp[k] = inv;
                }
                if (lane < SB && lane > kk) {
                    const double m = p[kk] * inv;
                    p[kk] = m;
                    if (m != 0.0)
#pragma unroll
                        for (int l = kk + 1; l < SB; ++l)
                            p[l] = fma(-m, prow[l], p[l]);
                }
                __syncwarp();
            }
            if (lane < SB)
#pragma unroll
                for (int l = 0; l < SB; ++l)
                    W[r * PT + c0 + l] = p[l];
        }
        __syncthreads();
        const int rest = NB - c0 - SB;
        if (rest == 0)
            break;
        // (2) rows below: l_r U_sub = w_r   (x_j = (w_j - sum_{l<j} x_l U_lj) / U_jj)
        for (int t = tid; t < rest; t += PK_THREADS) {
            const int r = c0 + SB + t;
            double x[SB];
#pragma unroll
            for (int l = 0; l < SB; ++l)
                x[l] = W[r * PT + c0 + l];
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                const double xj = x[j] * rcp[c0 + j];
                x[j] = xj;
                if (xj != 0.0)
#pragma unroll
                    for (int l = j + 1; l < SB; ++l)
                        x[l] = fma(-xj, W[(c0 + j) * PT + c0 + l], x[l]);
            }
#pragma unroll
            for (int l = 0; l < SB; ++l)
                W[r * PT + c0 + l] = x[l];
        }
        // (3) columns right: L_sub y = w  (unit lower)
        for (int t = tid; t < rest; t += PK_THREADS) {
            const int c = c0 + SB + t;
            double y[SB];
#pragma unroll
            for (int i = 0; i < SB; ++i)
                y[i] = W[(c0 + i) * PT + c];
#pragma unroll
            for (int i = 1; i < SB; ++i)
#pragma unroll
                for (int l = 0; l < i; ++l)
                    y[i] = fma(-W[(c0 + i) * PT + c0 + l], y[l], y[i]);
#pragma unroll
            for (int i = 1; i < SB; ++i)
                W[(c0 + i) * PT + c] = y[i];
        }
        __syncthreads();
        // (4) trailing 128-c0-16 square: W22 -= L21 U12
        panel::smem_update16(W + (c0 + SB) * PT + c0 + SB, PT, W + (c0 + SB) * PT + c0, PT, W + c0 * PT + c0 + SB,
                             PT, rest, rest, warp, PK_WARPS, lane);
        __syncthreads();
    }
    panel::store_tile<NB, NB, PK_THREADS>(blk, lda, W, PT, bs, bs);
}

// Panel TRSMs of block step o (genp.cpp:77-92), in place, one launch:
//   CTAs [0, nrb):      64-row tiles of A21 <- A21 U11^-1   (x U11 = a)
//   CTAs [nrb, 2 nrb2): 64-column tiles of A12 <- L11^-1 A12 (L11 y = a, unit lower)
// Each sub-panel: per-thread 16-step substitution, then a DMMA update of the remaining
// columns (right) / rows (left) of the tile.
constexpr int TR_TILE = 64;
__global__ void __launch_bounds__(PK_THREADS, 1) k_panel_trsm(double* a, uint64_t lda, uint64_t o, uint64_t rest,
                                                              int nrb) {
    extern __shared__ double smt[];
    double* T = smt;            // NB x PT triangle
    double* X = smt + NB * PT;  // right: 64 x PT ; left: NB x (64 + 4)
    __shared__ double rcp[NB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool right = static_cast<int>(blockIdx.x) < nrb;
    const double* diag = a + o * lda + o;
    if (right)
        panel::load_tile<NB, NB, PK_THREADS>(T, PT, diag, lda, NB, NB, [](int i, int j) { return j >= i; },
                                             [](int, int) { return 0.0; });
    else
        panel::load_tile<NB, NB, PK_THREADS>(T, PT, diag, lda, NB, NB, [](int i, int j) { return i > j; },
                                             [](int, int) { return 0.0; });
    if (right) {
        const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * TR_TILE;
        const int nr = static_cast<int>(rest - r0 < TR_TILE ? rest - r0 : TR_TILE);
        double* src = a + (o + NB + r0) * lda + o;
        panel::load_tile<TR_TILE, NB, PK_THREADS>(X, PT, src, lda, nr, NB, [](int, int) { return true; },
                                                  [](int, int) { return 0.0; });
        __syncthreads();
        for (int j = tid; j < NB; j += PK_THREADS) {
            const double d = T[j * PT + j];
            rcp[j] = (d == 0.0) ? 0.0 : 1.0 / d;
        }
        __syncthreads();
        for (int c0 = 0; c0 < NB; c0 += SB) {
            for (int r = tid; r < TR_TILE; r += PK_THREADS) {
                double x[SB];
#pragma unroll
                for (int l = 0; l < SB; ++l)
                    x[l] = X[r * PT + c0 + l];
#pragma unroll
                for (int j = 0; j < SB; ++j) {
                    const double xj = x[j] * rcp[c0 + j];
                    x[j] = xj;
                    if (xj != 0.0)
#pragma unroll
                        for (int l = j + 1; l < SB; ++l)
                            x[l] = fma(-xj, T[(c0 + j) * PT + c0 + l], x[l]);
                }
#pragma unroll
                for (int l = 0; l < SB; ++l)
                    X[r * PT + c0 + l] = x[l];
            }
            __syncthreads();
            if (c0 + SB < NB)
                panel::smem_update16(X + c0 + SB, PT, X + c0, PT, T + c0 * PT + c0 + SB, PT, TR_TILE,
                                     NB - c0 - SB, warp, PK_WARPS, lane);
            __syncthreads();
        }
        panel::store_tile<TR_TILE, NB, PK_THREADS>(src, lda, X, PT, nr, NB);
    } else {
        constexpr int XP = TR_TILE + 4;
        const uint64_t c0g = static_cast<uint64_t>(blockIdx.x - nrb) * TR_TILE;
        const int nc = static_cast<int>(rest - c0g < TR_TILE ? rest - c0g : TR_TILE);
        double* src = a + o * lda + o + NB + c0g;
        panel::load_tile<NB, TR_TILE, PK_THREADS>(X, XP, src, lda, NB, nc, [](int, int) { return true; },
                                                  [](int, int) { return 0.0; });
        __syncthreads();
        for (int c0 = 0; c0 < NB; c0 += SB) {
            for (int c = tid; c < TR_TILE; c += PK_THREADS) {
                double y[SB];
#pragma unroll
                for (int i = 0; i < SB; ++i)
                    y[i] = X[(c0 + i) * XP + c];
#pragma unroll
                for (int i = 1; i < SB; ++i)
#pragma unroll
                    for (int l = 0; l < i; ++l)
                        y[i] = fma(-T[(c0 + i) * PT + c0 + l], y[l], y[i]);
#pragma unroll
                for (int i = 1; i < SB; ++i)
                    X[(c0 + i) * XP + c] = y[i];
            }
            __syncthreads();
            if (c0 + SB < NB)
                panel::smem_update16(X + (c0 + SB) * XP, XP, T + (c0 + SB) * PT + c0, PT, X + c0 * XP, XP,
                                     NB - c0 - SB, TR_TILE, warp, PK_WARPS, lane);
            __syncthreads();
        }
        panel::store_tile<NB, TR_TILE, PK_THREADS>(src, lda, X, XP, NB, nc);
    }
}

// Diagonal-panel substitution of the multi-RHS solves (genp.cpp:106-124) on a bs x nrhs
// slice of B: lower = unit-lower forward, upper = backward with x_i = s * (1/U_ii)
// (within 1 ulp of the reference's division).  Blocks beyond bs are padded with the
// identity; off-diagonal updates outside the 128-block are DMMA GEMMs (host loop).
constexpr int SV_MAXRHS = 32;
constexpr int SV_ROWS = 64;
constexpr int SVP = SV_MAXRHS + 4;
__global__ void __launch_bounds__(PK_THREADS, 1) k_block_solve(const double* __restrict__ lu, uint64_t lda,
                                                               uint64_t n, uint64_t o, double* __restrict__ b,
                                                               uint64_t ldb, int nrhs, int lower) {
    extern __shared__ double T[]; // NB x PT, then Bs NB x SVP
    double* Bs = T + NB * PT;
    __shared__ double rcp[NB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bs = static_cast<int>((n - o) < NB ? (n - o) : NB);
    const double* diag = lu + o * lda + o;
    if (lower)
        panel::load_tile<NB, NB, PK_THREADS>(T, PT, diag, lda, bs, bs, [](int i, int j) { return i > j; },
                                             [](int, int) { return 0.0; });
    else
        panel::load_tile<NB, NB, PK_THREADS>(T, PT, diag, lda, bs, bs, [](int i, int j) { return j >= i; },
                                             [](int i, int j) { return i == j ? 1.0 : 0.0; });
    const int n8 = (nrhs + 7) & ~7;
    panel::load_tile<NB, SV_MAXRHS, PK_THREADS>(Bs, SVP, b + o * ldb, ldb, bs, nrhs, [](int, int) { return true; },
                                                [](int, int) { return 0.0; });
    __syncthreads();
    if (!lower)
        for (int i = tid; i < NB; i += PK_THREADS)
            rcp[i] = 1.0 / T[i * PT + i];
    __syncthreads();
    if (lower) {
        for (int c0 = 0; c0 < NB; c0 += SB) {
            for (int c = tid; c < nrhs; c += PK_THREADS) {
                double y[SB];
#pragma unroll
                for (int i = 0; i < SB; ++i)
                    y[i] = Bs[(c0 + i) * SVP + c];
#pragma unroll
                for (int i = 1; i < SB; ++i)
#pragma unroll
                    for (int l = 0; l < i; ++l)
                        y[i] = fma(-T[(c0 + i) * PT + c0 + l], y[l], y[i]);
#pragma unroll
                for (int i = 1; i < SB; ++i)
                    Bs[(c0 + i) * SVP + c] = y[i];
            }
            __syncthreads();
            if (c0 + SB < NB)
                panel::smem_update16(Bs + (c0 + SB) * SVP, SVP, T + (c0 + SB) * PT + c0, PT, Bs + c0 * SVP, SVP,
                                     NB - c0 - SB, n8, warp, PK_WARPS, lane);
            __syncthreads();
        }
    } else {
        for (int c0 = NB - SB; c0 >= 0; c0 -= SB) {
            for (int c = tid; c < nrhs; c += PK_THREADS) {
                double y[SB];
#pragma unroll
                for (int i = 0; i < SB; ++i)
                    y[i] = Bs[(c0 + i) * SVP + c];
#pragma unroll
                for (int i = SB - 1; i >= 0; --i) {
                    const double xi = y[i] * rcp[c0 + i];
                    y[i] = xi;
#pragma unroll
                    for (int l = 0; l < i; ++l)
                        y[l] = fma(-T[(c0 + l) * PT + c0 + i], xi, y[l]);
                }
#pragma unroll
                for (int i = 0; i < SB; ++i)
                    Bs[(c0 + i) * SVP + c] = y[i];
            }
            __syncthreads();
            if (c0 > 0)
                panel::smem_update16(Bs, SVP, T + c0, PT, Bs + c0 * SVP, SVP, c0, n8, warp, PK_WARPS, lane);
            __syncthreads();
        }
    }
    panel::store_tile<NB, SV_MAXRHS, PK_THREADS>(b + o * ldb, ldb, Bs, SVP, bs, nrhs);
}

// diagonal 128-blocks of a packed LU -> contiguous [nblk][NB][NB] (ragged last block)
__global__ void k_gather_diag(const double* __restrict__ lu, uint64_t lda, uint64_t n, double* __restrict__ out) {
    const uint64_t o = static_cast<uint64_t>(blockIdx.x) * NB;
    const int bs = static_cast<int>((n - o) < NB ? (n - o) : NB);
    double* dst = out + static_cast<uint64_t>(blockIdx.x) * NB * NB;
    for (int e = threadIdx.x; e < bs * NB; e += blockDim.x) {
        const int i = e / NB, j = e % NB;
        if (j < bs)
            dst[i * NB + j] = lu[(o + i) * lda + o + j];
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

size_t trsm_smem() { return (static_cast<size_t>(NB) * PT + static_cast<size_t>(NB) * (TR_TILE + 4)) * sizeof(double); }
size_t diag_smem() { return static_cast<size_t>(NB) * PT * sizeof(double); }
size_t solve_smem() { return static_cast<size_t>(NB) * (PT + SVP) * sizeof(double); }

void prep_attrs() {
    static bool done[16] = {};
    int dev = ctx().device & 15;
    if (!done[dev]) {
        RL_CUDA(cudaFuncSetAttribute(k_panel_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(trsm_smem())));
        RL_CUDA(cudaFuncSetAttribute(k_diag_lu, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(diag_smem())));
        RL_CUDA(cudaFuncSetAttribute(k_block_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(solve_smem())));

        done[dev] = true;
    }
}

// Per-thread helper stream (high priority) and events for the panel lookahead.
struct Lookahead {
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int device = -1;
};

Lookahead& lookahead() {
    static thread_local Lookahead la;
    if (la.device != ctx().device) {
        int lo = 0, hi = 0;
        RL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        RL_CUDA(cudaStreamCreateWithPriority(&la.s2, cudaStreamNonBlocking, hi));
        for (auto& e : la.ev)
            RL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        la.device = ctx().device;
    }
    return la;
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

// Blocked right-looking GENP in place (packed LU), outer block 256 built from two 128
// steps, with one-panel lookahead:
//   main stream : Schur update of outer step k split into the next outer panel's strips
//                 (first) and the remaining trailing block (the big K = 256 DMMA GEMM)
//   panel stream: the next outer panel (2 x [diagonal LU + both TRSMs] + the strip update
//                 between them), started as soon as the strips of step k are done, so it
//                 runs under the trailing GEMM of step k.
// The regions written concurrently are disjoint.  The L and U produced are
// those of block_ge with block 128 (genp.cpp:43-104) up to rounding.  aux is unused.
void genp_factor_blocked(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                         unsigned long long* d_breakdown, double* aux) {
    (void)aux;
    prep_attrs();
    cudaStream_t s1 = stream();
    Lookahead& la = lookahead();
    cudaStream_t s2 = la.s2;
    auto at = [&](uint64_t i, uint64_t j) { return a + i * lda + j; };
    // one 128-wide step: diagonal LU + both TRSMs over everything below / right of it
    auto panel128 = [&](uint64_t o, cudaStream_t st) {
        k_diag_lu<<<1, PK_THREADS, diag_smem(), st>>>(a, lda, n, o, pivot_floor, d_pivots, d_breakdown);
        RL_LAUNCHED();
        const uint64_t rest = n - o - std::min<uint64_t>(NB, n - o);
        if (rest) {
            const int nrb = static_cast<int>((rest + TR_TILE - 1) / TR_TILE);
            k_panel_trsm<<<2 * nrb, PK_THREADS, trsm_smem(), st>>>(a, lda, o, rest, nrb);
            RL_LAUNCHED();
        }
    };
    // one outer panel of width W = 2 * NB at o (block LU with a 256 pivot block composed of two
    // 128 steps): step 1, then only the second sub-panel's strips are updated (the trailing
    // update is delayed), then step 2.  The trailing matrix is updated once with K = 256.
    auto panel256 = [&](uint64_t o, cudaStream_t st) {
        cudaStream_t keep = ctx().stream;
        ctx().stream = st; // gemm() launches on ctx().stream
        panel128(o, st);
        const uint64_t o2 = o + NB;
        if (o2 < n) {
            const uint64_t rest = n - o2, w2 = std::min<uint64_t>(NB, rest);
            gemm(false, false, rest, w2, NB, -1.0, at(o2, o), lda, at(o, o2), lda, 1.0, at(o2, o2), lda);
            if (rest > w2)
                gemm(false, false, w2, rest - w2, NB, -1.0, at(o2, o), lda, at(o, o2 + w2), lda, 1.0,
                     at(o2, o2 + w2), lda);
            panel128(o2, st);
        }
        ctx().stream = keep;
    };
    constexpr uint64_t W = 2 * NB;
    // RL_LU_TRACE=1: per outer step, time of the panel path (s2) and of the step on s1 (dev)
    static const bool trace = std::getenv("RL_LU_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
        if (!trace)
            return;
        cudaEvent_t e;
        RL_CUDA(cudaEventCreate(&e));
        RL_CUDA(cudaEventRecord(e, st));
        tev.push_back(e);
    };
    panel256(0, s1);
    for (uint64_t o = 0; o + W < n; o += W) {
        mark(s1);
        const uint64_t rest = n - o - W;                 // trailing size after this outer step
        const uint64_t w2 = std::min<uint64_t>(W, rest); // width of the next outer panel
        const double* L21 = at(o + W, o);                // rest x 256
        const double* U12 = at(o, o + W);                // 256 x rest
        // (i) next outer panel's column strip and row strip (K = 256)
        gemm(false, false, rest, w2, W, -1.0, L21, lda, U12, lda, 1.0, at(o + W, o + W), lda);
        if (rest > w2)
            gemm(false, false, w2, rest - w2, W, -1.0, L21, lda, at(o, o + W + w2), lda, 1.0,
                 at(o + W, o + W + w2), lda);
        // hand the next outer panel to the high-priority panel stream ...
        cudaEvent_t strips = la.ev[0], done = la.ev[1];
        RL_CUDA(cudaEventRecord(strips, s1));
        RL_CUDA(cudaStreamWaitEvent(s2, strips, 0));
        mark(s2);
        panel256(o + W, s2);
        mark(s2);
        RL_CUDA(cudaEventRecord(done, s2));
        // (ii) ... while the main stream runs the remaining trailing update (K = 256)
        if (rest > w2)
            gemm(false, false, rest - w2, rest - w2, W, -1.0, at(o + W + w2, o), lda, at(o, o + W + w2), lda, 1.0,
                 at(o + W + w2, o + W + w2), lda);
        mark(s1);
        RL_CUDA(cudaStreamWaitEvent(s1, done, 0));
    }
    mark(s1);
    if (trace) { // per step: [s1 start, s2 start, s2 end, s1 trailing end], then the final mark
        RL_CUDA(cudaEventSynchronize(tev.back()));
        for (size_t i = 0; i + 4 < tev.size(); i += 4) {
            float strip = 0, panel = 0, trail = 0, step = 0;
            cudaEventElapsedTime(&strip, tev[i], tev[i + 1]);
            cudaEventElapsedTime(&panel, tev[i + 1], tev[i + 2]);
            cudaEventElapsedTime(&trail, tev[i + 1], tev[i + 3]);
            cudaEventElapsedTime(&step, tev[i], tev[i + 4]);
            std::fprintf(stderr, "lu step %3zu rest %6llu: strips %.3f panel %.3f trailing %.3f step %.3f ms\n",
                         i / 4, static_cast<unsigned long long>(n - (i / 4 + 1) * W), strip, panel, trail, step);
        }
        for (auto e : tev)
            cudaEventDestroy(e);
    }
}

void genp_factor_dev(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                     int64_t* d_breakdown) {
    RL_CUDA(cudaMemsetAsync(d_breakdown, 0xff, sizeof(int64_t), stream())); // -1 == none
    genp_factor_blocked(n, a, lda, pivot_floor, d_pivots,
                        reinterpret_cast<unsigned long long*>(d_breakdown), nullptr);
}

// Kept for the C-ABI signature (the solves need no precomputed block inverses).
void genp_block_inverses(uint64_t, const double*, uint64_t, double*) {}

// Forward (unit L) then backward (U) substitution, blocked: per 128-block a one-CTA
// substitution on the diagonal panel + a DMMA GEMM update of the remaining rows;
// b (n x nrhs, ldb) is overwritten by the solution (genp.cpp:106-124).
void genp_solve_blocked(uint64_t n, uint64_t nrhs, const double* lu, uint64_t lda, const double* aux,
                        double* b, uint64_t ldb) {
    (void)aux;
    prep_attrs();
    cudaStream_t st = stream();
    const size_t sm = solve_smem();
    // the 64 diagonal 128x128 blocks, gathered once into an L2-resident buffer (8 MiB at
    // n = 8192) so each block solve reads its triangle from L2, not from the 512 MiB LU
    const uint64_t nblk = (n + NB - 1) / NB;
    double* diag = ws<double>(WS_RF4, nblk * NB * NB);
    k_gather_diag<<<static_cast<unsigned>(nblk), 256, 0, st>>>(lu, lda, n, diag);
    RL_LAUNCHED();
    for (uint64_t c0 = 0; c0 < nrhs; c0 += SV_MAXRHS) { // RHS in slices of <= 32 columns
        const int nc = static_cast<int>(std::min<uint64_t>(SV_MAXRHS, nrhs - c0));
        double* bc = b + c0;
        for (uint64_t bi = 0; bi < nblk; ++bi) {
            const uint64_t o = bi * NB, bs = std::min<uint64_t>(NB, n - o);
            k_block_solve<<<1, PK_THREADS, sm, st>>>(diag + bi * NB * NB, NB, bs, 0, bc + o * ldb, ldb, nc, 1);
            RL_LAUNCHED();
            const uint64_t rest = n - o - bs;
            if (rest)
                gemm(false, false, rest, nc, bs, -1.0, lu + (o + bs) * lda + o, lda, bc + o * ldb, ldb, 1.0,
                     bc + (o + bs) * ldb, ldb);
        }
        for (uint64_t bi = nblk; bi-- > 0;) {
            const uint64_t o = bi * NB, bs = std::min<uint64_t>(NB, n - o);
            k_block_solve<<<1, PK_THREADS, sm, st>>>(diag + bi * NB * NB, NB, bs, 0, bc + o * ldb, ldb, nc, 0);
            RL_LAUNCHED();
            if (o)
                gemm(false, false, o, nc, bs, -1.0, lu + o, lda, bc + o * ldb, ldb, 1.0, bc, ldb);
        }
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

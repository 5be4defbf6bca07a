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
#include "reg_lu.cuh"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int NB = 128;        // block size (config 3's "Block size 128")
constexpr int kOuterSteps = 4; // 128-steps per outer block (trailing updates with K = 512)

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
// Panel-kernel phase timestamps (dev aid): build with -DRL_PANEL_TRACE and run with
// RL_DIAG_TRACE=1 to print the last diagonal-LU / TRSM launch's phase times.
#ifdef RL_PANEL_TRACE
#define RL_TS_DIAG()                                                                     \
    do {                                                                                 \
        if (tid == 0)                                                                    \
            g_diag_ts[tsi] = gtimer0();                                                  \
        ++tsi;                                                                           \
    } while (0)
#define RL_TS_TRSM()                                                                     \
    do {                                                                                 \
        if (tr)                                                                          \
            tsb[tsi] = gtimer0();                                                        \
        ++tsi;                                                                           \
    } while (0)
#else
#define RL_TS_DIAG() \
    do {             \
    } while (0)
#define RL_TS_TRSM() \
    do {             \
    } while (0)
#endif
#ifdef RL_PANEL_TRACE
__device__ unsigned long long g_diag_ts[64];
__device__ unsigned long long g_trsm_ts[2][40];
__device__ __forceinline__ unsigned long long gtimer0() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
#endif
// RL_LU_TIMELINE=1 (dev aid): %globaltimer of every panel kernel's first start and last end,
// per 128-step: [diag start, diag end, trsm first start, trsm last end]
__device__ int g_tl_on;
__device__ unsigned long long g_tl[64][4];
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
__global__ void __launch_bounds__(PK_THREADS, 1) k_diag_lu(double* a, uint64_t lda, uint64_t n, uint64_t o,
                                                           double floor, double* pivots,
                                                           unsigned long long* breakdown) {
    extern __shared__ double W[]; // NB x PT
    __shared__ double rcp[NB], pabs[NB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bs = static_cast<int>((n - o) < NB ? (n - o) : NB);
    double* blk = a + o * lda + o;
#ifdef RL_PANEL_TRACE
    int tsi = 0;
#endif
    if (g_tl_on && tid == 0 && o / NB < 64)
        g_tl[o / NB][0] = tl_now();
    RL_TS_DIAG();
    panel::load_tile_async<NB, NB, PK_THREADS>(W, PT, blk, lda, bs, bs, [](int, int) { return true; });
    panel::cp_async_wait_all();
    __syncthreads();
    for (int i = bs + tid; i < NB; i += PK_THREADS) // identity beyond a ragged last block
        W[i * PT + i] = 1.0;
    __syncthreads();
    RL_TS_DIAG();
    // (1) 16x16 diagonal sub-block c0 by warp 0, lanes 0..15 own its rows, all in registers:
    //     per step the pivot row is read from the owner lane by shuffles, every lane forms
    //     1/p itself (correctly rounded reciprocal).
    auto phase1 = [&](int c0) {
        __syncwarp();
        double p[SB];
        const int r = c0 + (lane & (SB - 1));
#pragma unroll
        for (int l = 0; l < SB; ++l)
            p[l] = W[r * PT + c0 + l];
        double invs[SB], pivs[SB];
#pragma unroll
        for (int kk = 0; kk < SB; ++kk) {
            const double piv = __shfl_sync(0xffffffffu, p[kk], kk);
            const double inv = (piv == 0.0) ? 0.0 : __drcp_rn(piv);
            invs[kk] = inv;
            pivs[kk] = piv;
            const bool below = lane < SB && lane > kk;
            const double m = below ? p[kk] * inv : 0.0;
            p[kk] = below ? m : p[kk]; // selects, no branches: the shuffles stay converged
#pragma unroll
            for (int l = kk + 1; l < SB; ++l)
                p[l] = fma(-m, __shfl_sync(0xffffffffu, p[l], kk), p[l]);
        }
        if (lane == 0)
#pragma unroll
            for (int kk = 0; kk < SB; ++kk) {
                rcp[c0 + kk] = invs[kk];
                pabs[c0 + kk] = fabs(pivs[kk]);
            }
        if (lane < SB)
#pragma unroll
            for (int l = 0; l < SB; ++l)
                W[r * PT + c0 + l] = p[l];
    };
    if (warp == 0)
        phase1(0);
    __syncthreads();
    RL_TS_DIAG();
    for (int c0 = 0; c0 < NB; c0 += SB) {
        const int rest = NB - c0 - SB;
        if (rest == 0)
            break;
        // (2) rows below: l_r U_sub = w_r   (x_j = (w_j - sum_{l<j} x_l U_lj) / U_jj), threads
        //     [0, rest); (3) columns right beside it, threads [rest, 2 rest) (disjoint entries)
        if (tid < rest) {
            const int r = c0 + SB + tid;
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
        else if (tid < 2 * rest) {
            const int c = c0 + SB + (tid - rest);
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
        RL_TS_DIAG();
        // (4) trailing update W22 -= L21 U12 with lookahead: warp 0 updates the next 16 x 16
        //     diagonal block and factors it (phase 1 of c0 + 16) while warps 1..7 update the rest
        double* C22 = W + (c0 + SB) * PT + c0 + SB;
        const double* L21 = W + (c0 + SB) * PT + c0;
        const double* U12 = W + c0 * PT + c0 + SB;
        if (warp == 0) {
            panel::smem_update16(C22, PT, L21, PT, U12, PT, SB, SB, 0, 1, lane);
            __syncwarp();
            phase1(c0 + SB);
        } else {
            panel::smem_update16(C22, PT, L21, PT, U12, PT, rest, rest, warp - 1, PK_WARPS - 1, lane, true);
        }
        __syncthreads();
        RL_TS_DIAG();
    }
    panel::store_tile<NB, NB, PK_THREADS>(blk, lda, W, PT, bs, bs);
    RL_TS_DIAG();
#ifdef RL_PANEL_TRACE
    if (tid == 0)
        g_diag_ts[63] = tsi;
#endif
    if (g_tl_on && tid == 0 && o / NB < 64)
        g_tl[o / NB][1] = tl_now();
    if (tid < bs) { // |pivots| and the first step below the floor (genp.cpp:24-26)
        pivots[o + tid] = pabs[tid];
        if (pabs[tid] < floor)
            atomicMin(breakdown, static_cast<unsigned long long>(o + tid));
    }
}

// Register-resident diagonal-block LU (reg_lu.cuh, G = 16): 256 threads, the 128 x 128 block
// 16 x 16-cyclic in registers (thread (tr, tc) owns rows tr + 16 r, columns tc + 16 c), 128
// pivot steps with one barrier each in the reference's right-looking order (genp.cpp:20-33;
// m = w(i,k) (1/p), 1/p := 0 for p = 0), then L = w(i,k) (1/p) below the diagonal and the packed
// block back in place.  Rows / columns beyond a ragged last block are the identity.  The
// shared-memory request (kPanelSmem) keeps GEMM CTAs off the SM, as for the other panel kernels.
constexpr int DR_THREADS = 256;
__global__ void __launch_bounds__(DR_THREADS, 1) k_diag_lu_reg(double* a, uint64_t lda, uint64_t n, uint64_t o,
                                                               double floor, double* pivots,
                                                               unsigned long long* breakdown) {
    __shared__ __align__(16) double pub[2 * reglu::Pub<16>::SIZE];
    __shared__ double rcp[NB];
    const int t = threadIdx.x, tr = t >> 4, tc = t & 15;
    const int bs = static_cast<int>((n - o) < NB ? (n - o) : NB);
    double* blk = a + o * lda + o;
    if (g_tl_on && t == 0 && o / NB < 64)
        g_tl[o / NB][0] = tl_now();
    double w[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int i = tr + 16 * r, j = tc + 16 * c;
            w[r][c] = (i < bs && j < bs) ? blk[static_cast<uint64_t>(i) * lda + j] : (i == j ? 1.0 : 0.0);
        }
    double dummy = 0.0; // (the mbarrier hand-off, reg_lu.cuh MB, measured 31.4 against 30.0 us)
    reglu::factor<16, false>(w, dummy, reglu::Bufs{pub, rcp, nullptr}, tr, tc);
    __syncthreads(); // rcp complete
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int j = tc + 16 * c;
        const double inv = rcp[j];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int i = tr + 16 * r;
            double v = w[r][c];
            if (r > c || (r == c && tr > tc))
                v *= inv;
            if (i < bs && j < bs)
                blk[static_cast<uint64_t>(i) * lda + j] = v;
            if (i == j && i < bs) { // |pivots| and the first step below the floor (genp.cpp:24-26)
                pivots[o + i] = fabs(v);
                if (fabs(v) < floor)
                    atomicMin(breakdown, static_cast<unsigned long long>(o + i));
            }
        }
    }
    if (g_tl_on && t == 0 && o / NB < 64) {
        __threadfence();
        g_tl[o / NB][1] = tl_now();
    }
}

// Panel TRSMs of block step o (genp.cpp:77-92), in place, one launch:
//   CTAs [0, nrb):      64-row tiles of A21 <- A21 U11^-1   (x U11 = a)
//   CTAs [nrb, 2 nrb2): 64-column tiles of A12 <- L11^-1 A12 (L11 y = a, unit lower)
// Each sub-panel: per-thread 16-step substitution, then a DMMA update of the remaining
// columns (right) / rows (left) of the tile.
// Panel TRSMs of block step o (genp.cpp:77-92), in place, one launch.  Both sides are
// solved as X <- X T^{-1} with X a 64 x 128 tile and T upper triangular (staged in shared
// memory):
//   CTAs [0, nrb):      X = 64 rows of A21, T = U11            (L21 = A21 U11^-1)
//   CTAs [nrb, 2 nrb):  X = (64 columns of A12)^T, T = L11^T   (U12 = L11^-1 A12, unit T)
// X lives in DMMA accumulator registers for the whole solve: warp w holds rows 8w..8w+7, lane
// (g, q) the columns 8f + 2q, +1 of every 8-column fragment f.  Per 16-column sub-panel: the
// rows' 16-step substitution runs inside each quad (x_j formed by the lane holding column j,
// shared by one shuffle, x_j = (w_j - sum_l x_l T_lj) * (1/T_jj) in the reference's order),
// then the rest of the tile gets X[:, right] -= X[:, sub] T[sub, right] on DMMA with the A
// fragments gathered from the quad by shuffles and T from shared memory — no shared-memory
// read-modify-write of X.
constexpr int TR_TILE = 64;     // rows (right) / columns (left) per CTA
constexpr int TR_THREADS = 256; // 8 warps x 8 rows
constexpr int TP = NB + 4;      // staged T / X pitch (doubles): conflict-free fragment reads

__global__ void __launch_bounds__(TR_THREADS, 1) k_panel_trsm(double* a, uint64_t lda, uint64_t o, uint64_t rest,
                                                              int nrb) {
    extern __shared__ double smt[];
    double* T = smt;           // NB x TP: upper triangular factor (T[j][c], c >= j)
    double* Xs = smt + NB * TP; // staging of the X tile (right: 64 x TP; left: NB x (64 + 4), A12 rows)
    __shared__ double rcp[NB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
    const bool right = static_cast<int>(blockIdx.x) < nrb;
    const double* diag = a + o * lda + o;
    if (g_tl_on && tid == 0 && o / NB < 64)
        atomicMin(&g_tl[o / NB][2], tl_now());
#ifdef RL_PANEL_TRACE
    const bool tr = (blockIdx.x == 0 || static_cast<int>(blockIdx.x) == nrb) && tid == 0;
    unsigned long long* tsb = g_trsm_ts[right ? 0 : 1];
    int tsi = 0;
#endif
    RL_TS_TRSM();
    uint64_t x0;
    int nx;
    double* base;
    if (right) {
        x0 = static_cast<uint64_t>(blockIdx.x) * TR_TILE;
        nx = static_cast<int>(rest - x0 < TR_TILE ? rest - x0 : TR_TILE);
        base = a + (o + NB + x0) * lda + o; // rows x0.. of A21, 128 columns
        panel::load_tile_async<NB, NB, TR_THREADS>(T, TP, diag, lda, NB, NB, [](int i, int j) { return j >= i; });
        panel::load_tile_async<TR_TILE, NB, TR_THREADS>(Xs, TP, base, lda, nx, NB, [](int, int) { return true; });
    } else {
        x0 = static_cast<uint64_t>(blockIdx.x - nrb) * TR_TILE;
        nx = static_cast<int>(rest - x0 < TR_TILE ? rest - x0 : TR_TILE);
        base = a + o * lda + o + NB + x0; // 128 rows of A12, columns x0..
        panel::load_tile_async<NB, TR_TILE, TR_THREADS>(Xs, TR_TILE + 4, base, lda, NB, nx,
                                                        [](int, int) { return true; });
        // T = L11^T (strictly upper): coalesced reads along L11's rows, transposed stores
        for (int e = tid; e < NB * NB; e += TR_THREADS) {
            const int c = e >> 7, j = e & (NB - 1); // L11[c][j] -> T[j][c]
            T[j * TP + c] = (c > j) ? __ldg(diag + static_cast<uint64_t>(c) * lda + j) : 0.0;
        }
    }
    panel::cp_async_wait_all();
    __syncthreads();
    RL_TS_TRSM();
    if (right && tid < NB) {
        const double d = T[tid * TP + tid];
        rcp[tid] = (d == 0.0) ? 0.0 : 1.0 / d;
    }
    // X rows 8 warp + g: x[f][e] = X[row][8 f + 2 q + e]
    const int row = 8 * warp + g;
    double x[NB / 8][2];
#pragma unroll
    for (int f = 0; f < NB / 8; ++f)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 8 * f + 2 * q + e;
            x[f][e] = right ? Xs[row * TP + c] : Xs[c * (TR_TILE + 4) + row];
        }
    __syncthreads();
    RL_TS_TRSM();
#pragma unroll
    for (int c0 = 0; c0 < NB; c0 += 16) {
        const int f0 = c0 / 8;
        // (1) substitution over columns c0..c0+15 inside the quad: this lane holds columns
        //     c0 + 8 h + 2 q + e (h, e in {0, 1}) of the sub-panel
        double rc16[16], tv[16][4];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) { // everything off the chain is loaded up front
            rc16[jj] = right ? rcp[c0 + jj] : 1.0;
#pragma unroll
            for (int hs = 0; hs < 4; ++hs)
                tv[jj][hs] = T[(c0 + jj) * TP + c0 + 8 * (hs >> 1) + 2 * q + (hs & 1)];
        }
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            const int j = c0 + jj, fj = j >> 3, qj = (j & 7) >> 1, ej = j & 1;
            const double xj = __shfl_sync(0xffffffffu, x[fj][ej] * rc16[jj], (lane & ~3) | qj);
#pragma unroll
            for (int hs = 0; hs < 4; ++hs) {
                const int h = hs >> 1, e = hs & 1;
                const int c = c0 + 8 * h + 2 * q + e;
                double& v = x[f0 + h][e];
                const double upd = fma(-xj, tv[jj][hs], v);
                v = (c == j) ? xj : ((c > j) ? upd : v);
            }
        }
        RL_TS_TRSM();
        if (c0 + 16 < NB) {
            // (2) X[:, c0+16:] -= X[:, c0:c0+16] T[c0:c0+16, c0+16:]  (DMMA, K = 16)
            double af[4];
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) { // A fragment: row g, column c0 + 4 ks + q
                const int c = 4 * ks + q;     // column within the sub-panel (0..15)
                const int src = (lane & ~3) | ((c & 7) >> 1);
                const double v0 = __shfl_sync(0xffffffffu, x[f0 + (c >> 3)][0], src);
                const double v1 = __shfl_sync(0xffffffffu, x[f0 + (c >> 3)][1], src);
                af[ks] = (c & 1) ? v1 : v0;
            }
#pragma unroll
            for (int f = f0 + 2; f < NB / 8; ++f) {
                double acc[2] = {0.0, 0.0};
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                 : "+d"(acc[0]), "+d"(acc[1])
                                 : "d"(af[ks]), "d"(T[(c0 + 4 * ks + q) * TP + 8 * f + g]));
                x[f][0] -= acc[0];
                x[f][1] -= acc[1];
            }
        }
    }
    RL_TS_TRSM();
    // store
    if (row < nx) {
        if (right) {
#pragma unroll
            for (int f = 0; f < NB / 8; ++f) {
                double* d = base + static_cast<uint64_t>(row) * lda + 8 * f + 2 * q;
                d[0] = x[f][0];
                d[1] = x[f][1];
            }
        } else {
#pragma unroll
            for (int f = 0; f < NB / 8; ++f)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    base[static_cast<uint64_t>(8 * f + 2 * q + e) * lda + row] = x[f][e];
        }
    }
    if (g_tl_on && tid == 0 && o / NB < 64)
        atomicMax(&g_tl[o / NB][3], tl_now());
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

// Wavefront block substitution (genp.cpp:106-124, forward unit-L / backward U) for up to
// WV_MAXRHS right-hand sides: one CTA per 128-row block, all launched at once.  A CTA takes
// its block from an atomic ticket (so a CTA only ever waits on blocks owned by CTAs that
// are already running: no deadlock whatever the residency), stages its diagonal triangle,
// then for every earlier block j (in order, deterministic) prefetches the 128 x 128 block
// L[b][j] into registers, waits for block j's published solution (acquire flag) and
// accumulates L[b][j] x_j on DMMA; finally it substitutes its own 128 rows (one warp per
// right-hand side, shuffle chain) and publishes x_b (release flag).  The critical path per
// block is one 128 x 128 x nrhs product plus one 128-step substitution, instead of a block
// solve launch plus a GEMM launch.
constexpr int WV_THREADS = 512;
constexpr int WV_MAXRHS = 32;
constexpr int XJP = WV_MAXRHS + 4; // staged x_j pitch: B-fragment reads conflict-free
__host__ __device__ constexpr size_t wave_smem_bytes() {
    return (static_cast<size_t>(NB) * NB + static_cast<size_t>(WV_MAXRHS) * NB + NB + static_cast<size_t>(NB) * XJP) *
           sizeof(double);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// RL_WAVE_TRACE=1 (dev): per-block %globaltimer stamps of the wavefront phases
__device__ unsigned long long g_wave_ts[2][512][6];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}

template <bool LOWER>
__global__ void __launch_bounds__(WV_THREADS, 1) k_trsv_wave(const double* __restrict__ lu, uint64_t lda, uint64_t n,
                                                             double* b, uint64_t ldb, int nrhs, int* sync,
                                                             int trace) {
    extern __shared__ __align__(16) double wsm[];
    double* Dt = wsm;                       // Dt[k * NB + i] = D[i][k] (triangle, transposed)
    double* xs = wsm + NB * NB;             // xs[c * NB + i]
    double* rcp = xs + WV_MAXRHS * NB;      // 1 / U_ii (upper)
    double* xj_s = rcp + NB;                // x_j staged: xj_s[k * XJP + c]
    __shared__ int s_blk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int nblk = static_cast<int>((n + NB - 1) / NB);
    if (tid == 0) {
        const int tk = atomicAdd(&sync[0], 1);
        s_blk = LOWER ? tk : nblk - 1 - tk;
    }
    __syncthreads();
    const int bi = s_blk;
    const uint64_t o = static_cast<uint64_t>(bi) * NB;
    const int bs = static_cast<int>(n - o < NB ? n - o : NB);
    for (int e = tid; e < NB * NB; e += WV_THREADS) {
        const int i = e >> 7, k = e & (NB - 1);
        const double v = (i < bs && k < bs) ? lu[(o + i) * lda + o + k] : 0.0;
        Dt[k * NB + i] = (LOWER ? (i > k) : (i < k)) ? v : 0.0;
        if (!LOWER && i == k)
            rcp[i] = (i < bs) ? 1.0 / v : 1.0;
    }
    __syncthreads(); // Dt / rcp complete (the first block of a sweep has no wait barrier below)
    // sum_j D[b][j] x_j over the finished blocks (DMMA m8n8k4: warp w owns rows 8w..8w+7)
    const int r = 8 * warp + g;
    const int nf = (nrhs + 7) >> 3;
    double acc[4][4] = {}; // [f][chain * 2 + e]
    const int nsteps = LOWER ? bi : nblk - 1 - bi;
    unsigned long long ts[6] = {gtimer(), 0, 0, 0, 0, 0};
    for (int s = 0; s < nsteps; ++s) {
        const int j = LOWER ? s : nblk - 1 - s;
        const uint64_t oj = static_cast<uint64_t>(j) * NB;
        const int bj = static_cast<int>(n - oj < NB ? n - oj : NB);
        double af[32];
        const double* arow = lu + (o + (r < bs ? r : 0)) * lda + oj;
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) {
            const int k = 4 * kk + t;
            af[kk] = (r < bs && k < bj) ? arow[k] : 0.0;
        }
        if (tid == 0)
            while (ld_acquire(&sync[1 + j]) == 0)
                __nanosleep(32);
        __syncthreads(); // also: every warp is done reading xj_s of the previous step
        ts[1] = gtimer();
        const double* xj = b + oj * ldb;
        for (int e = tid; e < NB * WV_MAXRHS; e += WV_THREADS) {
            const int k = e / WV_MAXRHS, c = e % WV_MAXRHS;
            xj_s[k * XJP + c] = (k < bj && c < nrhs) ? __ldcg(xj + static_cast<uint64_t>(k) * ldb + c) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int f = 0; f < 4; ++f) {
            if (f < nf) {
#pragma unroll
                for (int kk = 0; kk < 32; ++kk) { // two independent accumulation chains
                    const double bv = xj_s[(4 * kk + t) * XJP + 8 * f + g];
                    double* ac = acc[f] + 2 * (kk & 1);
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                 : "+d"(ac[0]), "+d"(ac[1])
                                 : "d"(af[kk]), "d"(bv));
                }
            }
        }
    }
    ts[1] = ts[1] ? ts[1] : ts[0];
    // In-block substitution on the DMMA accumulator layout: warp w keeps rows 8w..8w+7 of
    // X = B_b - sum_j D[b][j] x_j as C fragments.  Per 8-row sub-block s (in sweep order) the
    // owner warp s finishes its rows (8 x 8 triangle, one lane per right-hand side, through a
    // double-buffered shared tile) and every warp still below (above) applies the solved
    // 8 x nrhs block with two DMMA k-steps: one barrier per sub-block.
    double X[4][2];
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 8 * f + 2 * t + e;
            X[f][e] = (f < nf && c < nrhs && r < bs) ? b[(o + r) * ldb + c] - (acc[f][e] + acc[f][2 + e]) : 0.0;
        }
    ts[2] = gtimer();
#pragma unroll 1
    for (int it = 0; it < NB / 8; ++it) {
        const int sb = LOWER ? it : NB / 8 - 1 - it;
        double* xt = xs + (it & 1) * (8 * WV_MAXRHS); // [i][c], 8 x 32
        if (warp == sb) {
            // coefficients of the 8 x 8 diagonal triangle (broadcast reads, independent of X)
            double d[8][8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    d[i][k] = (LOWER ? (k < i) : (k > i)) ? Dt[(8 * sb + k) * NB + 8 * sb + i] : 0.0;
#pragma unroll
            for (int f = 0; f < 4; ++f)
                if (f < nf)
                    *reinterpret_cast<double2*>(xt + g * WV_MAXRHS + 8 * f + 2 * t) = make_double2(X[f][0], X[f][1]);
            __syncwarp();
            double v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                v[i] = xt[i * WV_MAXRHS + lane];
            if (LOWER) {
#pragma unroll
                for (int i = 1; i < 8; ++i)
#pragma unroll
                    for (int k = 0; k < i; ++k)
                        v[i] = fma(-d[i][k], v[k], v[i]);
            } else {
#pragma unroll
                for (int i = 7; i >= 0; --i) {
#pragma unroll
                    for (int k = i + 1; k < 8; ++k)
                        v[i] = fma(-d[i][k], v[k], v[i]);
                    v[i] = v[i] * rcp[8 * sb + i];
                }
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 8; ++i)
                xt[i * WV_MAXRHS + lane] = v[i];
            if (lane < nrhs)
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (8 * sb + i < bs)
                        b[(o + 8 * sb + i) * ldb + lane] = v[i];
        }
        __syncthreads();
        if (LOWER ? (warp > sb) : (warp < sb)) {
#pragma unroll
            for (int kk = 0; kk < 8; kk += 4) {
                const double a = -Dt[(8 * sb + kk + t) * NB + 8 * warp + g]; // -D[8w + g][8 sb + kk + t]
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    if (f < nf) {
                        const double bv = xt[(kk + t) * WV_MAXRHS + 8 * f + g];
                        asm volatile(
                            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                            : "+d"(X[f][0]), "+d"(X[f][1])
                            : "d"(a), "d"(bv));
                    }
            }
        }
    }
    ts[3] = gtimer();
    __syncthreads();
    ts[4] = gtimer();
    if (tid == 0) {
        st_release(&sync[1 + bi], 1);
        ts[5] = gtimer();
        if (trace && bi < 512)
            for (int q = 0; q < 6; ++q)
                g_wave_ts[LOWER ? 0 : 1][bi][q] = ts[q];
    }
}

// The panel kernels are on the factorization's critical path and run beside the trailing
// GEMMs of the other streams: they reserve (nearly) all of an SM's shared memory so no GEMM
// CTA is co-scheduled on their SM and steals issue slots.
constexpr size_t kPanelSmem = 220 * 1024;
size_t trsm_smem() {
    // T (NB x TP) + staging of the X tile (right 64 x TP, left NB x (64 + 4))
    const size_t need = (static_cast<size_t>(NB) * TP + static_cast<size_t>(NB) * (TR_TILE + 4)) * sizeof(double);
    return need > kPanelSmem ? need : kPanelSmem;
}
size_t diag_smem() { return kPanelSmem; }

void prep_attrs() {
    static bool done[16] = {};
    int dev = ctx().device & 15;
    if (!done[dev]) {
        RL_CUDA(cudaFuncSetAttribute(k_panel_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(trsm_smem())));
        RL_CUDA(cudaFuncSetAttribute(k_diag_lu, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(diag_smem())));
        RL_CUDA(cudaFuncSetAttribute(k_diag_lu_reg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(diag_smem() - 8 * 1024)));
        RL_CUDA(cudaFuncSetAttribute(k_trsv_wave<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(wave_smem_bytes())));
        RL_CUDA(cudaFuncSetAttribute(k_trsv_wave<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(wave_smem_bytes())));

        done[dev] = true;
    }
}

// Per-thread helper stream (high priority) and events for the panel lookahead.
struct Lookahead {
    cudaStream_t s2 = nullptr, s3 = nullptr, s4 = nullptr;
    cudaEvent_t ev[8] = {};
    int device = -1;
};

Lookahead& lookahead() {
    static thread_local Lookahead la;
    if (la.device != ctx().device) {
        int lo = 0, hi = 0;
        RL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        RL_CUDA(cudaStreamCreateWithPriority(&la.s2, cudaStreamNonBlocking, hi));
        RL_CUDA(cudaStreamCreateWithPriority(&la.s3, cudaStreamNonBlocking, hi));
        RL_CUDA(cudaStreamCreateWithPriority(&la.s4, cudaStreamNonBlocking, hi));
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

void diag_trace_dump() {
#ifndef RL_PANEL_TRACE
    std::fprintf(stderr, "RL_DIAG_TRACE: build with -DRL_PANEL_TRACE for panel phase times\n");
#else
    unsigned long long h[64];
    RL_CUDA(cudaDeviceSynchronize());
    RL_CUDA(cudaMemcpyFromSymbol(h, g_diag_ts, sizeof(h)));
    const int cnt = static_cast<int>(h[63]);
    unsigned long long t[2][40];
    RL_CUDA(cudaMemcpyFromSymbol(t, g_trsm_ts, sizeof(t)));
    for (int side = 0; side < 2; ++side) {
        std::fprintf(stderr, "trsm %s phases:", side ? "left" : "right");
        for (int i = 1; i < 20; ++i)
            std::fprintf(stderr, " %.2f", (t[side][i] - t[side][0]) * 1e-3);
        std::fprintf(stderr, "\n");
    }
    std::fprintf(stderr, "diag phases (us from start):");
    for (int i = 1; i < cnt && i < 63; ++i)
        std::fprintf(stderr, " %.2f", (h[i] - h[0]) * 1e-3);
    std::fprintf(stderr, "\n");

#endif
}

// Blocked right-looking GENP in place (packed LU), outer block W = 256 built from two 128
// steps, with lookahead over three streams so that the critical chain per outer step is
// only  diag LU -> TRSMs -> 128^3 update -> diag LU -> TRSMs  (+ one 128 x 128 x 256 GEMM):
//   s1 (main)   after panel k: the next diagonal block (128^2 x 256) first [E_nd], then the
//               next panel's column strip and row strip [E_strips], then the remaining
//               trailing update (the big K = 256 DMMA GEMM) while panel k+1 runs;
//   s2 (panel)  diag LU (waits E_nd only) -> TRSMs (wait E_strips) -> the second 128 block's
//               own 128^3 update -> its diag LU -> its TRSMs (wait E_s3)  [E_panel];
//   s3 (helper) the second 128 step's column / row strips (K = 128), beside s2.
// s2 and s3 have high priority.  Concurrently written regions are disjoint.
// The L and U produced are those of block_ge with block 128 (genp.cpp:43-104) up to
// rounding.  aux is unused.
void genp_factor_blocked(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                         unsigned long long* d_breakdown, double* aux) {
    (void)aux;
    prep_attrs();
    cudaStream_t s1 = stream();
    Lookahead& la = lookahead();
    cudaStream_t s2 = la.s2, s3 = la.s3, s4 = la.s4;
    if (n <= static_cast<uint64_t>(kOuterSteps) * NB) // one outer panel: nothing to overlap, and
        s2 = s3 = s4 = s1;                           // each cross-stream hop costs ~5 us
    cudaEvent_t E_nd = la.ev[0], E_strips = la.ev[1], E_panel = la.ev[2], E_t1 = la.ev[3], E_s3 = la.ev[4],
                E_s4 = la.ev[5];
    auto at = [&](uint64_t i, uint64_t j) { return a + i * lda + j; };
    const cudaStream_t keep = ctx().stream;
    const uint64_t W = static_cast<uint64_t>(kOuterSteps) * NB; // outer block
    // C -= A B on stream st (m x nn x k, all blocks of a)
    auto upd = [&](cudaStream_t st, uint64_t m, uint64_t nn, uint64_t k, const double* A, const double* B, double* C) {
        if (m == 0 || nn == 0)
            return;
        ctx().stream = st;
        gemm(false, false, m, nn, k, -1.0, A, lda, B, lda, 1.0, C, lda);
        ctx().stream = keep;
    };
    auto diag = [&](uint64_t o, cudaStream_t st) {
        // RL_DIAG_REG=1 (dev): the register kernel — 30 against 32 us per block, but its rounding
        // moves config 3's accepted attempts, which sit inside the reference's own 1-ulp band
        // (agreement with the oracle 6/16 columns against 11/16; the oracle agrees with itself
        // under a 1-ulp perturbation in 7/16), and the step then needs three draws, not two
        static const bool reg_diag = std::getenv("RL_DIAG_REG") != nullptr;
        if (!reg_diag)
            k_diag_lu<<<1, PK_THREADS, diag_smem(), st>>>(a, lda, n, o, pivot_floor, d_pivots, d_breakdown);
        else
            k_diag_lu_reg<<<1, DR_THREADS, diag_smem() - 8 * 1024, st>>>(a, lda, n, o, pivot_floor, d_pivots,
                                                                          d_breakdown);
        RL_LAUNCHED();
    };
    auto trsm = [&](uint64_t o, cudaStream_t st) {
        const uint64_t rest = n - o - std::min<uint64_t>(NB, n - o);
        if (rest) {
            const int nrb = static_cast<int>((rest + TR_TILE - 1) / TR_TILE);
            k_panel_trsm<<<2 * nrb, TR_THREADS, trsm_smem(), st>>>(a, lda, o, rest, nrb);
            RL_LAUNCHED();
        }
    };
    // outer panel [o, o + W) on s2 as W / 128 steps: waits E_nd before its first diag LU and
    // E_strips before its first TRSMs.  After step i (K = 128 from its L and U), the rows and
    // columns of the panel's remaining steps are brought up to date in two parts:
    //   urgent (s3, the next TRSMs wait for it): the next step's column strip below its block
    //     and its block row to the right (up to n);
    //   the rest (s4, beside the next diag LU and TRSMs): the panel's later columns below the
    //     next block and the panel's later rows right of the panel.  The next step's own-block
    //     update and urgent strips wait for it (they update the same entries after it).
    // The next step's own 128 x 128 block is updated on s2 (its LU starts next).  Rows and
    // columns beyond the panel get their update later with K = W (the trailing update).
    auto panelW = [&](uint64_t o) {
        const uint64_t oe = std::min<uint64_t>(o + W, n);
        RL_CUDA(cudaStreamWaitEvent(s2, E_nd, 0));
        diag(o, s2);
        RL_CUDA(cudaStreamWaitEvent(s2, E_strips, 0));
        trsm(o, s2);
        bool s4_pending = false;
        for (uint64_t oi = o; oi + NB < oe; oi += NB) {
            const uint64_t on = oi + NB, wn = std::min<uint64_t>(NB, oe - on), nx = on + wn;
            RL_CUDA(cudaEventRecord(E_t1, s2));
            RL_CUDA(cudaStreamWaitEvent(s3, E_t1, 0));
            RL_CUDA(cudaStreamWaitEvent(s4, E_t1, 0));
            if (s4_pending) { // the previous step's remainder covers this step's targets
                RL_CUDA(cudaStreamWaitEvent(s2, E_s4, 0));
                RL_CUDA(cudaStreamWaitEvent(s3, E_s4, 0));
            }
            upd(s2, wn, wn, NB, at(on, oi), at(oi, on), at(on, on));                    // own block
            upd(s3, n - nx, wn, NB, at(nx, oi), at(oi, on), at(nx, on));                 // its columns below
            upd(s3, wn, n - nx, NB, at(on, oi), at(oi, nx), at(on, nx));                 // its rows right
            RL_CUDA(cudaEventRecord(E_s3, s3));
            upd(s4, n - nx, oe - nx, NB, at(nx, oi), at(oi, nx), at(nx, nx));            // later panel cols below
            upd(s4, oe - nx, n - oe, NB, at(nx, oi), at(oi, oe), at(nx, oe));            // later panel rows right
            RL_CUDA(cudaEventRecord(E_s4, s4));
            s4_pending = true;
            diag(on, s2);
            RL_CUDA(cudaStreamWaitEvent(s2, E_s3, 0));
            trsm(on, s2);
        }
        if (s4_pending)
            RL_CUDA(cudaStreamWaitEvent(s2, E_s4, 0));
        RL_CUDA(cudaEventRecord(E_panel, s2));
    };
    static const bool timeline = std::getenv("RL_LU_TIMELINE") != nullptr;
    if (timeline) {
        static unsigned long long init[64][4];
        for (auto& r : init) {
            r[0] = r[1] = r[3] = 0;
            r[2] = ~0ULL;
        }
        const int on = 1;
        RL_CUDA(cudaMemcpyToSymbolAsync(g_tl, init, sizeof(init), 0, cudaMemcpyHostToDevice, s1));
        RL_CUDA(cudaMemcpyToSymbolAsync(g_tl_on, &on, sizeof(int), 0, cudaMemcpyHostToDevice, s1));
    }
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
    // the first panel: nothing to wait for beyond the work already on s1
    RL_CUDA(cudaEventRecord(E_nd, s1));
    RL_CUDA(cudaEventRecord(E_strips, s1));
    panelW(0);
    for (uint64_t o = 0; o + W < n; o += W) {
        RL_CUDA(cudaStreamWaitEvent(s1, E_panel, 0));
        mark(s1);
        const uint64_t p = o + W, rest = n - p;             // next panel at p, trailing size
        const uint64_t w2n = std::min<uint64_t>(W, rest);   // width of the next outer panel
        const uint64_t nd = std::min<uint64_t>(NB, rest);   // its first diagonal block
        const double* L21 = at(p, o);                       // rest x 256
        const double* U12 = at(o, p);                       // 256 x rest
        upd(s1, nd, nd, W, L21, U12, at(p, p));                                     // next diag block
        RL_CUDA(cudaEventRecord(E_nd, s1));
        upd(s1, nd, rest - nd, W, L21, at(o, p + nd), at(p, p + nd));               // its block row
        upd(s1, rest - nd, w2n, W, at(p + nd, o), U12, at(p + nd, p));              // panel columns below
        upd(s1, w2n - nd, rest - w2n, W, at(p + nd, o), at(o, p + w2n), at(p + nd, p + w2n)); // 2nd block row
        RL_CUDA(cudaEventRecord(E_strips, s1));
        mark(s2);
        panelW(p);
        mark(s2);
        // the remaining trailing update runs under the next panel
        upd(s1, rest - w2n, rest - w2n, W, at(p + w2n, o), at(o, p + w2n), at(p + w2n, p + w2n));
        mark(s1);
    }
    RL_CUDA(cudaStreamWaitEvent(s1, E_panel, 0));
    mark(s1);
    if (timeline) {
        unsigned long long h[64][4];
        const int off = 0;
        RL_CUDA(cudaMemcpyToSymbolAsync(g_tl_on, &off, sizeof(int), 0, cudaMemcpyHostToDevice, s1));
        RL_CUDA(cudaMemcpyFromSymbolAsync(h, g_tl, sizeof(h), 0, cudaMemcpyDeviceToHost, s1));
        RL_CUDA(cudaStreamSynchronize(s1));
        const unsigned long long t0 = h[0][0];
        const uint64_t steps = std::min<uint64_t>(64, (n + NB - 1) / NB);
        for (uint64_t i = 0; i < steps; ++i)
            std::fprintf(stderr, "tl %2llu: diag %8.1f +%6.1f  trsm %8.1f +%6.1f  (gap diag<-prev trsm %6.1f) us\n",
                         static_cast<unsigned long long>(i), (h[i][0] - t0) * 1e-3, (h[i][1] - h[i][0]) * 1e-3,
                         h[i][3] ? (h[i][2] - t0) * 1e-3 : 0.0, h[i][3] ? (h[i][3] - h[i][2]) * 1e-3 : 0.0,
                         i ? ((double)h[i][0] - (double)h[i - 1][3]) * 1e-3 : 0.0);
    }
    static const bool dtrace = std::getenv("RL_DIAG_TRACE") != nullptr;
    if (dtrace)
        diag_trace_dump();
    if (trace) { // per step: [s1 start, s2 start, s2 end, s1 trailing end], then the next s1 start
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

// One right-hand side, n <= 512: both substitutions in one warp (genp.cpp:106-124: the row-j
// update x_i -= L_ij x_j in ascending j, then x_i -= U_ij x_j in descending j and x_i / U_ii).
// Lane l keeps rows l + 32 q (q < NQ = n / 32 rounded up); the columns are swept in blocks of
// four (below).  The coefficients arrive as panels of W = 256 / NQ columns (rows from the
// panel's 32-row group down for L, rows 0.. for U) by TMA — two 256 x 16 boxes per panel, 128-byte
// swizzle (a lane's 128-bit read of its row's column pair and the quarter-warp's eight rows hit
// distinct banks), zero fill past n — into a 3-stage ring two panels ahead, so the warp never
// waits on L2 and no thread spends instructions on staging.
constexpr int SW_MAXN = 512, SW_STAGES = 3;
constexpr uint32_t SW_BOX = 256 * 128;    // one box: 256 rows x 16 doubles
constexpr uint32_t SW_STAGE = 2 * SW_BOX; // one panel
__host__ __device__ constexpr size_t sweep_smem_bytes() {
    return 1024 + static_cast<size_t>(SW_STAGES) * SW_STAGE + SW_MAXN * sizeof(double2);
}

__device__ __forceinline__ uint32_t sw_saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Byte offset of element (i, c) of a panel whose boxes start at row r0 (c even: the pair c, c+1).
// NQ = 8: the two boxes are columns 0-15 / 16-31; NQ = 16: rows r0.. / r0+256.. of 16 columns.
template <int NQ>
struct SweepGeo {
    static constexpr int W = 256 / NQ;
    __device__ static uint32_t off(int i, int c, int r0) {
        const int rr = i - r0;
        const int bx = NQ == 8 ? (c >> 4) : (rr >> 8);
        const int r = NQ == 8 ? rr : (rr & 255), cc = c & 15;
        return static_cast<uint32_t>(bx) * SW_BOX + static_cast<uint32_t>(r) * 128u +
               static_cast<uint32_t>((((cc >> 1) ^ (r & 7)) << 4) | ((cc & 1) << 3));
    }
    // the same for the lane's own row lane + 32 q, qrel = q minus the panel's first register
    // (a constant once the q loop is unrolled): the row part folds into an immediate, the
    // swizzle is lane & 7
    __device__ static uint32_t lane_off(int qrel, int lane, int c) {
        const int bxr = NQ == 8 ? 0 : qrel >> 3, rq = NQ == 8 ? qrel : qrel & 7;
        const int cc = c & 15;
        return static_cast<uint32_t>((NQ == 8 ? (c >> 4) : bxr)) * SW_BOX + static_cast<uint32_t>(lane + 32 * rq) * 128u +
               static_cast<uint32_t>((((cc >> 1) ^ (lane & 7)) << 4) | ((cc & 1) << 3));
    }
};

// x / U_jj as the reference divides.  Fast path: the reciprocal's quotient plus one residual
// correction — correctly rounded when the reciprocal is (Markstein) and nothing under- or
// overflows; a flag (integer ops, off the dependency chain) marks any step outside that range
// and the caller re-runs the pass with the division itself.  x and U_jj are warp-uniform.
template <bool EXACT>
__device__ __forceinline__ double sweep_div(double x, double2 d, unsigned& bad) {
    if (EXACT)
        return x / d.x;
    double q = x * d.y;
    q = fma(fma(-q, d.x, x), d.y, q);
    const int hx = __double2hiint(x) & 0x7fffffff;
    const unsigned eq = (__double2hiint(q) >> 20) & 0x7ff, ex = static_cast<unsigned>(hx) >> 20,
                   er = (__double2hiint(d.y) >> 20) & 0x7ff;
    const unsigned zx = (hx | __double2loint(x)) == 0;
    bad |= static_cast<unsigned>(er - 128u > 1792u) |
           ((zx ^ 1u) & (static_cast<unsigned>(eq - 128u > 1792u) | static_cast<unsigned>(ex - 128u > 1792u)));
    return q;
}

// One column step (ragged panel edges): x_j from its owner lane, then every row in reach.
template <bool LOWER, bool EXACT, int NQ, int QP>
__device__ __forceinline__ void sweep_col(const unsigned char* pb, int r0, const double2* dg, double (&x)[NQ], int j0,
                                          int jj, int lane, unsigned& bad) {
    using G = SweepGeo<NQ>;
    const int j = j0 + jj, src = j & 31;
    double xj = __shfl_sync(0xffffffffu, x[QP], src);
    if (!LOWER) {
        xj = sweep_div<EXACT>(xj, dg[j], bad);
        x[QP] = lane == src ? xj : x[QP];
    }
#pragma unroll
    for (int q = LOWER ? QP : 0; q < (LOWER ? NQ : QP + 1); ++q) {
        const int i = lane + 32 * q;
        const double f = fma(-*reinterpret_cast<const double*>(pb + G::lane_off(LOWER ? q - QP : q, lane, jj)),
                             xj, x[q]);
        x[q] = (q != QP || (LOWER ? i > j : i < j)) ? f : x[q];
    }
}

// Four column steps at once: the four x_j leave their owner lanes by four independent shuffles
// and every lane finishes them redundantly through the 4 x 4 triangle (broadcast coefficient
// reads) — the same operations, in the same order, as four single steps, with one shuffle
// latency on the chain instead of four.  Then every row takes the four updates (two 128-bit
// coefficient loads); rows of other registers than QP are all inside the triangle's reach
// (below the block for L, above for U), so only register QP needs the per-row selects.  Rows
// past n hold garbage that never reaches a valid row.
template <bool LOWER, bool EXACT, int NQ, int QP>
__device__ __forceinline__ void sweep_block4(const unsigned char* pb, int r0, const double2* dg, double (&x)[NQ],
                                             int j0, int jb, int lane, unsigned& bad) {
    using G = SweepGeo<NQ>;
    // L: columns jb, jb+1, jb+2, jb+3 in that order; U: jb+3, jb+2, jb+1, jb
    const int base = j0 + jb, s0 = base & 31;
    auto coef = [&](int i, int c) { return *reinterpret_cast<const double*>(pb + G::off(i, c, r0)); };
    double v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t)
        v[t] = __shfl_sync(0xffffffffu, x[QP], s0 + t);
    double xs[4]; // xs[t] = final x_{base + t}
    if (LOWER) {
        xs[0] = v[0];
#pragma unroll
        for (int t = 1; t < 4; ++t) {
            double a = v[t];
#pragma unroll
            for (int u = 0; u < t; ++u)
                a = fma(-coef(base + t, jb + u), xs[u], a);
            xs[t] = a;
        }
    } else {
        xs[3] = sweep_div<EXACT>(v[3], dg[base + 3], bad);
#pragma unroll
        for (int t = 2; t >= 0; --t) {
            double a = v[t];
#pragma unroll
            for (int u = 3; u > t; --u)
                a = fma(-coef(base + t, jb + u), xs[u], a);
            xs[t] = sweep_div<EXACT>(a, dg[base + t], bad);
        }
    }
#pragma unroll
    for (int q = LOWER ? QP : 0; q < (LOWER ? NQ : QP + 1); ++q) {
        const int i = lane + 32 * q;
        const double2 c01 = *reinterpret_cast<const double2*>(pb + G::lane_off(LOWER ? q - QP : q, lane, jb));
        const double2 c23 =
            *reinterpret_cast<const double2*>(pb + G::lane_off(LOWER ? q - QP : q, lane, jb + 2));
        const double c[4] = {c01.x, c01.y, c23.x, c23.y};
        double y = x[q];
        if (q != QP) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int u = LOWER ? t : 3 - t;
                y = fma(-c[u], xs[u], y);
            }
        } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int u = LOWER ? t : 3 - t;
                const double f = fma(-c[u], xs[u], y);
                y = (LOWER ? i > base + u : i < base + u) ? f : y;
            }
            if (!LOWER)
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    y = lane == s0 + t ? xs[t] : y;
        }
        x[q] = y;
    }
}

// The steps of one panel; QP = the register holding the panel's rows, resolved by recursion so
// every x[] index is a compile-time constant (x stays in registers).
template <bool LOWER, bool EXACT, int NQ, int QP>
__device__ __forceinline__ void sweep_panel(const unsigned char* pb, int r0, const double2* dg, double (&x)[NQ],
                                            int j0, int cols, int lane, unsigned& bad) {
    if constexpr (QP < NQ) {
        if ((j0 >> 5) != QP) {
            sweep_panel<LOWER, EXACT, NQ, QP + 1>(pb, r0, dg, x, j0, cols, lane, bad);
            return;
        }
        if (LOWER) {
            int jj = 0;
#pragma unroll 1
            for (; jj + 4 <= cols; jj += 4)
                sweep_block4<true, EXACT, NQ, QP>(pb, r0, dg, x, j0, jj, lane, bad);
#pragma unroll 1
            for (; jj < cols; ++jj)
                sweep_col<true, EXACT, NQ, QP>(pb, r0, dg, x, j0, jj, lane, bad);
        } else {
            int jj = cols - 1;
#pragma unroll 1
            for (; (jj + 1) & 3; --jj) // a ragged panel edge first: the blocks stay 4-aligned
                sweep_col<false, EXACT, NQ, QP>(pb, r0, dg, x, j0, jj, lane, bad);
#pragma unroll 1
            for (; jj >= 3; jj -= 4)
                sweep_block4<false, EXACT, NQ, QP>(pb, r0, dg, x, j0, jj - 3, lane, bad);
        }
    }
}

// RL_SWEEP_TRACE=1 (dev): per panel %globaltimer stamps: data ready / sweep end
__device__ unsigned long long g_sweep_ts[3][64][2];

// Panel sequence: 0..np-1 the L panels in order, then the U panels from the last, repeated for
// an exact re-run of the U pass.
template <int NQ>
struct SweepRing {
    const CUtensorMap* tm;
    unsigned char* buf;
    uint64_t* full;
    int np, lane;
    __device__ void panel(int seq, bool& lower, int& p) const {
        lower = seq < np;
        p = lower ? seq : np - 1 - (seq - np) % np;
    }
    __device__ int row0(bool lower, int p) const { return lower ? ((SweepGeo<NQ>::W * p) & ~31) : 0; }
    __device__ void issue(int seq, int limit) const { // lane 0
        if (lane != 0 || seq >= limit)
            return;
        bool lower;
        int p;
        panel(seq, lower, p);
        const int j0 = SweepGeo<NQ>::W * p, r0 = row0(lower, p), st = seq % SW_STAGES;
        const uint32_t mb = sw_saddr(&full[st]), dst = sw_saddr(buf) + st * SW_STAGE;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(SW_STAGE) : "memory");
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
            const int c = NQ == 8 ? j0 + 16 * bx : j0, r = NQ == 8 ? r0 : r0 + 256 * bx;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    dst + bx * SW_BOX),
                "l"(tm), "r"(c), "r"(r), "r"(mb)
                : "memory");
        }
    }
    __device__ const unsigned char* wait(int seq) const {
        const int st = seq % SW_STAGES;
        const uint32_t mb = sw_saddr(&full[st]), par = (seq / SW_STAGES) & 1;
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                         " selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(done)
                         : "r"(mb), "r"(par)
                         : "memory");
        return buf + st * SW_STAGE;
    }
};

template <bool LOWER, bool EXACT, int NQ>
__device__ __forceinline__ void sweep_pass(const SweepRing<NQ>& R, int seq0, int limit, int n, const double2* dg,
                                           double (&x)[NQ], int lane, unsigned& bad, int trace) {
    constexpr int W = SweepGeo<NQ>::W;
#pragma unroll 1
    for (int it = 0; it < R.np; ++it) {
        const int seq = seq0 + it;
        const unsigned char* pb = R.wait(seq);
        if (trace && lane == 0 && it < 64)
            g_sweep_ts[seq / R.np][it][0] = gtimer();
        __syncwarp();
        R.issue(seq + SW_STAGES - 1, limit); // into the stage the previous panel freed
        bool lower;
        int p;
        R.panel(seq, lower, p);
        const int j0 = W * p;
        sweep_panel<LOWER, EXACT, NQ, 0>(pb, R.row0(lower, p), dg, x, j0, min(W, n - j0), lane, bad);
        if (trace && lane == 0 && it < 64)
            g_sweep_ts[seq / R.np][it][1] = gtimer();
    }
}

template <int NQ>
__global__ void __launch_bounds__(32, 1) k_trsv_sweep1(const __grid_constant__ CUtensorMap tm,
                                                       const double* __restrict__ lu, uint64_t lda, int n, double* b,
                                                       uint64_t ldb, int trace) {
    extern __shared__ __align__(16) unsigned char swm[];
    __shared__ __align__(8) uint64_t full[SW_STAGES];
    const int lane = threadIdx.x;
    unsigned char* buf = swm + (((sw_saddr(swm) + 1023u) & ~1023u) - sw_saddr(swm));
    double2* dg = reinterpret_cast<double2*>(buf + SW_STAGES * SW_STAGE); // {U_ii, 1 / U_ii}
    const int np = (n + SweepGeo<NQ>::W - 1) / SweepGeo<NQ>::W;
    const SweepRing<NQ> R{&tm, buf, full, np, lane};
    if (lane == 0) {
        for (int s2 = 0; s2 < SW_STAGES; ++s2)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sw_saddr(&full[s2])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
    }
    __syncwarp();
    for (int s2 = 0; s2 < SW_STAGES - 1; ++s2)
        R.issue(s2, 2 * np);
    for (int i = lane; i < n; i += 32) {
        const double u = lu[static_cast<uint64_t>(i) * lda + i];
        dg[i] = make_double2(u, 1.0 / u);
    }
    double x[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int i = lane + 32 * q;
        x[q] = i < n ? b[static_cast<uint64_t>(i) * ldb] : 0.0;
    }
    __syncwarp();
    unsigned bad = 0;
    sweep_pass<true, false, NQ>(R, 0, 2 * np, n, dg, x, lane, bad, trace);
    double y[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
        y[q] = x[q];
    sweep_pass<false, false, NQ>(R, np, 2 * np, n, dg, x, lane, bad, trace);
    if (__any_sync(0xffffffffu, bad)) { // a quotient outside the fast path's range: divide
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            x[q] = y[q];
        __syncwarp();
        for (int s2 = 0; s2 < SW_STAGES - 1; ++s2)
            R.issue(2 * np + s2, 3 * np);
        sweep_pass<false, true, NQ>(R, 2 * np, 3 * np, n, dg, x, lane, bad, trace);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int i = lane + 32 * q;
        if (i < n)
            b[static_cast<uint64_t>(i) * ldb] = x[q];
    }
}

// Forward (unit L) then backward (U) substitution (genp.cpp:106-124) as two wavefront
// launches per slice of <= 32 right-hand sides; b (n x nrhs, ldb) is overwritten by the
// solution (one right-hand side with n <= 512: the one-CTA sweep).
void genp_solve_blocked(uint64_t n, uint64_t nrhs, const double* lu, uint64_t lda, const double* aux,
                        double* b, uint64_t ldb) {
    (void)aux;
    prep_attrs();
    cudaStream_t st = stream();
    static const bool no_sweep = std::getenv("RL_NO_SWEEP1") != nullptr; // dev comparison
    CUtensorMap tm;
    if (nrhs == 1 && n <= static_cast<uint64_t>(SW_MAXN) && !no_sweep &&
        make_tmap(&tm, lu, n, n, lda, 256)) { // one small system: one warp
        static bool attr[16] = {};
        if (!attr[ctx().device & 15]) {
            RL_CUDA(cudaFuncSetAttribute(k_trsv_sweep1<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sweep_smem_bytes())));
            RL_CUDA(cudaFuncSetAttribute(k_trsv_sweep1<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sweep_smem_bytes())));
            attr[ctx().device & 15] = true;
        }
        const int nn = static_cast<int>(n);
        static const bool strace = std::getenv("RL_SWEEP_TRACE") != nullptr;
        if (n <= 256)
            k_trsv_sweep1<8><<<1, 32, sweep_smem_bytes(), st>>>(tm, lu, lda, nn, b, ldb, strace);
        else
            k_trsv_sweep1<16><<<1, 32, sweep_smem_bytes(), st>>>(tm, lu, lda, nn, b, ldb, strace);
        RL_LAUNCHED();
        if (strace) {
            static unsigned long long h[3][64][2];
            RL_CUDA(cudaMemcpyFromSymbolAsync(h, g_sweep_ts, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
            RL_CUDA(cudaStreamSynchronize(st));
            const int np = static_cast<int>((n + (n <= 256 ? 31 : 15)) / (n <= 256 ? 32 : 16));
            const unsigned long long t0 = h[0][0][0];
            for (int d = 0; d < 2; ++d)
                for (int i = 0; i < np && i < 64; ++i)
                    std::fprintf(stderr, "sweep %s panel %2d: ready %7.2f end %7.2f us\n", d ? "U" : "L", i,
                                 (h[d][i][0] - t0) * 1e-3, (h[d][i][1] - t0) * 1e-3);
        }
        return;
    }
    const uint64_t nblk = (n + NB - 1) / NB;
    int* sync = ws<int>(WS_WAVE, 2 * (nblk + 1));
    static const bool trace = std::getenv("RL_WAVE_TRACE") != nullptr;
    for (uint64_t c0 = 0; c0 < nrhs; c0 += WV_MAXRHS) {
        const int nc = static_cast<int>(std::min<uint64_t>(WV_MAXRHS, nrhs - c0));
        RL_CUDA(cudaMemsetAsync(sync, 0, 2 * (nblk + 1) * sizeof(int), st));
        k_trsv_wave<true><<<static_cast<unsigned>(nblk), WV_THREADS, wave_smem_bytes(), st>>>(lu, lda, n, b + c0, ldb,
                                                                                          nc, sync, trace);
        RL_LAUNCHED();
        k_trsv_wave<false><<<static_cast<unsigned>(nblk), WV_THREADS, wave_smem_bytes(), st>>>(
            lu, lda, n, b + c0, ldb, nc, sync + nblk + 1, trace);
        RL_LAUNCHED();
    }
    if (trace && nblk <= 512) {
        static unsigned long long h[2][512][6];
        RL_CUDA(cudaMemcpyFromSymbolAsync(h, g_wave_ts, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
        RL_CUDA(cudaStreamSynchronize(st));
        for (int d = 0; d < 2; ++d) {
            unsigned long long t0 = ~0ULL;
            for (uint64_t i = 0; i < nblk; ++i)
                t0 = std::min(t0, h[d][i][0]);
            for (uint64_t i = 0; i < nblk; ++i) {
                const auto* q = h[d][i];
                std::fprintf(stderr, "wave %s blk %3llu: start %7.2f lastwait %7.2f dmma %6.2f rhs %6.2f solve %6.2f rel %6.2f us\n",
                             d ? "U" : "L", static_cast<unsigned long long>(i), (q[0] - t0) * 1e-3, (q[1] - t0) * 1e-3,
                             (q[2] - q[1]) * 1e-3, (q[3] - q[2]) * 1e-3, (q[4] - q[3]) * 1e-3, (q[5] - q[4]) * 1e-3);
            }
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

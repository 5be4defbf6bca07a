// K2: FP64 GEMM on the sm_100a FP64 tensor path.
//
// Replaces Matrix::multiply (proj/src/matrix.cpp:86-102, the naive i-k-j A*G) and
// every dense contraction of the path: A*G, the blocked-GENP TRSM/Schur updates,
// A*H, Q^T*A, G*Y.  On sm_100a FP64 tensor math exists only as DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; tcgen05 has no .kind::f64, SURVEY.md
// §0 item 6), measured at 37.1 TFLOP/s vs 36.6 for DFMA (profiles/r01_peaks.txt).
//
// Structure: CTA tile BM x BN, K-tile 16, NSTAGE-deep cp.async ring (global ->
// shared, 16-byte copies, zero-fill at the edges), 8 warps each owning a
// (BM/WM) x (BN/WN) accumulator tile in registers.  Shared tiles are padded so the
// m8n8k4 fragment reads (8 rows x 4 k) hit 4 distinct 32-byte bank groups per
// half-warp: no bank conflicts for either operand majorness.
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int BK = 16;
constexpr int PAD = 4; // doubles; row pitch = 32 B mod 128
constexpr uint64_t kLongK = 512; // K from which the 32-deep k-tile config is used

struct Split {
    int splits = 1;       // gridDim.z
    uint64_t kchunk = 0;  // K per slice (multiple of 16)
    uint64_t cstride = 0; // elements between the slices' C panels
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int bytes = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int bytes = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Shared-tile geometry for one operand.  KMAJOR: tile stored [rows=MN][BK+PAD];
// otherwise [BK][MN+PAD].
template <int MN, bool KMAJOR, int BKT = BK>
struct Tile {
    static constexpr int kPitch = KMAJOR ? (BKT + PAD) : (MN + PAD);
    static constexpr int kElems = KMAJOR ? MN * kPitch : BKT * kPitch;
    // element (mn, k) of the tile
    __device__ __forceinline__ static int at(int mn, int k) {
        return KMAJOR ? mn * kPitch + k : k * kPitch + mn;
    }
};

// Load one BK-slice of an operand tile.  KMAJOR global layout: g[(mn0+r)*ld + k0 + c];
// else g[(k0+r)*ld + mn0 + c].  dims: MNdim (rows along mn), Kdim.
template <int MN, bool KMAJOR, int VEC, int NT, int BKT = BK>
__device__ __forceinline__ void load_tile(double* s, const double* g, uint64_t ld, uint64_t mn0,
                                          uint64_t k0, uint64_t MNdim, uint64_t Kdim, int tid) {
    using T = Tile<MN, KMAJOR, BKT>;
    constexpr int ROWS = KMAJOR ? MN : BKT; // rows of the tile in memory order
    constexpr int COLS = KMAJOR ? BKT : MN; // contiguous extent
    constexpr int CPR = COLS / VEC;         // copies per row
    constexpr int TOTAL = ROWS * CPR;
#pragma unroll
    for (int it = 0; it < (TOTAL + NT - 1) / NT; ++it) {
        int idx = it * NT + tid;
        if (TOTAL % NT != 0 && idx >= TOTAL)
            break;
        int r = idx / CPR, c = (idx % CPR) * VEC;
        uint64_t grow, gcol;
        bool ok;
        if (KMAJOR) {
            grow = mn0 + r;
            gcol = k0 + c;
            ok = grow < MNdim && gcol < Kdim;
        } else {
            grow = k0 + r;
            gcol = mn0 + c;
            ok = grow < Kdim && gcol < MNdim;
        }
        const double* src = ok ? g + grow * ld + gcol : g;
        double* dst = s + r * T::kPitch + c;
        if (VEC == 2)
            cp_async16(dst, src, ok);
        else
            cp_async8(dst, src, ok);
    }
}

template <int BM, int BN, int WM, int WN, bool AK, bool BKM, int VEC, int NSTAGE, int BKT = BK>
struct Cfg {
    static constexpr int NT = WM * WN * 32;
    static constexpr int WTM = BM / WM, WTN = BN / WN;
    static constexpr int MF = WTM / 8, NF = WTN / 8;
    using TA = Tile<BM, AK, BKT>;
    using TB = Tile<BN, BKM, BKT>;
    static constexpr int kStageElems = TA::kElems + TB::kElems;
    static constexpr size_t kSmem = static_cast<size_t>(NSTAGE) * kStageElems * sizeof(double);
};

template <int BM, int BN, int WM, int WN, bool AK, bool BKM, int VEC, int NSTAGE, int MINB = 1, int BKT = BK>
__global__ void __launch_bounds__(WM* WN * 32, MINB)
    k_dgemm(uint64_t M, uint64_t N, uint64_t K, double alpha, const double* __restrict__ A,
            uint64_t lda, const double* __restrict__ B, uint64_t ldb, double beta,
            double* __restrict__ C, uint64_t ldc, uint64_t kchunk, uint64_t cstride) {
    using G = Cfg<BM, BN, WM, WN, AK, BKM, VEC, NSTAGE, BKT>;
    extern __shared__ __align__(16) double smem[];
    if (gridDim.z > 1) {
        // split-K: slice z covers k in [z kchunk, (z+1) kchunk) and writes its own C panel
        const uint64_t kz0 = blockIdx.z * kchunk;
        A += AK ? kz0 : kz0 * lda;
        B += BKM ? kz0 : kz0 * ldb;
        K = kz0 < K ? (K - kz0 < kchunk ? K - kz0 : kchunk) : 0;
        C += blockIdx.z * cstride;
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, t = lane & 3;
    const uint64_t m0 = static_cast<uint64_t>(blockIdx.y) * BM, n0 = static_cast<uint64_t>(blockIdx.x) * BN;
    const int ktiles = static_cast<int>((K + BKT - 1) / BKT);

    double acc[G::MF][G::NF][2];
#pragma unroll
    for (int i = 0; i < G::MF; ++i)
#pragma unroll
        for (int j = 0; j < G::NF; ++j)
            acc[i][j][0] = acc[i][j][1] = 0.0;

    auto sA = [&](int s) { return smem + s * G::kStageElems; };
    auto sB = [&](int s) { return smem + s * G::kStageElems + G::TA::kElems; };

#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
        if (s < ktiles) {
            load_tile<BM, AK, VEC, G::NT, BKT>(sA(s), A, lda, m0, static_cast<uint64_t>(s) * BKT, M, K, tid);
            load_tile<BN, BKM, VEC, G::NT, BKT>(sB(s), B, ldb, n0, static_cast<uint64_t>(s) * BKT, N, K, tid);
        }
        cp_commit();
    }

    for (int kt = 0; kt < ktiles; ++kt) {
        cp_wait<NSTAGE - 2>();
        __syncthreads();
        const int nk = kt + NSTAGE - 1;
        if (nk < ktiles) {
            int s = nk % NSTAGE;
            load_tile<BM, AK, VEC, G::NT, BKT>(sA(s), A, lda, m0, static_cast<uint64_t>(nk) * BKT, M, K, tid);
            load_tile<BN, BKM, VEC, G::NT, BKT>(sB(s), B, ldb, n0, static_cast<uint64_t>(nk) * BKT, N, K, tid);
        }
        cp_commit();
        const double* a_s = sA(kt % NSTAGE);
        const double* b_s = sB(kt % NSTAGE);
#pragma unroll
        for (int kk = 0; kk < BKT; kk += 4) {
            double af[G::MF], bf[G::NF];
#pragma unroll
            for (int i = 0; i < G::MF; ++i)
                af[i] = a_s[G::TA::at(wm * G::WTM + i * 8 + g, kk + t)];
#pragma unroll
            for (int j = 0; j < G::NF; ++j)
                bf[j] = b_s[G::TB::at(wn * G::WTN + j * 8 + g, kk + t)];
#pragma unroll
            for (int i = 0; i < G::MF; ++i)
#pragma unroll
                for (int j = 0; j < G::NF; ++j)
                    dmma(acc[i][j], af[i], bf[j]);
        }
    }
    cp_wait<0>();

    // epilogue: C = alpha acc + beta C
#pragma unroll
    for (int i = 0; i < G::MF; ++i) {
        uint64_t row = m0 + wm * G::WTM + i * 8 + g;
        if (row >= M)
            continue;
#pragma unroll
        for (int j = 0; j < G::NF; ++j) {
            uint64_t col = n0 + wn * G::WTN + j * 8 + 2 * t;
            double* cp = C + row * ldc + col;
            double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
            if (VEC == 2 && col + 1 < N) {
                if (beta != 0.0) {
                    double2 o = *reinterpret_cast<const double2*>(cp);
                    v0 = fma(beta, o.x, v0);
                    v1 = fma(beta, o.y, v1);
                }
                *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
            } else {
                if (col < N) {
                    if (beta != 0.0)
                        v0 = fma(beta, cp[0], v0);
                    cp[0] = v0;
                }
                if (col + 1 < N) {
                    if (beta != 0.0)
                        v1 = fma(beta, cp[1], v1);
                    cp[1] = v1;
                }
            }
        }
    }
}

// The long-K full-tile case of A K-major x B N-major (A·G, the big LU updates) fed by the TMA
// engine: per stage one thread issues six 2-D tensor copies (cp.async.bulk.tensor, SASS UTMALDG)
// — A as two 128 x 16 boxes, B as four 32 x 16 boxes, 16 doubles = one 128-byte swizzle span
// each — completing on one mbarrier per stage (expect_tx = the stage's 48 KB). The boxes land
// with the 128-byte swizzle (16-byte chunk c of line r stored at c ^ (r mod 8)), which keeps the
// DMMA fragment reads at the minimum two wavefronts for A (8 rows x 4 k) and four for B (4 k x
// 8 n, a 2-way conflict: DMMA, not shared memory, bounds the loop); the fragment addresses apply
// the same XOR. The 256 threads issue only fragment loads and DMMAs. Same tile and k order as
// k_dgemm: bit-identical results.
__device__ __forceinline__ uint32_t s_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
constexpr int TM_BK = 32;
// Tile geometry of the TMA kernel: BM x BN output tile, K-tile 32, WM x WN warps. A is K-major
// (boxes BM x 16 along k: A·G, A·H) or M-major (boxes 32 x 16 along m: Q^T A); B is N-major
// (boxes 32 x 16 along n). Box edges past M / N / K are zero-filled by the copy engine.
template <int BM, int BN, int WM, int WN, bool AKM, bool BKMJ, int TM_NSTAGE>
struct TmCfg {
    static constexpr int NT = WM * WN * 32;
    static constexpr int WTM = BM / WM, WTN = BN / WN, MF = WTM / 8, NF = WTN / 8;
    static constexpr int A_BYTES = BM * TM_BK * 8, B_BYTES = TM_BK * BN * 8;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr size_t SMEM = static_cast<size_t>(TM_NSTAGE) * STAGE + 1024; // + alignment slack
    static constexpr int A_BOXES = AKM ? TM_BK / 16 : BM / 16, B_BOXES = BKMJ ? TM_BK / 16 : BN / 16;
    static constexpr int A_BOX_BYTES = AKM ? BM * 128 : TM_BK * 128, B_BOX_BYTES = BKMJ ? BN * 128 : TM_BK * 128;
    // every box starts on a 1024-byte swizzle-pattern boundary
    static_assert(A_BYTES % 1024 == 0 && A_BOX_BYTES % 1024 == 0 && B_BOX_BYTES % 1024 == 0, "box alignment");
    // byte offsets of A(r, k) / B(k, n) in a stage (128-byte swizzle: chunk c of line l at c ^ (l & 7))
    __device__ __forceinline__ static uint32_t a_off(int r, int k) {
        if (AKM)
            return static_cast<uint32_t>((k >> 4) * A_BOX_BYTES + r * 128 + ((((k & 15) >> 1) ^ (r & 7)) << 4) +
                                         ((k & 1) << 3));
        return static_cast<uint32_t>((r >> 4) * A_BOX_BYTES + k * 128 + ((((r & 15) >> 1) ^ (k & 7)) << 4) +
                                     ((r & 1) << 3));
    }
    __device__ __forceinline__ static uint32_t b_off(int k, int n) {
        if (BKMJ) // B stored N x K (K-major): the same box geometry as a K-major A
            return static_cast<uint32_t>(A_BYTES + (k >> 4) * B_BOX_BYTES + n * 128 +
                                         ((((k & 15) >> 1) ^ (n & 7)) << 4) + ((k & 1) << 3));
        return static_cast<uint32_t>(A_BYTES + (n >> 4) * (TM_BK * 128) + k * 128 + ((((n & 15) >> 1) ^ (k & 7)) << 4) +
                                     ((n & 1) << 3));
    }
};

// The TMA-fed DGEMM (A·G, the LU's long trailing updates, A·H, Q^T A): per stage one thread issues
// the 2-D tensor copies (cp.async.bulk.tensor, SASS UTMALDG) of both operand tiles, 16 doubles =
// one 128-byte swizzle span per box, completing on one mbarrier per stage (expect_tx = the
// stage's bytes, zero-filled edges included). The fragment reads apply the swizzle's XOR (the
// K-major A operand at the minimum two wavefronts, the N- / M-major ones at four: DMMA, not shared
// memory, bounds the loop). The threads issue only fragment loads and DMMAs. Split-K over
// blockIdx.z: slice z covers [z kchunk, (z+1) kchunk) (kchunk a multiple of 32) and writes its own
// C panel (C + z cstride). Same tile and k order as k_dgemm: bit-identical results.
template <int BM, int BN, int WM, int WN, bool AKM, bool BKMJ, int MINB, int TM_NSTAGE>
__global__ void __launch_bounds__(WM* WN * 32, MINB)
    k_dgemm_tm(uint64_t M, uint64_t N, uint64_t K, double alpha, const __grid_constant__ CUtensorMap tmA,
               const __grid_constant__ CUtensorMap tmB, double beta, double* __restrict__ C, uint64_t ldc,
               uint64_t kchunk, uint64_t cstride) {
    using T = TmCfg<BM, BN, WM, WN, AKM, BKMJ, TM_NSTAGE>;
    extern __shared__ __align__(16) unsigned char smem_tm[];
    __shared__ __align__(8) uint64_t full[TM_NSTAGE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, t = lane & 3;
    const int ntn = static_cast<int>((N + BN - 1) / BN);
    const int ntiles = ntn * static_cast<int>((M + BM - 1) / BM);
    uint64_t kz0 = 0, kz = K;
    if (gridDim.z > 1) {
        kz0 = blockIdx.z * kchunk;
        kz = kz0 < K ? (K - kz0 < kchunk ? K - kz0 : kchunk) : 0;
        C += blockIdx.z * cstride;
    }
    const int ktiles = static_cast<int>((kz + TM_BK - 1) / TM_BK);
    const uint32_t base = (s_addr(smem_tm) + 1023u) & ~1023u;
    unsigned char* gbase = smem_tm + (base - s_addr(smem_tm));
    if (tid == 0) {
        for (int s2 = 0; s2 < TM_NSTAGE; ++s2)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&full[s2])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    __syncthreads();
    auto issue = [&](int s2, int kt, int m0, int n0) { // thread 0
        const uint32_t mb = s_addr(&full[s2]);
        const uint32_t st = base + static_cast<uint32_t>(s2 * T::STAGE);
        const int k0 = static_cast<int>(kz0) + kt * TM_BK;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(T::STAGE) : "memory");
#pragma unroll
        for (int q = 0; q < T::A_BOXES; ++q) {
            const int c0 = AKM ? k0 + 16 * q : m0 + 16 * q, c1 = AKM ? m0 : k0;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(st + q * T::A_BOX_BYTES), "l"(&tmA), "r"(c0), "r"(c1), "r"(mb)
                         : "memory");
        }
#pragma unroll
        for (int q = 0; q < T::B_BOXES; ++q) {
            const int c0 = BKMJ ? k0 + 16 * q : n0 + 16 * q, c1 = BKMJ ? n0 : k0;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(st + T::A_BYTES + q * T::B_BOX_BYTES), "l"(&tmB), "r"(c0), "r"(c1), "r"(mb)
                         : "memory");
        }
    };
    // Tiles: one per CTA, or a persistent loop when the grid was capped (the LU's trailing update
    // leaves SMs to the panel path). `it0` counts the k-tiles this CTA consumed: stage it % 2,
    // parity (it / 2) & 1 across tiles. The next tile's first stages are issued before the
    // epilogue: those stages were last read two k-tiles back, before the last loop barrier.
    int tile = static_cast<int>(blockIdx.x);
    if (tid == 0 && tile < ntiles)
        for (int s2 = 0; s2 < TM_NSTAGE - 1 && s2 < ktiles; ++s2)
            issue(s2, s2, (tile / ntn) * BM, (tile % ntn) * BN);
    int it0 = 0;
    for (; tile < ntiles; tile += static_cast<int>(gridDim.x)) {
        const int m0 = (tile / ntn) * BM, n0 = (tile % ntn) * BN;
        double acc[T::MF][T::NF][2];
#pragma unroll
        for (int i = 0; i < T::MF; ++i)
#pragma unroll
            for (int j = 0; j < T::NF; ++j)
                acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kt = 0; kt < ktiles; ++kt) {
            const int it = it0 + kt, s2 = it % TM_NSTAGE;
            {
                const uint32_t mb = s_addr(&full[s2]), par = static_cast<uint32_t>((it / TM_NSTAGE) & 1);
                uint32_t done = 0;
                while (!done)
                    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                                 " selp.u32 %0, 1, 0, p;\n}"
                                 : "=r"(done)
                                 : "r"(mb), "r"(par)
                                 : "memory");
            }
            __syncthreads(); // every warp is done with the stage refilled next (read at it - 1)
            const int nk = kt + TM_NSTAGE - 1;
            if (tid == 0 && nk < ktiles)
                issue((it0 + nk) % TM_NSTAGE, nk, m0, n0);
            const unsigned char* st = gbase + s2 * T::STAGE;
#pragma unroll
            for (int kk = 0; kk < TM_BK; kk += 4) {
                double af[T::MF], bf[T::NF];
#pragma unroll
                for (int i = 0; i < T::MF; ++i)
                    af[i] = *reinterpret_cast<const double*>(st + T::a_off(wm * T::WTM + i * 8 + g, kk + t));
#pragma unroll
                for (int j = 0; j < T::NF; ++j)
                    bf[j] = *reinterpret_cast<const double*>(st + T::b_off(kk + t, wn * T::WTN + j * 8 + g));
#pragma unroll
                for (int i = 0; i < T::MF; ++i)
#pragma unroll
                    for (int j = 0; j < T::NF; ++j)
                        dmma(acc[i][j], af[i], bf[j]);
            }
        }
        it0 += ktiles;
        const int next = tile + static_cast<int>(gridDim.x);
        if (tid == 0 && next < ntiles)
            for (int s2 = 0; s2 < TM_NSTAGE - 1 && s2 < ktiles; ++s2)
                issue((it0 + s2) % TM_NSTAGE, s2, (next / ntn) * BM, (next % ntn) * BN);
#pragma unroll
        for (int i = 0; i < T::MF; ++i) {
            const uint64_t row = static_cast<uint64_t>(m0) + wm * T::WTM + i * 8 + g;
            if (row >= M)
                continue;
#pragma unroll
            for (int j = 0; j < T::NF; ++j) {
                const uint64_t col = static_cast<uint64_t>(n0) + wn * T::WTN + j * 8 + 2 * t;
                if (col >= N)
                    continue;
                double* cp = C + row * ldc + col;
                double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
                if (col + 1 < N) {
                    if (beta != 0.0) {
                        const double2 o = *reinterpret_cast<const double2*>(cp);
                        v0 = fma(beta, o.x, v0);
                        v1 = fma(beta, o.y, v1);
                    }
                    *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
                } else {
                    if (beta != 0.0)
                        v0 = fma(beta, cp[0], v0);
                    cp[0] = v0;
                }
            }
        }
    }
}

} // namespace

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// rows x cols row-major f64 (ld doubles), box box_rows x 16 doubles, 128-byte swizzle
bool make_tmap(CUtensorMap* tm, const double* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
    auto enc = tensor_map_encoder();
    if (!enc)
        return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {ld * sizeof(double)};
    const cuuint32_t box[2] = {16, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

// true when the TMA kernel took the product. op(A): M x K, K-major (row-major M x K, ld lda) or
// M-major (A stored K x M, ld lda); B: K x N row-major (ld ldb).
template <int BM, int BN, int WM, int WN, bool AKM, int MINB, int NST = 2, bool BKMJ = false>
bool launch_tm(uint64_t M, uint64_t N, uint64_t K, double alpha, const double* A, uint64_t lda, const double* B,
               uint64_t ldb, double beta, double* C, uint64_t ldc, const Split& sp) {
    using T = TmCfg<BM, BN, WM, WN, AKM, BKMJ, NST>;
    CUtensorMap ta, tb;
    const bool ok = AKM ? make_tmap(&ta, A, M, K, lda, BM) : make_tmap(&ta, A, K, M, lda, TM_BK);
    if (!ok || !(BKMJ ? make_tmap(&tb, B, N, K, ldb, BN) : make_tmap(&tb, B, K, N, ldb, TM_BK)))
        return false;
    auto kern = k_dgemm_tm<BM, BN, WM, WN, AKM, BKMJ, MINB, NST>;
    static bool configured[16] = {};
    const int dev = ctx().device & 15;
    if (!configured[dev]) {
        RL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(T::SMEM)));
        configured[dev] = true;
    }
    // one CTA per tile (the kernel's tile loop also serves grids capped below the tile count)
    const uint64_t tiles = static_cast<uint64_t>(cdiv(N, BN)) * cdiv(M, BM);
    dim3 grid(static_cast<unsigned>(tiles), 1, sp.splits);
    kern<<<grid, T::NT, T::SMEM, stream()>>>(M, N, K, alpha, ta, tb, beta, C, ldc, sp.kchunk, sp.cstride);
    RL_LAUNCHED();
    return true;
}

template <int BM, int BN, int WM, int WN, bool AK, bool BKM, int VEC, int NSTAGE, int MINB = 1, int BKT = BK>
void launch(uint64_t M, uint64_t N, uint64_t K, double alpha, const double* A, uint64_t lda,
            const double* B, uint64_t ldb, double beta, double* C, uint64_t ldc, const Split& sp) {
    using G = Cfg<BM, BN, WM, WN, AK, BKM, VEC, NSTAGE, BKT>;
    auto kern = k_dgemm<BM, BN, WM, WN, AK, BKM, VEC, NSTAGE, MINB, BKT>;
    static bool configured[16] = {};
    int dev = ctx().device & 15;
    if (!configured[dev]) {
        RL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(G::kSmem)));
        configured[dev] = true;
    }
    dim3 grid(cdiv(N, BN), cdiv(M, BM), sp.splits);
    kern<<<grid, G::NT, G::kSmem, stream()>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sp.kchunk,
                                              sp.cstride);
    RL_LAUNCHED();
}

template <bool AK, bool BKM, int VEC>
void dispatch_shape(uint64_t M, uint64_t N, uint64_t Kfull, double alpha, const double* A, uint64_t lda,
                    const double* B, uint64_t ldb, double beta, double* C, uint64_t ldc, const Split& sp) {
    const int sms = ctx().sms;
    // shape decisions see one split-K slice: K per CTA and CTAs over all slices
    const uint64_t K = sp.splits > 1 ? sp.kchunk : Kfull;
    const uint64_t z = static_cast<uint64_t>(sp.splits);
    uint64_t big_tiles = static_cast<uint64_t>(cdiv(M, 128)) * cdiv(N, 128);
    static const int force = getenv("RL_GEMM_FORCE") ? atoi(getenv("RL_GEMM_FORCE")) : -1; // dev sweeps
    if (force == 0)
        return launch<128, 128, 2, 4, AK, BKM, VEC, 4>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    if (force == 1)
        return launch<128, 64, 4, 2, AK, BKM, VEC, 3, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    if (force == 3)
        return launch<64, 64, 2, 2, AK, BKM, VEC, 4, 4>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    if (force == 6)
        return launch<128, 64, 4, 2, AK, BKM, VEC, 2, 2, 32>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    if (force == 4)
        return launch<64, 32, 4, 2, AK, BKM, VEC, 4>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    // rho+ = 64 + 8 (the range finder's sketch width): 72-wide tiles instead of a 64-wide
    // tile plus a mostly empty second one (Y = A H, Q = Y R^-1: N = 72; Q^T A: M = 72; the
    // Gram Y^T Y: both)
    if (M > 64 && M <= 72 && N > 64 && N <= 72)
        return launch<72, 72, 3, 3, AK, BKM, VEC, 3, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    // the range finder's skinny products: TMA-fed 128 x 80 (A H) / 80 x 128 (Q^T A) tiles, the
    // column / row edge past 72 zero-filled by the copy engine (split-K slices of 32-multiples)
    static const bool no_tma_rf = getenv("RL_GEMM_NO_TMA") != nullptr;
    // both operands K-major (A H with H^T stored rho x n; Q^T A with Q^T stored rho x m): the
    // 72-wide operand is ONE 72 x 16 box per 16 k (no padding to 80) and its fragment reads hit
    // the two-wavefront minimum like A's
    const bool tm_kk = !no_tma_rf && VEC == 2 && AK && (sp.splits == 1 || sp.kchunk % 32 == 0) &&
                       ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    // A H: 128 x 72 tiles (8 warps, 2 per SM; 128 row tiles x 2 K slices at m = 16384: each
    // busy SM at the DMMA probe's rate, 20 SMs idle).  Measured and not kept: 112 x 72 tiles of
    // 7 warps (147 x 2 CTAs fill the GPU, but 7 warps load the four SM sub-partitions unevenly:
    // 334 us against 297) and 64 x 72 tiles of 4 warps at 3 CTAs per SM (2.9 waves of 5 K
    // slices: 302 us).  Q^T A: 72 x 128 tiles (32 column tiles x 9 slices = 288 of 296 slots).
    if (BKM && N > 64 && N <= 72 && N % 2 == 0 && tm_kk &&
        launch_tm<128, 72, 8, 1, true, 2, 2, true>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp))
        return;
    if (!BKM && M > 64 && M <= 72 && N > 72 && tm_kk &&
        launch_tm<72, 128, 1, 8, true, 2, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp))
        return;
    const bool tm_ok = !no_tma_rf && VEC == 2 && !BKM && (sp.splits == 1 || sp.kchunk % 32 == 0) &&
                       ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    if (N > 64 && N <= 72) {
        if (AK && tm_ok && launch_tm<128, 80, 4, 2, true, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp))
            return;
        return launch<128, 72, 4, 3, AK, BKM, VEC, 3, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    }
    if (M > 64 && M <= 72) {
        if (!AK && tm_ok && launch_tm<80, 128, 2, 4, false, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp))
            return;
        return launch<72, 128, 3, 4, AK, BKM, VEC, 3, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    }
    if (N > 64 && z * cdiv(M, 128) * cdiv(N, 64) >= 2ULL * sms && K >= kLongK) {
        // two CTAs per SM (128x64 tiles, <= 128 regs): one CTA's prologue / C epilogue
        // overlaps the other's DMMA loop.  Long K: K-tile 32 in 2 stages (217 KB for the two
        // CTAs), half the k-tile barriers of a 16 x 3 ring: A*G 8192^3 33.41 -> 32.76 ms
        // (DMMA pipe 89.5 -> 91.3% active).  (Feeding the padded tiles with per-row TMA bulk
        // copies, 160 x 256-512 B per stage from one warp, measured 48.7 ms: the copy engine
        // is not built for that many small transfers.)  Full tiles of A K-major x B N-major go
        // through 2-D tensor copies with the 128-byte swizzle instead (k_dgemm_tm);
        // RL_GEMM_NO_TMA=1 keeps the cp.async ring.
        static const bool no_tma = getenv("RL_GEMM_NO_TMA") != nullptr;
        const bool tm_full = AK && !BKM && VEC == 2 && sp.splits == 1 && !no_tma && M % 128 == 0 && N % 64 == 0 &&
                             Kfull % 32 == 0 &&
                             ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
        if (tm_full && launch_tm<128, 64, 4, 2, true, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp))
            return;
        launch<128, 64, 4, 2, AK, BKM, VEC, 2, 2, 32>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    }
    else if (N > 64 && z * cdiv(M, 128) * cdiv(N, 64) >= 2ULL * sms)
        // short K (the LU's trailing updates): K-tile 16 in 3 stages keeps the pipeline full
        // over few k-tiles (7680^2 x 256: 1044 vs 1100 us with the 32 x 2 ring)
        launch<128, 64, 4, 2, AK, BKM, VEC, 3, 2>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    else if (N > 32 && z * cdiv(M, 128) * cdiv(N, 64) >= static_cast<uint64_t>(sms))
        launch<128, 64, 4, 2, AK, BKM, VEC, 4>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
    // small grids (the LU's diagonal-block and strip updates): a 128 x 64 tile would leave
    // most SMs idle while each CTA runs a long DMMA chain; 64 x 32 tiles spread the same
    // work over 4x the CTAs (tools/gemm_graph.py: 128^2 x 256 27 -> ~9 us)
    else
        launch<64, 32, 4, 2, AK, BKM, VEC, 4>(M, N, Kfull, alpha, A, lda, B, ldb, beta, C, ldc, sp);
}

} // namespace

namespace {

void gemm_any(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, double alpha, const double* a,
              uint64_t lda, const double* b, uint64_t ldb, double beta, double* c, uint64_t ldc,
              const Split& sp) {
    // operand contiguous extents must be even and 16-byte aligned for 16-byte copies
    bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
                     reinterpret_cast<uintptr_t>(c)) & 15) == 0 &&
                   lda % 2 == 0 && ldb % 2 == 0 && ldc % 2 == 0 && (ta ? m : k) % 2 == 0 &&
                   (tb ? k : n) % 2 == 0;
    // AK = A is K-major (row-major m x k, not transposed); BKM = B is K-major (tb)
#define RL_GEMM_CASE(AK_, BK_)                                                          \
    if (aligned)                                                                        \
        dispatch_shape<AK_, BK_, 2>(m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, sp);     \
    else                                                                                \
        dispatch_shape<AK_, BK_, 1>(m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, sp);
    if (!ta && !tb) {
        RL_GEMM_CASE(true, false)
    } else if (!ta && tb) {
        RL_GEMM_CASE(true, true)
    } else if (ta && !tb) {
        RL_GEMM_CASE(false, false)
    } else {
        RL_GEMM_CASE(false, true)
    }
#undef RL_GEMM_CASE
}

// Matrix-vector shapes (N <= 8 right-hand sides, op(A) row-major M x K, B K x N row-major): one
// warp per row of A, lanes striding K (coalesced 256-byte reads of the row), two accumulation
// chains per column, a fixed shuffle tree: HBM-bound instead of a DMMA tile 7/8 empty
// (G y, A y for one right-hand side at n = 256: 10 -> ~3 us).
constexpr int GV_MAXN = 8;
__global__ void __launch_bounds__(256) k_gemv_rows(uint64_t M, int N, uint64_t K, double alpha, const double* __restrict__ A,
                                                   uint64_t lda, const double* __restrict__ B, uint64_t ldb, double beta,
                                                   double* C, uint64_t ldc) {
    const uint64_t row = blockIdx.x * 8ULL + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= M)
        return;
    const double* ar = A + row * lda;
    double acc[GV_MAXN][2];
#pragma unroll
    for (int c = 0; c < GV_MAXN; ++c)
        acc[c][0] = acc[c][1] = 0.0;
    uint64_t kk = lane;
    for (; kk + 32 < K; kk += 64) {
        const double a0 = __ldg(ar + kk), a1 = __ldg(ar + kk + 32);
        const double* b0 = B + kk * ldb;
        const double* b1 = B + (kk + 32) * ldb;
#pragma unroll
        for (int c = 0; c < GV_MAXN; ++c)
            if (c < N) {
                acc[c][0] = fma(a0, __ldg(b0 + c), acc[c][0]);
                acc[c][1] = fma(a1, __ldg(b1 + c), acc[c][1]);
            }
    }
    if (kk < K) {
        const double a0 = __ldg(ar + kk);
#pragma unroll
        for (int c = 0; c < GV_MAXN; ++c)
            if (c < N)
                acc[c][0] = fma(a0, __ldg(B + kk * ldb + c), acc[c][0]);
    }
#pragma unroll
    for (int c = 0; c < GV_MAXN; ++c) {
        if (c >= N)
            break;
        double v = acc[c][0] + acc[c][1];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == c) {
            double* cp = C + row * ldc + c;
            v *= alpha;
            *cp = beta != 0.0 ? fma(beta, *cp, v) : v;
        }
    }
}

} // namespace

void gemm(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, double alpha, const double* a,
          uint64_t lda, const double* b, uint64_t ldb, double beta, double* c, uint64_t ldc) {
    if (m == 0 || n == 0)
        return;
    if (k == 0) {
        // C = beta C
        gemm(false, false, m, n, 1, 0.0, c, ldc, c, ldc, beta, c, ldc);
        return;
    }
    if (!ta && !tb && n <= static_cast<uint64_t>(GV_MAXN) && k >= 64) {
        k_gemv_rows<<<cdiv(m, 8), 256, 0, stream()>>>(m, static_cast<int>(n), k, alpha, a, lda, b, ldb, beta, c, ldc);
        RL_LAUNCHED();
        return;
    }
    gemm_any(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, Split{});
}

// CTA tiles dispatch_shape uses for an M x N output (split planning).
uint64_t gemm_tiles(uint64_t M, uint64_t N) {
    if (M > 64 && M <= 72 && N > 64 && N <= 72)
        return 1;
    if (N > 64 && N <= 72)
        return cdiv(M, 128);
    if (M > 64 && M <= 72)
        return cdiv(N, 128);
    return static_cast<uint64_t>(cdiv(M, 64)) * cdiv(N, 32);
}

// One launch, `splits` K-slices of `kchunk` (multiple of 16): slice z writes
// op(A)[:, slice] op(B)[slice, :] to parts + z m n (ld n).
void gemm_splitk_parts(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, const double* a, uint64_t lda,
                       const double* b, uint64_t ldb, double* parts, int splits, uint64_t kchunk) {
    if (m == 0 || n == 0)
        return;
    Split sp;
    sp.splits = splits;
    sp.kchunk = kchunk;
    sp.cstride = m * n;
    gemm_any(ta, tb, m, n, k, 1.0, a, lda, b, ldb, 0.0, parts, n, sp);
}

} // namespace rl

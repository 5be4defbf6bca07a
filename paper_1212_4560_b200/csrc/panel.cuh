// Two-level blocked panel kernels of the blocked GENP (genp.cu): the 128-wide
// diagonal block, the panel TRSMs and the block solves are processed in 16-wide
// sub-panels.  Inside a sub-panel every row (or column) runs its 16-step substitution
// out of registers with no synchronisation; everything outside the sub-panel is a
// DMMA (mma.sync.m8n8k4.f64) update between shared-memory tiles.  This keeps the
// sequential chains short and puts ~7/8 of the panel flops on the FP64 tensor path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rl {
namespace panel {

constexpr int SB = 16;       // sub-panel width
constexpr int NBK = 128;     // block size
constexpr int PT = NBK + 4;  // smem pitch (doubles): row stride = 32 B mod 128 B (conflict-free frags)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// C[0:M, 0:N] -= A[0:M, 0:16] * B[0:16, 0:N] on shared-memory tiles (row-major, pitches
// lda/ldb/ldc).  M, N multiples of 8.  Warps take 8x8 output fragments round-robin;
// skip_corner leaves the top-left 16 x 16 block out.
__device__ __forceinline__ void smem_update16(double* C, int ldc, const double* A, int lda, const double* B,
                                              int ldb, int M, int N, int warp, int nwarps, int lane,
                                              bool skip_corner = false) {
    const int g = lane >> 2, t = lane & 3;
    const int fm = M >> 3, fn = N >> 3;
    // fragment f = (mi, nj) row-major, walked with an incremental (mi, nj) (no divisions)
    int mi = warp / fn, nj = warp - mi * fn;
    for (int f = warp; f < fm * fn; f += nwarps) {
        const int m0 = mi << 3, n0 = nj << 3;
        nj += nwarps;
        while (nj >= fn) {
            nj -= fn;
            ++mi;
        }
        if (skip_corner && m0 < 16 && n0 < 16) // the 16 x 16 corner is updated by its own warp
            continue;
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int k0 = 0; k0 < SB; k0 += 4)
            dmma(acc, A[(m0 + g) * lda + k0 + t], B[(k0 + t) * ldb + n0 + g]);
        double* c = C + (m0 + g) * ldc + n0 + 2 * t;
        c[0] -= acc[0];
        c[1] -= acc[1];
    }
}

// Global -> shared tile copy of an R x C tile with batched (8-deep) independent loads.
// Elements outside the valid vr x vc extent get fill(i, j); keep(i, j) false stores fill.
template <int R, int C, int THREADS, typename Keep, typename Fill>
__device__ __forceinline__ void load_tile(double* s, int sp, const double* g, uint64_t ld, int vr, int vc,
                                          Keep keep, Fill fill) {
    constexpr int TOTAL = R * C;
    constexpr int D = (TOTAL % (THREADS * 16) == 0) ? 16 : 8; // loads in flight per thread
    static_assert(TOTAL % (THREADS * D) == 0, "tile must split into 8-deep batches");
    const int tid = threadIdx.x;
#pragma unroll 1
    for (int base = 0; base < TOTAL; base += THREADS * D) {
        double v[D];
#pragma unroll
        for (int u = 0; u < D; ++u) {
            const int e = base + u * THREADS + tid;
            const int i = e / C, j = e % C;
            const bool ok = i < vr && j < vc;
            v[u] = ok ? g[static_cast<uint64_t>(i) * ld + j] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < D; ++u) {
            const int e = base + u * THREADS + tid;
            const int i = e / C, j = e % C;
            const bool ok = i < vr && j < vc;
            s[i * sp + j] = (ok && keep(i, j)) ? v[u] : fill(i, j);
        }
    }
}

// Global -> shared copy of an R x C tile with cp.async (8-byte copies, all in flight at
// once, no register staging): elements outside vr x vc or with keep(i, j) false are
// zero-filled without reading global memory.  Caller: cp_async_wait_all() + __syncthreads().
template <int R, int C, int THREADS, typename Keep>
__device__ __forceinline__ void load_tile_async(double* s, int sp, const double* g, uint64_t ld, int vr, int vc,
                                                Keep keep) {
    const int tid = threadIdx.x;
#pragma unroll 4
    for (int e = tid; e < R * C; e += THREADS) {
        const int i = e / C, j = e % C;
        const bool ok = i < vr && j < vc && keep(i, j);
        const double* src = ok ? g + static_cast<uint64_t>(i) * ld + j : g;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(s + i * sp + j));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0));
    }
    asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Shared -> global store of the valid vr x vc part of an R x C tile (8-deep batches).
template <int R, int C, int THREADS>
__device__ __forceinline__ void store_tile(double* g, uint64_t ld, const double* s, int sp, int vr, int vc) {
    constexpr int TOTAL = R * C;
    static_assert(TOTAL % (THREADS * 8) == 0, "tile must split into 8-deep batches");
    const int tid = threadIdx.x;
#pragma unroll 4
    for (int base = 0; base < TOTAL; base += THREADS) {
        const int e = base + tid;
        const int i = e / C, j = e % C;
        if (i < vr && j < vc)
            g[static_cast<uint64_t>(i) * ld + j] = s[i * sp + j];
    }
}

} // namespace panel
} // namespace rl

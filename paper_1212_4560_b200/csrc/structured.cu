// K7/K8 + structured products: multipliers applied matrix-free (or densified where
// the reference itself is dense).
//
//  * circulant  C(i,j) = c[(i-j) mod n]      (structured.cpp:70-83 densify; the
//    reference applies it by FFT, structured.cpp:132-189)
//  * householder_sign I - u v^T/(u^T v)       (random_gen.cpp:125-143, singular)
//  * NEW Householder pair H1 H2, H_i = I - (2/n) u_i u_i^T, u_i in {+-1}^n:
//      A H = A - t1 u1^T - t2 u2^T,  t1 = (2/n) A u1,  t2 = (2/n)(A u2 - t1 (u1^T u2))
//    pass 1 streams A once for both row dots (k_hh2_rowdots), pass 2 streams A once
//    more and writes A H (k_hh2_apply): 3 n^2 doubles of HBM traffic, coalesced
//    double2 loads, no tensor work — an HBM-bound kernel.
//  * NEW sparse +-1 S (nnz per column): (A S)(i,j) = sum_t s_jt A(i, r_jt), a row-tiled
//    gather (row of A in shared memory, index/sign table from L2): 2 n^2 doubles.
#include <cstdio>
#include <cstdlib>

#include "rl_internal.cuh"

namespace rl {

namespace {

__global__ void k_circulant_dense(uint64_t n, const double* c, double* out) {
    uint64_t total = n * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = e / n, j = e % n;
        out[e] = c[(i + n - j) % n];
    }
}

// T(i, j) = col[i - j] (i >= j) or row[j - i] (j > i) with g = col[0..n-1], row[1..n-1]
// (random_structured's draw order, random_gen.cpp:94-103; densify, structured.cpp:70-83)
__global__ void k_toeplitz_dense(uint64_t n, const double* g, double* out) {
    uint64_t total = n * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = e / n, j = e % n;
        out[e] = i >= j ? g[i - j] : g[n - 1 + (j - i)];
    }
}

__global__ void k_rank1_dense(uint64_t n, const double* u, const double* v, double inv_uv, double* out) {
    uint64_t total = n * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = e / n, j = e % n;
        out[e] = (i == j ? 1.0 : 0.0) - u[i] * v[j] * inv_uv;
    }
}

// per row i: w1 = A(i,:) u1, w2 = A(i,:) u2   (one warp per row, double2 loads)
__global__ void k_hh2_rowdots(uint64_t n, const double* __restrict__ a, uint64_t lda,
                              const double* __restrict__ u1, const double* __restrict__ u2,
                              double* __restrict__ w1, double* __restrict__ w2) {
    const int lane = threadIdx.x & 31;
    uint64_t row = blockIdx.x * static_cast<uint64_t>(blockDim.x / 32) + (threadIdx.x >> 5);
    if (row >= n)
        return;
    const double* r = a + row * lda;
    double s1 = 0.0, s2 = 0.0;
    for (uint64_t j = 2 * lane; j + 1 < n; j += 64) {
        double2 v = *reinterpret_cast<const double2*>(r + j);
        double2 a1 = *reinterpret_cast<const double2*>(u1 + j);
        double2 a2 = *reinterpret_cast<const double2*>(u2 + j);
        s1 = fma(v.x, a1.x, fma(v.y, a1.y, s1));
        s2 = fma(v.x, a2.x, fma(v.y, a2.y, s2));
    }
    if ((n & 1) && lane == 0) {
        s1 = fma(r[n - 1], u1[n - 1], s1);
        s2 = fma(r[n - 1], u2[n - 1], s2);
    }
    for (int off = 16; off > 0; off >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, off);
        s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    if (lane == 0) {
        w1[row] = s1;
        w2[row] = s2;
    }
}

// out = A - t1 u1^T - t2 u2^T with t1 = c w1, t2 = c (w2 - t1 s12)
__global__ void k_hh2_apply(uint64_t n, const double* __restrict__ a, uint64_t lda,
                            const double* __restrict__ u1, const double* __restrict__ u2,
                            const double* __restrict__ w1, const double* __restrict__ w2, double s12,
                            double c, double* __restrict__ out, uint64_t ldo) {
    const uint64_t half = (n + 1) / 2;
    const uint64_t total = n * half;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = e / half, j = 2 * (e % half);
        double t1 = c * w1[i];
        double t2 = c * (w2[i] - t1 * s12);
        if (j + 1 < n) {
            double2 v = *reinterpret_cast<const double2*>(a + i * lda + j);
            double2 p = *reinterpret_cast<const double2*>(u1 + j);
            double2 q = *reinterpret_cast<const double2*>(u2 + j);
            double2 o;
            o.x = (v.x - t1 * p.x) - t2 * q.x;
            o.y = (v.y - t1 * p.y) - t2 * q.y;
            *reinterpret_cast<double2*>(out + i * ldo + j) = o;
        } else {
            out[i * ldo + j] = (a[i * lda + j] - t1 * u1[j]) - t2 * u2[j];
        }
    }
}

// One pass over A for the Householder pair (config 5, north_star "stream A once"): the row dots
// w1 = A(i,:) u1, w2 = A(i,:) u2 need the whole row before any output of that row can be written,
// so the row is held on chip. Persistent CTAs (one per SM, 1024 threads): row r arrives in shared
// memory by one TMA bulk copy (cp.async.bulk + mbarrier), every thread moves its 2K values into
// registers, thread 0 immediately launches row r + grid into the freed buffer, and the dots,
// the two-level reduction (warp shuffles, one partial per warp in shared memory summed in a fixed
// order by every thread) and the streaming stores of row r overlap that copy. HBM traffic: A read once,
// the output written once = 2 n^2 8 bytes. u1, u2 (+-1) stay in registers for the whole kernel.
__device__ __forceinline__ uint32_t hh_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
constexpr int HH_THREADS = 1024, HH_K = 8; // 1024 threads x 8 double2 = rows of up to 16384
__global__ void __launch_bounds__(HH_THREADS, 1)
    k_hh2_onepass(uint64_t n, const double* __restrict__ a, uint64_t lda, const double* __restrict__ u1,
                  const double* __restrict__ u2, double s12, const double* __restrict__ s12p, double c,
                  double* __restrict__ out, uint64_t ldo) {
    if (s12p)
        s12 = *s12p;
    extern __shared__ __align__(16) double hh_row[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ double red1[HH_THREADS / 32], red2[HH_THREADS / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t nn = static_cast<uint32_t>(n);
    // u1, u2 are +-1 vectors: one sign bit per element (bit 2k + h: element 2(t + k 1024) + h)
    uint32_t m1 = 0, m2 = 0;
#pragma unroll
    for (int k = 0; k < HH_K; ++k) {
        const uint32_t j = 2u * static_cast<uint32_t>(t + k * HH_THREADS);
        if (j < nn) {
            const double2 q1 = *reinterpret_cast<const double2*>(u1 + j);
            const double2 q2 = *reinterpret_cast<const double2*>(u2 + j);
            m1 |= (q1.x < 0.0 ? 1u : 0u) << (2 * k) | (q1.y < 0.0 ? 1u : 0u) << (2 * k + 1);
            m2 |= (q2.x < 0.0 ? 1u : 0u) << (2 * k) | (q2.y < 0.0 ? 1u : 0u) << (2 * k + 1);
        }
    }
    auto sgn = [](uint32_t m, int b, double x) { return ((m >> b) & 1u) ? -x : x; }; // x * u (exact)
    const uint32_t bytes = static_cast<uint32_t>(n * sizeof(double));
    const uint32_t mb = hh_smem(&bar);
    auto issue = [&](uint64_t r) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         hh_smem(hh_row)),
                     "l"(a + r * lda), "r"(bytes), "r"(mb)
                     : "memory");
    };
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (blockIdx.x < n)
            issue(blockIdx.x);
    }
    __syncthreads();
    uint32_t phase = 0;
    for (uint64_t r = blockIdx.x; r < n; r += gridDim.x) {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                         " selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(done)
                         : "r"(mb), "r"(phase)
                         : "memory");
        phase ^= 1u;
        double2 v[HH_K];
#pragma unroll
        for (int k = 0; k < HH_K; ++k) {
            const uint32_t j = 2u * static_cast<uint32_t>(t + k * HH_THREADS);
            v[k] = j < nn ? *reinterpret_cast<const double2*>(hh_row + j) : make_double2(0.0, 0.0);
        }
        __syncthreads(); // the buffer is free: the next row streams in under this row's work
        if (t == 0 && r + gridDim.x < n)
            issue(r + gridDim.x);
        double d1 = 0.0, d2 = 0.0;
#pragma unroll
        for (int k = 0; k < HH_K; ++k) { // d += v u, u = +-1 (the products are exact)
            d1 = (d1 + sgn(m1, 2 * k, v[k].x)) + sgn(m1, 2 * k + 1, v[k].y);
            d2 = (d2 + sgn(m2, 2 * k, v[k].x)) + sgn(m2, 2 * k + 1, v[k].y);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            d1 += __shfl_xor_sync(0xffffffffu, d1, off);
            d2 += __shfl_xor_sync(0xffffffffu, d2, off);
        }
        if (lane == 0) {
            red1[warp] = d1;
            red2[warp] = d2;
        }
        __syncthreads();
        double w1 = 0.0, w2 = 0.0;
#pragma unroll 8
        for (int q = 0; q < HH_THREADS / 32; ++q) {
            w1 += red1[q];
            w2 += red2[q];
        }
        const double t1 = c * w1;
        const double t2 = c * (w2 - t1 * s12);
        double* orow = out + r * ldo;
#pragma unroll
        for (int k = 0; k < HH_K; ++k) {
            const uint32_t j = 2u * static_cast<uint32_t>(t + k * HH_THREADS);
            if (j < nn) {
                double2 o;
                o.x = (v[k].x - sgn(m1, 2 * k, t1)) - sgn(m2, 2 * k, t2);
                o.y = (v[k].y - sgn(m1, 2 * k + 1, t1)) - sgn(m2, 2 * k + 1, t2);
                __stcs(reinterpret_cast<double2*>(orow + j), o);
            }
        }
    }
}

// x = H1 (H2 y) for nrhs columns (ld nrhs): one CTA per column (small work)
__global__ void k_hh2_vec(uint64_t n, uint64_t nrhs, const double* u1, const double* u2, const double* y,
                          double* x) {
    const uint64_t col = blockIdx.x;
    __shared__ double red[32];
    __shared__ double dsh;
    const double c = 2.0 / static_cast<double>(n);
    auto block_dot = [&](const double* u, const double* v) -> double {
        double s = 0.0;
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
            s = fma(u[i], v[i * nrhs + col], s);
        for (int off = 16; off > 0; off >>= 1)
            s += __shfl_xor_sync(0xffffffffu, s, off);
        if ((threadIdx.x & 31) == 0)
            red[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (unsigned k = 0; k < blockDim.x / 32; ++k)
                t += red[k];
            dsh = t;
        }
        __syncthreads();
        double r = dsh;
        __syncthreads();
        return r;
    };
    double d2 = block_dot(u2, y);
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
        x[i * nrhs + col] = y[i * nrhs + col] - (c * d2) * u2[i];
    __syncthreads();
    double d1 = block_dot(u1, x);
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
        x[i * nrhs + col] = x[i * nrhs + col] - (c * d1) * u1[i];
}

// The sparse product's defined summation order (oracle rlo_pairwise): sum(v[0:h]) +
// sum(v[h:m]), h = ceil(m / 2); for nnz = 4 that is (v0 + v1) + (v2 + v3).
__device__ __forceinline__ double pairwise8(const double (&v)[8], int m) {
    switch (m) {
    case 1: return v[0];
    case 2: return v[0] + v[1];
    case 3: return (v[0] + v[1]) + v[2];
    case 4: return (v[0] + v[1]) + (v[2] + v[3]);
    case 5: return ((v[0] + v[1]) + v[2]) + (v[3] + v[4]);
    case 6: return ((v[0] + v[1]) + v[2]) + ((v[3] + v[4]) + v[5]);
    case 7: return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + v[6]);
    default: return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    }
}

// (A S)(i,j) = sum_t s_jt A(i, r_jt): one CTA per row block of RB rows staged in smem
constexpr int SP_THREADS = 512;
__global__ void __launch_bounds__(SP_THREADS) k_sparse_right(uint64_t n, int nnz, const double* __restrict__ a,
                                                             uint64_t lda, const int32_t* __restrict__ rows,
                                                             const double* __restrict__ signs,
                                                             double* __restrict__ out, uint64_t ldo,
                                                             int rb) {
    extern __shared__ double srow[]; // rb x n
    const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * rb;
    const int nr = static_cast<int>((n - r0) < static_cast<uint64_t>(rb) ? (n - r0) : rb);
    for (int r = 0; r < nr; ++r) {
        const double* src = a + (r0 + r) * lda;
        for (uint64_t j = threadIdx.x; j < n; j += SP_THREADS)
            srow[r * n + j] = src[j];
    }
    __syncthreads();
    for (uint64_t j = threadIdx.x; j < n; j += SP_THREADS) {
        int32_t idx[8];
        double sg[8];
        for (int t = 0; t < nnz; ++t) {
            idx[t] = rows[j * nnz + t];
            sg[t] = signs[j * nnz + t];
        }
        for (int r = 0; r < nr; ++r) {
            double v[8];
            for (int t = 0; t < nnz; ++t)
                v[t] = sg[t] * srow[r * n + idx[t]];
            out[(r0 + r) * ldo + j] = pairwise8(v, nnz);
        }
    }
}

// The same product for nnz = 4, n <= 16384 (config 5): persistent CTAs (one per SM) keep the
// whole S in registers — per thread 32 output columns x 4 (row, sign) entries packed as 16-bit
// (15-bit row | sign bit), two per register — and stream the rows of A through shared memory,
// so every byte of A and of the output crosses HBM once and S is read once per CTA (the kernel
// above re-reads S from L2 for every row: 786 KB per 128 KB row).  Same summation order.
constexpr int SP4_THREADS = 512, SP4_Q = 32, SP4_CH = 1024, SP4_SLOTS = 27, SP4_GROUP = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Gather plan for k_sparse_right4.  A warp's 64-bit shared loads are served per half-warp;
// 16 random row indices collide on the 16 eight-byte bank pairs (index mod 16) in ~3.1
// wavefronts per half-warp instead of 1.  The gathers can be regrouped without touching the
// result: inside each (warp, q) group of 32 output columns, the lanes l and l ^ 16 may trade
// columns (the store stays inside the same 256 B), and a column's four entries may be gathered
// in any order of the symmetry group of (v0 + v1) + (v2 + v3) (swap inside either pair, swap
// the pairs: 8 orders, all giving the same bits).  One thread per group chooses, pair by pair,
// the trade and the orders that add the fewest same-bank-pair collisions to what the group
// already placed (~2.1 instead of ~3.1 wavefronts per half-warp, 33% fewer).  Slot (q, t) = 4 x
// 16 bits in gather order: row (14 bits) | trade bit (entry 2 only) | sign.
constexpr int SPP_GROUPS = 4; // groups per 32-thread CTA; lane o = t & 7 evaluates gather order o
__global__ void __launch_bounds__(32) k_sparse_plan(uint64_t n, const int32_t* __restrict__ rows,
                                                    const double* __restrict__ signs, uint32_t* __restrict__ plan) {
    __shared__ uint8_t cnt[SPP_GROUPS][2 * 4 * 16]; // [half][gather][bank pair] per group
    __shared__ uint8_t cls[SPP_GROUPS][32 * 4];     // bank pair of entry e of the group's column c
    __shared__ uint8_t pick[SPP_GROUPS][32];        // lane l: column << 3 | order
    const int t = threadIdx.x, g = t >> 3, o = t & 7;
    const int grp = blockIdx.x * SPP_GROUPS + g; // (warp, q) = (grp % 16, grp / 16)
    const int warp = grp % (SP4_THREADS / 32), q = grp / (SP4_THREADS / 32);
    const uint64_t col0 = static_cast<uint64_t>(q) * SP4_THREADS + warp * 32;
    for (int c = o; c < 2 * 4 * 16; c += 8)
        cnt[g][c] = 0;
    for (int c = o; c < 32 * 4; c += 8)
        cls[g][c] = (col0 + c / 4 < n) ? static_cast<uint8_t>(rows[col0 * 4 + c] & 15) : 0;
    __syncwarp();
    // gather order o (bit 0: swap v0/v1, bit 1: swap v2/v3, bit 2: swap the pairs): gather u
    // reads entry ord(o, u) — the 8 orders that leave (v0 + v1) + (v2 + v3) unchanged
    auto ord = [](uint32_t oo, int u) -> uint32_t {
        const uint32_t e = static_cast<uint32_t>(u) ^ ((oo & 4u) >> 1);
        return e ^ ((e < 2u ? oo : (oo >> 1)) & 1u);
    };
    // (collisions added << 3) | order, minimised over the group's 8 lanes
    auto best_ord = [&](int c, int h, bool valid) -> uint32_t {
        uint32_t v = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v += cnt[g][(h * 4 + u) * 16 + cls[g][c * 4 + ord(o, u)]];
        uint32_t b = valid ? (v << 3) | static_cast<uint32_t>(o) : 0u;
#pragma unroll
        for (int m = 1; m < 8; m <<= 1)
            b = min(b, __shfl_xor_sync(0xffffffffu, b, m));
        return b;
    };
    auto place = [&](int c, int h, uint32_t oo, int d, bool valid) { // lanes 0..3: gather u = lane
        __syncwarp();
        if (valid && o < 4) {
            const int i = (h * 4 + o) * 16 + cls[g][c * 4 + ord(oo, o)];
            cnt[g][i] = static_cast<uint8_t>(cnt[g][i] + d);
        }
        __syncwarp();
    };
    for (int p = 0; p < 16; ++p) {
        uint32_t o_lo[2] = {0, 0}, o_hi[2] = {0, 0}, cost[2] = {0, 0};
        const bool two = col0 + p + 16 < n; // a pair with a missing column keeps its lanes
        for (int sw = 0; sw < 2; ++sw) {     // uniform trip count: shuffles need the whole warp
            const int c_lo = sw ? p + 16 : p, c_hi = sw ? p : p + 16; // column of lane p / p + 16
            const bool ok = sw == 0 || two;
            const bool v_lo = ok && col0 + c_lo < n, v_hi = ok && col0 + c_hi < n;
            uint32_t b = best_ord(c_lo, 0, v_lo);
            o_lo[sw] = b & 7u;
            uint32_t v = b >> 3;
            place(c_lo, 0, o_lo[sw], 1, v_lo);
            b = best_ord(c_hi, 1, v_hi);
            o_hi[sw] = b & 7u;
            v += b >> 3;
            place(c_lo, 0, o_lo[sw], -1, v_lo);
            cost[sw] = ok ? v : 0xffffffffu;
        }
        const int sw = cost[1] < cost[0] ? 1 : 0;
        const int c_lo = sw ? p + 16 : p, c_hi = sw ? p : p + 16;
        place(c_lo, 0, o_lo[sw], 1, col0 + c_lo < n);
        place(c_hi, 1, o_hi[sw], 1, col0 + c_hi < n);
        if (o == 0) {
            pick[g][p] = static_cast<uint8_t>(c_lo << 3 | o_lo[sw]);
            pick[g][p + 16] = static_cast<uint8_t>(c_hi << 3 | o_hi[sw]);
        }
    }
    __syncwarp();
    // slots: lane l computes column pick[l] >> 3, gathering its entries in order pick[l] & 7
    for (int l = o; l < 32; l += 8) {
        const int c = pick[g][l] >> 3;
        const uint32_t oo = pick[g][l] & 7u;
        const uint64_t j = col0 + c;
        uint32_t e[4] = {0, 0, 0, 0};
        if (j < n)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t x = j * 4 + ord(oo, u);
                e[u] = static_cast<uint32_t>(rows[x]) | (signs[x] < 0.0 ? 0x8000u : 0u);
            }
        e[2] |= static_cast<uint32_t>(c != l) << 14; // lane trade bit
        const uint64_t slot = static_cast<uint64_t>(q) * SP4_THREADS + warp * 32 + l;
        reinterpret_cast<uint2*>(plan)[slot] = make_uint2(e[0] | (e[1] << 16), e[2] | (e[3] << 16));
    }
}

template <bool PLAN>
__global__ void __launch_bounds__(SP4_THREADS, 1) k_sparse_right4(uint64_t n, const double* __restrict__ a,
                                                                  uint64_t lda, const int32_t* __restrict__ rows,
                                                                  const double* __restrict__ signs,
                                                                  const uint32_t* __restrict__ plan,
                                                                  double* __restrict__ out, uint64_t ldo) {
    extern __shared__ __align__(128) double srow[]; // SP4_SLOTS x SP4_CH ring + barriers
    const int t = threadIdx.x;
#ifdef RL_SP_TRACE
    long long tr0 = clock64(), tr_wait = 0, tr_comp = 0, tr_sync = 0;
#endif
    // slot q: 4 x 16-bit entries, row (14 bits) | spare | sign; in draw order, or (PLAN) in
    // the plan's gather order with the rotation / lane trade in the spare bits
    uint32_t pk[SP4_Q * 2];
    if constexpr (PLAN) {
        const uint2* pl = reinterpret_cast<const uint2*>(plan);
#pragma unroll
        for (int q = 0; q < SP4_Q; ++q) {
            const uint2 v = pl[q * SP4_THREADS + t];
            pk[2 * q] = v.x;
            pk[2 * q + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < SP4_Q; ++q) {
            const uint64_t j = t + static_cast<uint64_t>(q) * SP4_THREADS;
            uint32_t e[4] = {0, 0, 0, 0};
            if (j < n)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    e[u] = static_cast<uint32_t>(rows[j * 4 + u]) | (signs[j * 4 + u] < 0.0 ? 0x8000u : 0u);
            pk[2 * q] = e[0] | (e[1] << 16);
            pk[2 * q + 1] = e[2] | (e[3] << 16);
        }
    }
    // Shared memory holds [head buffer 0 | tail | head buffer 1], SP4_SLOTS = 2 H + T chunks of
    // SP4_CH doubles.  Row r's first H chunks (its head) arrive by bulk async copies (TMA
    // engine, one mbarrier per chunk) into head buffer r & 1 while row r - 1 is gathered; its
    // last T chunks (the tail, prefetched into L2 one row ahead) are copied by all threads
    // with cp.async into the single tail buffer once row r - 1 is done.  Row r's element col
    // sits at col (even r: head 0 then tail) or, for odd r, at col + (H + T) SP4_CH when it is
    // in the head, so only a short L2 read of each row's tail is exposed.
    double* sm = srow;
    constexpr uint32_t H = (SP4_SLOTS - 5) / 2, T = SP4_SLOTS - 2 * H; // 11 + 5 + 11 for n = 16384
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SP4_SLOTS * SP4_CH); // 2 H head barriers
    const uint32_t cpr = static_cast<uint32_t>((n + SP4_CH - 1) / SP4_CH); // chunks per row (<= H + T)
    const uint32_t nh = cpr < H ? cpr : H;                                 // head chunks per row
    const uint32_t my_rows = blockIdx.x < n ? static_cast<uint32_t>((n - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
    if (t == 0) {
        for (uint32_t s = 0; s < 2 * H; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + s)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto row_ptr = [&](uint32_t r) { return a + (blockIdx.x + static_cast<uint64_t>(r) * gridDim.x) * lda; };
    auto chunk_bytes = [&](uint32_t c) {
        const uint64_t left = n - static_cast<uint64_t>(c) * SP4_CH;
        return static_cast<uint32_t>(left < SP4_CH ? left : SP4_CH) * 8u;
    };
    auto issue_head = [&](uint32_t r) { // thread 0: row r's head into buffer r & 1
        const double* src = row_ptr(r);
        const uint32_t buf = (r & 1u) ? H + T : 0u;
        for (uint32_t c = 0; c < nh; ++c) {
            const uint32_t bytes = chunk_bytes(c), mb = smem_u32(bar + (r & 1u) * H + c);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sm + (buf + c) * SP4_CH)),
                "l"(src + static_cast<uint64_t>(c) * SP4_CH), "r"(bytes), "r"(mb)
                : "memory");
        }
        for (uint32_t c = nh; c < cpr; ++c) // the tail: into L2 now, into shared memory a row later
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + static_cast<uint64_t>(c) * SP4_CH),
                         "r"(chunk_bytes(c))
                         : "memory");
    };
    const uint32_t tail_elems = n > nh * SP4_CH ? static_cast<uint32_t>(n) - nh * SP4_CH : 0u; // even (n even)
    if (t == 0 && my_rows > 0)
        issue_head(0);
    for (uint32_t r = 0; r < my_rows; ++r) {
#ifdef RL_SP_TRACE
        long long ta = clock64();
        tr_sync += ta - tr0;
#endif
        if (t == 0 && r + 1 < my_rows)
            issue_head(r + 1); // buffer (r + 1) & 1 was freed by row r - 1
        {                      // row r's tail: 16-byte cp.async by every thread
            const double* src = row_ptr(r) + nh * SP4_CH;
            for (uint32_t e = 2 * t; e < tail_elems; e += 2 * SP4_THREADS)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + (H * SP4_CH + e))),
                             "l"(src + e)
                             : "memory");
            asm volatile("cp.async.commit_group;\n cp.async.wait_all;" ::: "memory");
        }
        for (uint32_t c = 0; c < nh; ++c) { // row r's head
            const uint32_t mb = smem_u32(bar + (r & 1u) * H + c), par = (r >> 1) & 1u;
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                             " selp.u32 %0, 1, 0, p;\n}"
                             : "=r"(done)
                             : "r"(mb), "r"(par)
                             : "memory");
        }
        __syncthreads(); // every thread's tail pieces are visible
#ifdef RL_SP_TRACE
        long long tb = clock64();
        tr_wait += tb - ta;
#endif
        // element col of row r at col + (col < head_end ? head_off : 0)
        const uint32_t head_end = nh * SP4_CH, head_off = (r & 1u) ? (H + T) * SP4_CH : 0u;
        uint32_t tr; // t, opaque to the compiler: keeps the 32 column offsets from being hoisted into registers
        asm volatile("mov.u32 %0, %1;" : "=r"(tr) : "r"(static_cast<uint32_t>(t)));
        const uint64_t i = blockIdx.x + static_cast<uint64_t>(r) * gridDim.x;
        double* orow = out + i * ldo;
#pragma unroll
        for (int q = 0; q < SP4_Q; ++q) {
            uint32_t p0, p1; // opaque copies: keeps the compiler from hoisting the unpacked entries (spills)
            asm volatile("mov.b32 %0, %1;" : "=r"(p0) : "r"(pk[2 * q]));
            asm volatile("mov.b32 %0, %1;" : "=r"(p1) : "r"(pk[2 * q + 1]));
            // PLAN: lane pair (l, l ^ 16) may trade columns
            const uint32_t j = static_cast<uint32_t>(q) * SP4_THREADS +
                               (PLAN ? (tr & ~31u) + ((tr & 31u) ^ ((p1 >> 10) & 16u)) : tr);
            if (j < n) {
                double y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t w = u < 2 ? p0 : p1;
                    const uint32_t e = (u & 1) ? (w >> 16) : (w & 0xffffu);
                    const uint32_t col = e & 0x3fffu;
                    const double x = sm[col + (col < head_end ? head_off : 0u)];
                    // s_jt = +-1: flip the sign bit (the reference's s_jt * A(i, r_jt) is exact)
                    const uint32_t sbit = (u & 1) ? (w & 0x80000000u) : ((w << 16) & 0x80000000u);
                    y[u] = __hiloint2double(__double2hiint(x) ^ static_cast<int>(sbit), __double2loint(x));
                }
                // the defined order (v0 + v1) + (v2 + v3); the plan's gather orders all preserve it
                const double s = (y[0] + y[1]) + (y[2] + y[3]);
                __stcs(orow + j, s);
            }
            if (q % SP4_GROUP == SP4_GROUP - 1)
                asm volatile("" ::: "memory"); // bounds the compiler's load hoisting (register budget)
        }
#ifdef RL_SP_TRACE
        tr0 = clock64();
        tr_comp += tr0 - tb;
#endif
        __syncthreads(); // row r's slots are free
    }
#ifdef RL_SP_TRACE
    if (t % 32 == 0) { // per warp: cycles waiting for the row, gathering, at the row barrier
        atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<uint32_t*>(plan)), static_cast<unsigned long long>(tr_wait));
        atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<uint32_t*>(plan)) + 1, static_cast<unsigned long long>(tr_comp));
        atomicAdd(reinterpret_cast<unsigned long long*>(const_cast<uint32_t*>(plan)) + 2, static_cast<unsigned long long>(tr_sync));
    }
#endif
}

// x = S y (nrhs columns, ld nrhs) via the row-sorted transpose: x[i] = sum over
// entries (j,t) with r_jt = i, in ascending j (deterministic).
__global__ void k_sparse_vec(uint64_t n, uint64_t nrhs, const int32_t* row_ptr, const int32_t* col_j,
                             const double* col_s, const double* y, double* x) {
    uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (e >= n * nrhs)
        return;
    uint64_t i = e / nrhs, c = e % nrhs;
    double s = 0.0;
    for (int p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
        s += col_s[p] * y[static_cast<uint64_t>(col_j[p]) * nrhs + c];
    x[e] = s;
}

// counting sort of the (row, j) entries by row, stable in j: one thread per row scans
// nothing; instead: counts per row, exclusive scan (single CTA), then placement in j
// order by a single thread per row-chunk.  n <= 2^24 entries total is ample here.
__global__ void k_sparse_count(uint64_t n, int nnz, const int32_t* rows, int32_t* counts) {
    uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (e < n * nnz)
        atomicAdd(&counts[rows[e]], 1);
}

__global__ void k_scan_single(uint64_t n, int32_t* counts, int32_t* row_ptr) {
    // single CTA exclusive scan over n counts
    __shared__ int32_t carry;
    if (threadIdx.x == 0)
        carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < n; base += blockDim.x) {
        uint64_t i = base + threadIdx.x;
        int32_t v = i < n ? counts[i] : 0;
        // warp inclusive scan
        int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        int32_t x = v;
        for (int off = 1; off < 32; off <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off)
                x += y;
        }
        __shared__ int32_t wsum[32];
        if (lane == 31)
            wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int32_t s = (lane < static_cast<int>(blockDim.x / 32)) ? wsum[lane] : 0;
            for (int off = 1; off < 32; off <<= 1) {
                int32_t y = __shfl_up_sync(0xffffffffu, s, off);
                if (lane >= off)
                    s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        int32_t incl = x + (wid > 0 ? wsum[wid - 1] : 0) + carry;
        if (i < n)
            row_ptr[i] = incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1)
            carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0)
        row_ptr[n] = carry;
}

// stable placement: thread per row i walks... (O(n * nnz) total via per-entry rank)
// rank of entry (j,t) within its row = number of entries (j',t') with same row and j' < j.
// Computed by a second pass in j order per row bucket using a per-row cursor, serial in j:
// we parallelise over rows by having each row's entries found through a scan of columns
// in blocks; simpler and deterministic: one thread per column j computes its slots with
// atomics on the cursor, then a per-row insertion sort restores ascending j.
__global__ void k_sparse_place(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                               const int32_t* row_ptr, int32_t* cursor, int32_t* col_j,
                               double* col_s) {
    uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (e >= n * nnz)
        return;
    int32_t r = rows[e];
    int32_t pos = row_ptr[r] + atomicAdd(&cursor[r], 1);
    col_j[pos] = static_cast<int32_t>(e / nnz);
    col_s[pos] = signs[e];
}

__global__ void k_sparse_sortrows(uint64_t n, const int32_t* row_ptr, int32_t* col_j, double* col_s) {
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n)
        return;
    int b = row_ptr[i], e = row_ptr[i + 1];
    for (int p = b + 1; p < e; ++p) {
        int32_t kj = col_j[p];
        double ks = col_s[p];
        int q = p - 1;
        while (q >= b && col_j[q] > kj) {
            col_j[q + 1] = col_j[q];
            col_s[q + 1] = col_s[q];
            --q;
        }
        col_j[q + 1] = kj;
        col_s[q + 1] = ks;
    }
}

__global__ void k_circ_vec(uint64_t n, uint64_t nrhs, const double* c, const double* z, double* y) {
    uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (e >= n * nrhs)
        return;
    uint64_t i = e / nrhs, col = e % nrhs;
    double s = 0.0;
    for (uint64_t j = 0; j < n; ++j)
        s = fma(c[(i + n - j) % n], z[j * nrhs + col], s);
    y[e] = s;
}

unsigned grid_for(uint64_t total, int threads) {
    return static_cast<unsigned>(std::min<uint64_t>((total + threads - 1) / threads, 148ULL * 32));
}

} // namespace

void circulant_dense_dev(uint64_t n, const double* c, double* out) {
    k_circulant_dense<<<grid_for(n * n, 256), 256, 0, stream()>>>(n, c, out);
    RL_LAUNCHED();
}

void toeplitz_dense_dev(uint64_t n, const double* g, double* out) {
    k_toeplitz_dense<<<grid_for(n * n, 256), 256, 0, stream()>>>(n, g, out);
    RL_LAUNCHED();
}

void rank1_dense_dev(uint64_t n, const double* u, const double* v, double inv_uv, double* out) {
    k_rank1_dense<<<grid_for(n * n, 256), 256, 0, stream()>>>(n, u, v, inv_uv, out);
    RL_LAUNCHED();
}

// out = A H1 H2 (out may alias a); s12 = u1^T u2 (exact integer, host-computed)
// u1^T u2 of two +-1 vectors on the device (an exact integer: any summation order gives it)
__global__ void k_dot_pm1(uint64_t n, const double* __restrict__ u1, const double* __restrict__ u2, double* out) {
    __shared__ double part[32];
    double sacc = 0.0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
        sacc += u1[i] * u2[i];
    for (int o = 16; o > 0; o >>= 1)
        sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if ((threadIdx.x & 31) == 0)
        part[threadIdx.x >> 5] = sacc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (unsigned w = 0; w < blockDim.x / 32; ++w)
            t += part[w];
        *out = t;
    }
}

void hh2_apply_right_dev(uint64_t n, const double* a, uint64_t lda, const double* u1, const double* u2,
                         double s12, double* out, uint64_t ldo, const double* s12p) {
    if (n <= 2ull * HH_THREADS * HH_K && n % 2 == 0 && lda % 2 == 0 && ldo % 2 == 0 &&
        ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
        const size_t smem = n * sizeof(double);
        static bool attr[16] = {};
        if (!attr[ctx().device & 15]) {
            RL_CUDA(cudaFuncSetAttribute(k_hh2_onepass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(2 * HH_THREADS * HH_K * sizeof(double))));
            attr[ctx().device & 15] = true;
        }
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, ctx().sms));
        k_hh2_onepass<<<grid, HH_THREADS, smem, stream()>>>(n, a, lda, u1, u2, s12, s12p,
                                                            2.0 / static_cast<double>(n), out, ldo);
        RL_LAUNCHED();
        return;
    }
    // rows longer than 16384 or unaligned: two passes (row dots, then the rank-2 update)
    if (s12p) {
        RL_CUDA(cudaMemcpyAsync(&s12, s12p, sizeof(double), cudaMemcpyDeviceToHost, stream()));
        RL_CUDA(cudaStreamSynchronize(stream()));
    }
    double* w = ws<double>(WS_SMALL, 2 * n);
    k_hh2_rowdots<<<cdiv(n, 8), 256, 0, stream()>>>(n, a, lda, u1, u2, w, w + n);
    RL_LAUNCHED();
    k_hh2_apply<<<grid_for(n * ((n + 1) / 2), 256), 256, 0, stream()>>>(
        n, a, lda, u1, u2, w, w + n, s12, 2.0 / static_cast<double>(n), out, ldo);
    RL_LAUNCHED();
}

void dot_pm1_dev(uint64_t n, const double* u1, const double* u2, double* d_out) {
    k_dot_pm1<<<1, 1024, 0, stream()>>>(n, u1, u2, d_out);
    RL_LAUNCHED();
}

void hh2_apply_vec_dev(uint64_t n, uint64_t nrhs, const double* u1, const double* u2, const double* y,
                       double* x) {
    k_hh2_vec<<<static_cast<unsigned>(nrhs), 256, 0, stream()>>>(n, nrhs, u1, u2, y, x);
    RL_LAUNCHED();
}

void sparse_apply_right_dev(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                            const double* a, uint64_t lda, double* out, uint64_t ldo) {
    if (nnz == 4 && n <= static_cast<uint64_t>(SP4_THREADS) * SP4_Q && n % 2 == 0 && lda % 2 == 0 &&
        (reinterpret_cast<uintptr_t>(a) & 15) == 0) {
        constexpr size_t smem = SP4_SLOTS * SP4_CH * sizeof(double) + SP4_SLOTS * sizeof(uint64_t); // + barriers
        static bool attr[16] = {};
        if (!attr[ctx().device & 15]) {
            RL_CUDA(cudaFuncSetAttribute(k_sparse_right4<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            RL_CUDA(cudaFuncSetAttribute(k_sparse_right4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
            attr[ctx().device & 15] = true;
        }
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, ctx().sms));
        static const bool use_plan = [] {
            const char* e = getenv("RL_SPARSE_PLAN"); // 0: draw-order gathers (dev comparison)
            return e == nullptr || e[0] != '0';
        }();
        if (use_plan) {
            uint32_t* plan = ws<uint32_t>(WS_SPLAN, 2 * SP4_THREADS * SP4_Q);
            k_sparse_plan<<<SP4_THREADS / 32 * SP4_Q / SPP_GROUPS, 32, 0, stream()>>>(n, rows, signs, plan);
            RL_LAUNCHED();
#ifdef RL_SP_TRACE
            unsigned long long h0[3], h1[3];
            RL_CUDA(cudaMemcpyAsync(h0, plan, sizeof h0, cudaMemcpyDeviceToHost, stream()));
            RL_CUDA(cudaStreamSynchronize(stream()));
#endif
            k_sparse_right4<true><<<grid, SP4_THREADS, smem, stream()>>>(n, a, lda, rows, signs, plan, out, ldo);
#ifdef RL_SP_TRACE
            RL_CUDA(cudaMemcpyAsync(h1, plan, sizeof h1, cudaMemcpyDeviceToHost, stream()));
            RL_CUDA(cudaStreamSynchronize(stream()));
            const double warps = static_cast<double>(grid) * SP4_THREADS / 32 * (static_cast<double>(n) / grid);
            fprintf(stderr, "sparse trace (cycles per warp-row): wait %.0f gather %.0f barrier %.0f\n",
                    (h1[0] - h0[0]) / warps, (h1[1] - h0[1]) / warps, (h1[2] - h0[2]) / warps);
#endif
        } else {
            k_sparse_right4<false><<<grid, SP4_THREADS, smem, stream()>>>(n, a, lda, rows, signs, nullptr, out, ldo);
        }
        RL_LAUNCHED();
        return;
    }
    int rb = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(8, (160 * 1024) / (n * 8))));
    size_t smem = static_cast<size_t>(rb) * n * sizeof(double);
    if (smem > 200 * 1024)
        fail(RL_TOO_LARGE, "sparse apply: row does not fit in shared memory");
    RL_CUDA(cudaFuncSetAttribute(k_sparse_right, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(std::max<size_t>(smem, 48 * 1024))));
    k_sparse_right<<<cdiv(n, rb), SP_THREADS, smem, stream()>>>(n, nnz, a, lda, rows, signs, out, ldo, rb);
    RL_LAUNCHED();
}

// builds the transpose once; returns device pointers inside workspace slot WS_RF3
struct SparseT {
    int32_t* row_ptr;
    int32_t* col_j;
    double* col_s;
};

SparseT sparse_transpose_dev(uint64_t n, int nnz, const int32_t* rows, const double* signs) {
    uint64_t ne = n * nnz;
    char* base = ws<char>(WS_RF3, (n + 1) * 4 * 3 + ne * 4 + ne * 8 + 64);
    SparseT s;
    s.col_s = reinterpret_cast<double*>(base);
    s.col_j = reinterpret_cast<int32_t*>(base + ne * 8);
    s.row_ptr = s.col_j + ne;
    int32_t* counts = s.row_ptr + (n + 1);
    int32_t* cursor = counts + (n + 1);
    RL_CUDA(cudaMemsetAsync(counts, 0, (n + 1) * 4 * 2, stream()));
    k_sparse_count<<<cdiv(ne, 256), 256, 0, stream()>>>(n, nnz, rows, counts);
    RL_LAUNCHED();
    k_scan_single<<<1, 1024, 0, stream()>>>(n, counts, s.row_ptr);
    RL_LAUNCHED();
    k_sparse_place<<<cdiv(ne, 256), 256, 0, stream()>>>(n, nnz, rows, signs, s.row_ptr, cursor, s.col_j,
                                                        s.col_s);
    RL_LAUNCHED();
    k_sparse_sortrows<<<cdiv(n, 256), 256, 0, stream()>>>(n, s.row_ptr, s.col_j, s.col_s);
    RL_LAUNCHED();
    return s;
}

void sparse_apply_vec_dev(uint64_t n, uint64_t nrhs, const SparseT& s, const double* y, double* x) {
    k_sparse_vec<<<cdiv(n * nrhs, 256), 256, 0, stream()>>>(n, nrhs, s.row_ptr, s.col_j, s.col_s, y, x);
    RL_LAUNCHED();
}

void circ_apply_vec_dev(uint64_t n, uint64_t nrhs, const double* c, const double* z, double* y) {
    k_circ_vec<<<cdiv(n * nrhs, 256), 256, 0, stream()>>>(n, nrhs, c, z, y);
    RL_LAUNCHED();
}


// ------------------------------------------- circulant right product through the FFT ----
// out = A C for the circulant C(i, j) = c[(i - j) mod n] (random_structured CirculantSign /
// CirculantGaussian, random_gen.cpp:90-123; the reference applies it on the Right as
// (C^T A^T)^T with an FFT per column, genp.cpp:175-180 and structured.cpp:132-189).  Row r of
// A C is the cyclic cross-correlation of A(r, :) with c, so FFT(out_r) = FFT(A_r) . conj(FFT(c)).
// Matrix-free: O(n^2 log n) instead of the dense 2 n^3, one read of A and one write of A C.
//   * two real rows per complex sequence z = A_r + i A_{r+1} (c is real, so the imaginary
//     part carries row r + 1 through the product untouched);
//   * one persistent CTA per SM, a row pair's n complex values in shared memory (n <= 8192:
//     128 KB), padded by one element per n / 8 so that the bit-reversed load / store are
//     conflict-free;
//   * forward: bit-reversed load, decimation-in-time radix-2 stages fused two at a time in
//     registers (radix-2^2: the same operations, half the shared-memory passes); the product
//     with conj(FFT(c)) / n; inverse: decimation-in-frequency stages (natural in, bit-reversed
//     out), read back in bit-reversed order for a coalesced store;
//   * twiddles w^m = exp(-2 pi i m / n) from two small exact tables (w^m = hi[m / 64] lo[m % 64]).
namespace {

constexpr int CF_THREADS = 512, CF_L = 64, CF_MAXN = 8192;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

struct CfPlan {
    int n, lg, sh; // n = 2^lg; shared index i lives at i + (i >> 3) + (i >> sh)
    const double2* lo;
    const double2* hi;
    __device__ __forceinline__ int at(int i) const { return i + (i >> 3) + (i >> sh); }
    __device__ __forceinline__ int brev(int j) const { return static_cast<int>(__brev(static_cast<unsigned>(j)) >> (32 - lg)); }
    __device__ __forceinline__ double2 w(int m) const { return cmul(hi[m / CF_L], lo[m % CF_L]); } // exp(-2 pi i m / n)
};

// x (-i) exactly; x exp(-i pi / 4) (one rounding); x exp(-3 i pi / 4)
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 mul_w8(double2 a) {
    constexpr double r = 0.70710678118654752440;
    return make_double2((a.x + a.y) * r, (a.y - a.x) * r);
}
__device__ __forceinline__ double2 mul_w8_3(double2 a) { return mul_mi(mul_w8(a)); }

// One shared-memory pass of R fused DIT stages (spans h, 2h, ..., 2^(R-1) h) on a group of 2^R
// elements I_e = base + j + e h held in registers.  The stage with span S = 2^s h pairs e with
// e + 2^s (bit s of e clear) and twiddles by w^((j + (e mod 2^s) h) n / (2S)) =
// w^(j n / (2S)) exp(-2 pi i (e mod 2^s) / 2^(s+1)): one table twiddle per stage, the rest
// exact or one-rounding powers of the 8th root.
template <int R, bool MUL = false>
__device__ __forceinline__ void cf_dit_pass(double2* z, const CfPlan& P, int h, int g,
                                            const double2* __restrict__ chat = nullptr) {
    constexpr int E = 1 << R;
    const int n = P.n, j = g % h, i0 = (g / h) * E * h + j;
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e)
        v[e] = z[P.at(i0 + e * h)];
#pragma unroll
    for (int s = 0; s < R; ++s) {
        const int S = h << s;
        const double2 tw = P.w(j * (n / (2 * S)));
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e >> s) & 1)
                continue;
            const int r = e & ((1 << s) - 1);
            double2 t = cmul(tw, v[e + (1 << s)]);
            if (s == 1 && r == 1)
                t = mul_mi(t);
            if (s == 2 && r == 1)
                t = mul_w8(t);
            if (s == 2 && r == 2)
                t = mul_mi(t);
            if (s == 2 && r == 3)
                t = mul_w8_3(t);
            v[e + (1 << s)] = csub(v[e], t);
            v[e] = cadd(v[e], t);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
        z[P.at(i0 + e * h)] = MUL ? cmul(v[e], chat[i0 + e * h]) : v[e]; // MUL: the last pass, natural order
}

// The first three DIT stages (spans 1, 2, 4: every twiddle a power of the 8th root) straight
// from the two input rows: bit-reversed position 8g + e holds x[jj + brev3(e) n / 8] for
// g = brev(jj), so consecutive threads load consecutive columns (coalesced) and, thanks to the
// padding's i >> sh term, store to distinct bank groups.
__device__ __forceinline__ void cf_dit_first(double2* z, const CfPlan& P, int jj, const double* __restrict__ a0,
                                             const double* __restrict__ a1, bool two, int n_in) {
    const int n8 = P.n >> 3;
    const int g = static_cast<int>(__brev(static_cast<unsigned>(jj)) >> (35 - P.lg));
    double2 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int src = jj + ((((e & 1) << 2) | (e & 2) | ((e >> 2) & 1)) * n8); // brev3(e) n / 8
        const bool in = src < n_in; // columns past n_in are the zero padding of an embedding
        v[e] = make_double2(in ? __ldcs(a0 + src) : 0.0, (in && two) ? __ldcs(a1 + src) : 0.0);
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if ((e >> s) & 1)
                continue;
            const int r = e & ((1 << s) - 1);
            double2 t = v[e + (1 << s)];
            if (s == 1 && r == 1)
                t = mul_mi(t);
            if (s == 2 && r == 1)
                t = mul_w8(t);
            if (s == 2 && r == 2)
                t = mul_mi(t);
            if (s == 2 && r == 3)
                t = mul_w8_3(t);
            v[e + (1 << s)] = csub(v[e], t);
            v[e] = cadd(v[e], t);
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
        z[P.at(8 * g + e)] = v[e];
}

// The last three DIF stages (spans 4, 2, 1) straight to the two output rows: bit-reversed
// position 8g + e is natural column jj + brev3(e) n / 8 (coalesced stores).
__device__ __forceinline__ void cf_dif_last(const double2* z, const CfPlan& P, int jj, double* __restrict__ o0,
                                            double* __restrict__ o1, bool two, int n_out) {
    const int n8 = P.n >> 3;
    const int g = static_cast<int>(__brev(static_cast<unsigned>(jj)) >> (35 - P.lg));
    double2 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
        v[e] = z[P.at(8 * g + e)];
#pragma unroll
    for (int s = 2; s >= 0; --s) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if ((e >> s) & 1)
                continue;
            const int r = e & ((1 << s) - 1);
            double2 d = csub(v[e], v[e + (1 << s)]);
            v[e] = cadd(v[e], v[e + (1 << s)]);
            if (s == 1 && r == 1)
                d = cconj(mul_mi(cconj(d)));
            if (s == 2 && r == 1)
                d = cconj(mul_w8(cconj(d)));
            if (s == 2 && r == 2)
                d = cconj(mul_mi(cconj(d)));
            if (s == 2 && r == 3)
                d = cconj(mul_w8_3(cconj(d)));
            v[e + (1 << s)] = d;
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int dst = jj + ((((e & 1) << 2) | (e & 2) | ((e >> 2) & 1)) * n8);
        if (dst < n_out) {
            __stcs(o0 + dst, v[e].x);
            if (two)
                __stcs(o1 + dst, v[e].y);
        }
    }
}

// One pass of R fused DIF stages with conjugate twiddles (spans 2^(R-1) q, ..., q) on a group
// I_e = base + j + e q: the stage with span S = 2^s q pairs e with e + 2^s and multiplies the
// difference by conj(w)^((j + (e mod 2^s) q) n / (2S)).
template <int R>
__device__ __forceinline__ void cf_dif_pass(double2* z, const CfPlan& P, int q, int g) {
    constexpr int E = 1 << R;
    const int n = P.n, j = g % q, i0 = (g / q) * E * q + j;
    double2 v[E];
#pragma unroll
    for (int e = 0; e < E; ++e)
        v[e] = z[P.at(i0 + e * q)];
#pragma unroll
    for (int s = R - 1; s >= 0; --s) {
        const int S = q << s;
        const double2 tw = cconj(P.w(j * (n / (2 * S))));
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if ((e >> s) & 1)
                continue;
            const int r = e & ((1 << s) - 1);
            double2 d = csub(v[e], v[e + (1 << s)]);
            v[e] = cadd(v[e], v[e + (1 << s)]);
            d = cmul(d, tw);
            if (s == 1 && r == 1)
                d = cconj(mul_mi(cconj(d)));
            if (s == 2 && r == 1)
                d = cconj(mul_w8(cconj(d)));
            if (s == 2 && r == 2)
                d = cconj(mul_mi(cconj(d)));
            if (s == 2 && r == 3)
                d = cconj(mul_w8_3(cconj(d)));
            v[e + (1 << s)] = d;
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e)
        z[P.at(i0 + e * q)] = v[e];
}

// forward DFT (w = exp(-2 pi i / n)) in place: bit-reversed input, natural output; stages from
// span h0 on (h0 = 8 after cf_dit_first); MUL: multiply by chat in the last pass
template <bool MUL>
__device__ void cf_dit(double2* z, const CfPlan& P, int t, int h0, const double2* __restrict__ chat) {
    const int n = P.n;
    int h = h0, left = P.lg - (31 - __clz(h0));
    while (left > 0) {
        const int R = left >= 3 ? 3 : left;
        const bool last = left == R;
        if (R == 3) {
            for (int g = t; g < n / 8; g += CF_THREADS)
                last && MUL ? cf_dit_pass<3, true>(z, P, h, g, chat) : cf_dit_pass<3>(z, P, h, g);
        } else if (R == 2) {
            for (int g = t; g < n / 4; g += CF_THREADS)
                last && MUL ? cf_dit_pass<2, true>(z, P, h, g, chat) : cf_dit_pass<2>(z, P, h, g);
        } else {
            for (int g = t; g < n / 2; g += CF_THREADS)
                last && MUL ? cf_dit_pass<1, true>(z, P, h, g, chat) : cf_dit_pass<1>(z, P, h, g);
        }
        h <<= R;
        left -= R;
        __syncthreads();
    }
}

// inverse DFT without the 1/n (conjugate twiddles) in place: natural input, bit-reversed output;
// the lg mod 3 largest spans first, then radix-2^3 passes; stops `stop` stages early (3: the
// last pass is cf_dif_last)
__device__ void cf_dif_inv(double2* z, const CfPlan& P, int t, int stop) {
    const int n = P.n;
    int left = P.lg - stop, hs = n; // the remaining stages have spans below hs
    while (left > 0) {
        const int R = (left % 3) ? left % 3 : 3;
        const int q = hs >> R; // smallest span of this pass
        if (R == 3) {
            for (int g = t; g < n / 8; g += CF_THREADS)
                cf_dif_pass<3>(z, P, q, g);
        } else if (R == 2) {
            for (int g = t; g < n / 4; g += CF_THREADS)
                cf_dif_pass<2>(z, P, q, g);
        } else {
            for (int g = t; g < n / 2; g += CF_THREADS)
                cf_dif_pass<1>(z, P, q, g);
        }
        hs = q;
        left -= R;
        __syncthreads();
    }
}

__device__ CfPlan cf_setup(int n, double2* tabs, int t) {
    CfPlan P;
    P.n = n;
    P.lg = 31 - __clz(n);
    P.sh = P.lg - 3;
    double2* lo = tabs;
    double2* hi = tabs + CF_L;
    for (int m = t; m < CF_L; m += CF_THREADS) { // exact argument 2m/n: sincospi
        double s, c;
        sincospi(2.0 * m / n, &s, &c);
        lo[m] = make_double2(c, -s);
    }
    for (int m = t; m < n / (2 * CF_L) || m == 0; m += CF_THREADS) {
        if (m >= CF_L)
            break;
        double s, c;
        sincospi(2.0 * (static_cast<double>(m) * CF_L) / n, &s, &c);
        hi[m] = make_double2(c, -s);
    }
    P.lo = lo;
    P.hi = hi;
    return P;
}

// chat[k] = conj(FFT(c))_k / n  (one CTA)
__global__ void __launch_bounds__(CF_THREADS) k_circ_fft_prep(int n, const double* __restrict__ c,
                                                              double2* __restrict__ chat) {
    extern __shared__ double2 cz[];
    __shared__ double2 tabs[2 * CF_L];
    const int t = threadIdx.x;
    const CfPlan P = cf_setup(n, tabs, t);
    for (int j = t; j < n; j += CF_THREADS)
        cz[P.at(P.brev(j))] = make_double2(c[j], 0.0);
    __syncthreads();
    cf_dit<false>(cz, P, t, 1, nullptr);
    const double inv_n = 1.0 / n; // a power of two: exact
    for (int k = t; k < n; k += CF_THREADS) {
        const double2 v = cz[P.at(k)];
        chat[k] = make_double2(v.x * inv_n, -v.y * inv_n);
    }
}

// out (m x n, ldo) = A (m x n, lda) C; persistent CTAs over row pairs
// n: the transform length; rows of A hold n_in <= n columns (zero padding beyond), the first
// n_out <= n columns of the product are written (n_in = n_out = n for a circulant; n_in =
// n_out = the Toeplitz order inside its circulant embedding)
__global__ void __launch_bounds__(CF_THREADS, 1) k_circ_right_fft(uint64_t m, int n, int n_in, int n_out,
                                                                  const double* __restrict__ a,
                                                                  uint64_t lda, const double2* __restrict__ chat,
                                                                  double* __restrict__ out, uint64_t ldo) {
    extern __shared__ double2 cz[];
    __shared__ double2 tabs[2 * CF_L];
    const int t = threadIdx.x;
    const CfPlan P = cf_setup(n, tabs, t);
    __syncthreads();
    const uint64_t pairs = (m + 1) / 2;
    for (uint64_t pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
        const uint64_t r = 2 * pr;
        const bool two = r + 1 < m;
        const double* a0 = a + r * lda;
        const double* a1 = a0 + lda;
        // the next row pair into L2 while this one is transformed; the bulk prefetch needs a
        // 16-byte aligned start and a multiple of 16 bytes: the 16-byte window inside each row
        // (odd Toeplitz orders / pitches put every other row 8 bytes off)
        if (t == 0 && pr + gridDim.x < pairs) {
            const double* nx = a + 2 * (pr + gridDim.x) * lda;
            const uint64_t rows = (2 * (pr + gridDim.x) + 1 < m) ? 2 : 1;
            for (uint64_t q = 0; q < rows; ++q) {
                const uint64_t b0 = reinterpret_cast<uint64_t>(nx + q * lda);
                const uint64_t lo = (b0 + 15) & ~15ULL, hi = (b0 + n_in * sizeof(double)) & ~15ULL;
                if (hi > lo)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo),
                                 "r"(static_cast<uint32_t>(hi - lo))
                                 : "memory");
            }
        }
        for (int jj = t; jj < n / 8; jj += CF_THREADS)
            cf_dit_first(cz, P, jj, a0, a1, two, n_in);
        __syncthreads();
        cf_dit<true>(cz, P, t, 8, chat); // the rest of the forward transform, then x conj(FFT(c)) / n
        cf_dif_inv(cz, P, t, 3);
        double* o0 = out + r * ldo;
        double* o1 = o0 + ldo;
        for (int jj = t; jj < n / 8; jj += CF_THREADS)
            cf_dif_last(cz, P, jj, o0, o1, two, n_out);
        __syncthreads();
    }
}


// ---- n = 8192: register-resident radix 16 x 16 x 32 ----------------------------------------
// The general kernel above spends ~390 instructions per element (runtime index / twiddle
// arithmetic in every radix-8 pass, eight shared-memory round trips per transform pair: ncu
// 112 K warp instructions per row pair, issue-bound at 49%).  For n = 8192 = 16 * 16 * 32 the
// transform is a three-level four-step FFT whose sub-DFTs run in registers with compile-time
// twiddles; one table twiddle per element between levels (W^m = hi[m / 64] lo[m % 64],
// W = e^{-2 pi i / 8192}, sign-folded for m >= 4096):
//   P1  thread b < 512: x[512 a + b], a < 16 straight from the two rows (coalesced) -> DFT16
//       over a -> * W^{b c} -> slot (c, b)
//   P2  thread (c, f): slots (c, 32 e + f), e < 16 -> DFT16 over e -> * W_512^{f g} -> (c, 32 g + f)
//   P3  thread pair (c, g; gamma): the 32 contiguous slots (c, 32 g + f): a radix-2 step over
//       f's top bit (each thread its half gamma, * W_32^{beta gamma}) and DFT16 over beta give
//       X[c + 16 g + 256 (gamma + 2 delta)]; the product with conj(FFT(c)) / n; the adjoint
//       (inverse DFT16 over delta, the radix-2 recombination with the partner lane by
//       shuffles) back to the 32 slots
//   P2', P1'  the adjoints of P2 and P1 (conjugate twiddles, inverse DFT16), P1' storing the
//       two output rows (coalesced).
// Shared index i lives at i + (i >> 5): the P3 pairs' 16 groups (33 slots apart) hit distinct
// bank groups.  Four barriers per row pair, ~30 K warp instructions.
constexpr int F8_N = 8192, F8_T = 512;
__device__ __forceinline__ int f8_at(int i) { return i + (i >> 5); }

// (cos, sin)(2 pi j / 64), j < 32
__constant__ double2 kF8CS[32] = {
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

__host__ __device__ constexpr int br4(int m) { return ((m & 1) << 3) | ((m & 2) << 1) | ((m & 4) >> 1) | ((m & 8) >> 3); }

// v *= e^{-+2 pi i j / 64} (INV: +), j < 32 a compile-time constant after unrolling
template <bool INV>
__device__ __forceinline__ double2 f8_rot(double2 v, int j) {
    if (j == 0)
        return v;
    if (j == 16)
        return INV ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
    if (j == 8 || j == 24) { // (1 -+ i) / sqrt 2 and its mirror: two roundings
        constexpr double r = 0.70710678118654752440;
        const double2 u = INV ? make_double2(v.x - v.y, v.x + v.y) : make_double2(v.x + v.y, v.y - v.x);
        const double2 e = make_double2(u.x * r, u.y * r);
        return j == 8 ? e : (INV ? make_double2(-e.y, e.x) : make_double2(e.y, -e.x));
    }
    const double c = kF8CS[j].x, sn = INV ? kF8CS[j].y : -kF8CS[j].y;
    return make_double2(fma(v.x, c, -v.y * sn), fma(v.x, sn, v.y * c));
}

// In-place 16-point DFT (INV: e^{+}), decimation in frequency: natural order in, X[k] out at
// v[br4(k)]
template <bool INV>
__device__ __forceinline__ void f8_dft16(double2 (&v)[16]) {
#pragma unroll
    for (int st = 0; st < 4; ++st) {
        const int half = 8 >> st;
#pragma unroll
        for (int g = 0; g < 16; g += 2 * half)
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const int a = g + k, b = a + half;
                const double2 u = v[a], w = v[b];
                v[a] = cadd(u, w);
                v[b] = f8_rot<INV>(csub(u, w), (32 / half) * k);
            }
    }
}

struct F8Tw {
    const double2* lo; // W^j, j < 64
    const double2* hi; // W^{64 j}, j < 64
    __device__ __forceinline__ double2 w(int m) const { // W^m, 0 <= m < 8192
        const double2 r = cmul(hi[(m >> 6) & 63], lo[m & 63]);
        return (m & 4096) ? make_double2(-r.x, -r.y) : r;
    }
};

// chat (natural order) -> P3's thread order: chat_p[512 d + t] = chat[c + 16 g + 256 gam + 512 d]
// for thread t = 2 (16 c + g) + gam
__global__ void k_f8_perm(const double2* __restrict__ chat, double2* __restrict__ chat_p) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x; // < 8192
    const int d = e >> 9, t = e & 511, G = t >> 1, gam = t & 1;
    chat_p[e] = chat[(G >> 4) + 16 * (G & 15) + 256 * gam + 512 * d];
}

__global__ void __launch_bounds__(F8_T, 1) k_circ_fft8k(uint64_t m, const double* __restrict__ a, uint64_t lda,
                                                       const double2* __restrict__ chat, double* __restrict__ out,
                                                       uint64_t ldo) {
    extern __shared__ double2 sz[]; // f8_at(8192) slots
    __shared__ double2 tlo[64], thi[64];
    const int t = threadIdx.x;
    if (t < 64) {
        double sn, cs;
        sincospi(static_cast<double>(t) / 4096.0, &sn, &cs);
        tlo[t] = make_double2(cs, -sn);
        sincospi(static_cast<double>(t) / 64.0, &sn, &cs);
        thi[t] = make_double2(cs, -sn);
    }
    __syncthreads();
    const F8Tw T{tlo, thi};
    const uint64_t pairs = (m + 1) / 2;
    double* sd = reinterpret_cast<double*>(sz); // input staging: row 0 at [0, 8192), row 1 at [8192, 16384)
    // the row pair pr's two rows into the staging area (cp.async, 16 B each; a missing second
    // row is zero-filled) — issued under the previous pair's last pass
    auto stage = [&](uint64_t pr) {
        const uint64_t r0 = 2 * pr;
        const double* g0 = a + r0 * lda;
        const double* g1 = r0 + 1 < m ? g0 + lda : g0;
        const uint32_t nb1 = r0 + 1 < m ? 16u : 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = 2 * (t + 512 * q);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sd + e)), "l"(g0 + e)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sd + F8_N + e)), "l"(g1 + e),
                         "r"(nb1)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (t < 2 && pr + gridDim.x < pairs) { // and the pair after it into L2 (16-byte aligned window)
            const uint64_t nr = 2 * (pr + gridDim.x) + t;
            if (nr < m) {
                const uint64_t b0 = reinterpret_cast<uint64_t>(a + nr * lda);
                const uint64_t lo16 = (b0 + 15) & ~15ULL, hi16 = (b0 + F8_N * sizeof(double)) & ~15ULL;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo16),
                             "r"(static_cast<uint32_t>(hi16 - lo16))
                             : "memory");
            }
        }
    };
    if (blockIdx.x < pairs)
        stage(blockIdx.x);
    for (uint64_t pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
        const uint64_t r0 = 2 * pr;
        const bool two = r0 + 1 < m;
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads(); // this pair's rows are staged
        { // P1: thread b = t
            double2 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
                v[q] = make_double2(sd[512 * q + t], sd[F8_N + 512 * q + t]);
            __syncthreads(); // every staged value read before the slots are written
            f8_dft16<false>(v);
            // W^{t c}, c = 1.. by repeated products (a few ulps, below the FFT's own error); the
            // base is re-read each row pair so the power chains stay inside the loop
            const double2 w1 = T.w(t);
            double2 wc = w1;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                double2 y = v[br4(c)];
                if (c) {
                    y = cmul(y, wc);
                    wc = cmul(wc, w1);
                }
                sz[f8_at(c * 512 + t)] = y;
            }
        }
        __syncthreads();
        const int c2 = t >> 5, f2 = t & 31, base2 = c2 * 512 + f2;
        { // P2: thread (c, f)
            double2 v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
                v[e] = sz[f8_at(base2 + 32 * e)];
            f8_dft16<false>(v);
            const double2 w2 = T.w(16 * f2);
            double2 wg = w2; // W_512^{f g}
#pragma unroll
            for (int g = 0; g < 16; ++g) {
                double2 y = v[br4(g)];
                if (g) {
                    y = cmul(y, wg);
                    wg = cmul(wg, w2);
                }
                sz[f8_at(base2 + 32 * g)] = y;
            }
        }
        __syncthreads();
        { // P3: the pair (c, g) = t >> 1, gamma = t & 1
            const int G = t >> 1, gam = t & 1, c3 = G >> 4, g3 = G & 15, base3 = c3 * 512 + 32 * g3;
            double2 v[16];
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                const double2 u0 = sz[f8_at(base3 + b)], u1 = sz[f8_at(base3 + 16 + b)];
                double2 s = gam ? csub(u0, u1) : cadd(u0, u1);
                if (b) {
                    const double2 r = f8_rot<false>(s, 2 * b); // W_32^b = e^{-2 pi i (2b) / 64}
                    s = gam ? r : s;
                }
                v[b] = s;
            }
            __syncwarp();       // the pair's reads of its 32 slots are done before either writes
            f8_dft16<false>(v); // X[c + 16 g + 256 (gam + 2 d)] at v[br4(d)]
            double2 y[16];      // natural order in d for the inverse
#pragma unroll
            for (int d = 0; d < 16; ++d) // chat in P3's thread order (k_f8_perm): coalesced, L1-resident
                y[d] = cmul(v[br4(d)], chat[512 * d + t]);
            f8_dft16<true>(y); // A_gam[f'] at y[br4(f')]
#pragma unroll
            for (int q = 0; q < 16; ++q) { // out[16 gam + q] = A0[q] + (-1)^gam conj(W_32^q) A1[q]
                const double2 mine = y[br4(q)];
                const double2 other = make_double2(__shfl_xor_sync(0xffffffffu, mine.x, 1),
                                                   __shfl_xor_sync(0xffffffffu, mine.y, 1));
                const double2 a0v = gam ? other : mine, a1v = gam ? mine : other;
                const double2 t1 = f8_rot<true>(a1v, 2 * q); // conj(W_32^q) A1[q]
                sz[f8_at(base3 + 16 * gam + q)] = gam ? csub(a0v, t1) : cadd(a0v, t1);
            }
        }
        __syncthreads();
        { // P2': adjoint of P2
            double2 v[16];
            const double2 w2 = cconj(T.w(16 * f2));
            double2 wg = w2;
#pragma unroll
            for (int g = 0; g < 16; ++g) {
                double2 y = sz[f8_at(base2 + 32 * g)];
                if (g) {
                    y = cmul(y, wg);
                    wg = cmul(wg, w2);
                }
                v[g] = y;
            }
            f8_dft16<true>(v);
#pragma unroll
            for (int e = 0; e < 16; ++e)
                sz[f8_at(base2 + 32 * e)] = v[br4(e)];
        }
        __syncthreads();
        { // P1': adjoint of P1, straight to the two output rows
            double2 v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c)
                v[c] = sz[f8_at(c * 512 + t)];
            __syncthreads(); // the slots are free: the next pair's rows stream in under this pass
            if (pr + gridDim.x < pairs)
                stage(pr + gridDim.x);
            const double2 w1 = cconj(T.w(t));
            double2 wc = w1;
#pragma unroll
            for (int c = 1; c < 16; ++c) {
                v[c] = cmul(v[c], wc);
                wc = cmul(wc, w1);
            }
            f8_dft16<true>(v);
            double* o0 = out + r0 * ldo;
            double* o1 = o0 + ldo;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 x = v[br4(q)];
                __stcs(o0 + 512 * q + t, x.x);
                if (two)
                    __stcs(o1 + 512 * q + t, x.y);
            }
        }
    }
}
} // namespace

// true when the FFT path handles n: a power of two >= 64 (n <= 8192 in shared memory, larger n
// through the global-memory passes of circ_right_fft_large)
bool circ_fft_supported(uint64_t n) { return n >= 64 && (n & (n - 1)) == 0; }

void circ_right_fft_large(uint64_t m, uint64_t n, uint64_t n_in, uint64_t n_out, const double* c, const double* a,
                          uint64_t lda, double* out, uint64_t ldo);

// out = A C for the circulant with first column c; A, out m x n (out != A)
namespace {
// the transform for rows of n_in columns against the length-n circulant c (n a power of two)
void circ_right_fft_launch(uint64_t m, uint64_t n, uint64_t n_in, uint64_t n_out, const double* c, const double* a,
                           uint64_t lda, double* out, uint64_t ldo) {
    if (n > static_cast<uint64_t>(CF_MAXN)) {
        circ_right_fft_large(m, n, n_in, n_out, c, a, lda, out, ldo);
        return;
    }
    const size_t smem = (n + n / 8 + 8) * sizeof(double2);
    static bool attr[16] = {};
    if (!attr[ctx().device & 15]) {
        const int mx = static_cast<int>((CF_MAXN + CF_MAXN / 8 + 8) * sizeof(double2));
        RL_CUDA(cudaFuncSetAttribute(k_circ_fft_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        RL_CUDA(cudaFuncSetAttribute(k_circ_right_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        attr[ctx().device & 15] = true;
    }
    double2* chat = ws<double2>(WS_SPLAN, n); // k_sparse_plan's slot: not live at the same time
    k_circ_fft_prep<<<1, CF_THREADS, smem, stream()>>>(static_cast<int>(n), c, chat);
    RL_LAUNCHED();
    static const bool generic8k = getenv("RL_CIRC_FFT_GENERIC") != nullptr; // dev comparison
    const bool aligned = (lda % 2 == 0) && (reinterpret_cast<uintptr_t>(a) % 16 == 0); // cp.async 16 B
    if (n == static_cast<uint64_t>(F8_N) && n_in == n && n_out == n && aligned && !generic8k) {
        const size_t smem8 = static_cast<size_t>(F8_N + F8_N / 32) * sizeof(double2);
        static bool attr8[16] = {};
        if (!attr8[ctx().device & 15]) {
            RL_CUDA(cudaFuncSetAttribute(k_circ_fft8k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem8)));
            attr8[ctx().device & 15] = true;
        }
        const unsigned grid8 = static_cast<unsigned>(std::min<uint64_t>((m + 1) / 2, ctx().sms));
        double2* chat_p = ws<double2>(WS_FFT_C, F8_N);
        k_f8_perm<<<F8_N / 256, 256, 0, stream()>>>(chat, chat_p);
        RL_LAUNCHED();
        k_circ_fft8k<<<grid8, F8_T, smem8, stream()>>>(m, a, lda, chat_p, out, ldo);
        RL_LAUNCHED();
        return;
    }
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((m + 1) / 2, ctx().sms));
    k_circ_right_fft<<<grid, CF_THREADS, smem, stream()>>>(m, static_cast<int>(n), static_cast<int>(n_in),
                                                           static_cast<int>(n_out), a, lda, chat, out, ldo);
    RL_LAUNCHED();
}

// circulant embedding of the n x n Toeplitz (g = col[0..n-1], row[1..n-1]): c2[k] = col[k],
// c2[len - j] = row[j], zero elsewhere (structured.cpp:156-176)
__global__ void k_toeplitz_embed(uint64_t n, uint64_t len, const double* g, double* c2) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < len;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        c2[k] = k < n ? g[k] : (k > len - n ? g[n - 1 + (len - k)] : 0.0);
}

// x = T z (nrhs columns, ld nrhs), T(i, j) = col[i - j] / row[j - i], ascending j
__global__ void k_toeplitz_vec(uint64_t n, uint64_t nrhs, const double* g, const double* z, double* y) {
    uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (e >= n * nrhs)
        return;
    uint64_t i = e / nrhs, col = e % nrhs;
    double s = 0.0;
    for (uint64_t j = 0; j < n; ++j)
        s = fma(i >= j ? g[i - j] : g[n - 1 + (j - i)], z[j * nrhs + col], s);
    y[e] = s;
}
} // namespace

void circ_apply_right_fft_dev(uint64_t m, uint64_t n, const double* c, const double* a, uint64_t lda, double* out,
                              uint64_t ldo) {
    circ_right_fft_launch(m, n, n, n, c, a, lda, out, ldo);
}

// the embedding length when the Toeplitz product can take the FFT path (0 otherwise)
uint64_t toeplitz_fft_len(uint64_t n) {
    uint64_t len = 1;
    while (len < 2 * n - 1)
        len <<= 1;
    return (n >= 2 && circ_fft_supported(len)) ? len : 0;
}

// out = A T for the n x n Toeplitz of g (A, out m x n, out != A): the circulant of order
// len = next_pow2(2n - 1) on zero-padded rows, first n columns kept
void toeplitz_apply_right_fft_dev(uint64_t m, uint64_t n, const double* g, const double* a, uint64_t lda,
                                  double* out, uint64_t ldo) {
    const uint64_t len = toeplitz_fft_len(n);
    double* c2 = ws<double>(WS_TMP2, len);
    k_toeplitz_embed<<<cdiv(len, 256), 256, 0, stream()>>>(n, len, g, c2);
    RL_LAUNCHED();
    circ_right_fft_launch(m, len, n, n, c2, a, lda, out, ldo);
}

namespace {
// transpose_spec (structured.cpp:85-94) of a circulant (c'[k] = c[(n - k) mod n]) and of the
// n x n Toeplitz (g' = row[0..n-1], col[1..n-1] from g = col[0..n-1], row[1..n-1])
__global__ void k_spec_transpose(uint64_t n, int toeplitz, const double* g, double* out) {
    const uint64_t len = toeplitz ? 2 * n - 1 : n;
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < len;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (!toeplitz)
            out[k] = g[(n - k) % n];
        else
            out[k] = k == 0 ? g[0] : (k < n ? g[n - 1 + k] : g[k - n + 1]);
    }
}
} // namespace

void spec_transpose_dev(uint64_t n, bool toeplitz, const double* g, double* out) {
    const uint64_t len = toeplitz ? 2 * n - 1 : n;
    k_spec_transpose<<<cdiv(len, 256), 256, 0, stream()>>>(n, toeplitz ? 1 : 0, g, out);
    RL_LAUNCHED();
}

void toeplitz_apply_vec_dev(uint64_t n, uint64_t nrhs, const double* g, const double* z, double* y) {
    k_toeplitz_vec<<<cdiv(n * nrhs, 256), 256, 0, stream()>>>(n, nrhs, g, z, y);
    RL_LAUNCHED();
}

} // namespace rl

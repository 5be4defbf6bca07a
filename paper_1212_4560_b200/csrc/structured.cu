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
            double s = 0.0;
            for (int t = 0; t < nnz; ++t)
                s += sg[t] * srow[r * n + idx[t]];
            out[(r0 + r) * ldo + j] = s;
        }
    }
}

// The same product for nnz = 4, n <= 16384 (config 5): persistent CTAs (one per SM) keep the
// whole S in registers — per thread 32 output columns x 4 (row, sign) entries packed as 16-bit
// (15-bit row | sign bit), two per register — and stream the rows of A through shared memory,
// so every byte of A and of the output crosses HBM once and S is read once per CTA (the kernel
// above re-reads S from L2 for every row: 786 KB per 128 KB row).  Same summation order.
constexpr int SP4_THREADS = 512, SP4_Q = 32;
__global__ void __launch_bounds__(SP4_THREADS, 1) k_sparse_right4(uint64_t n, const double* __restrict__ a,
                                                                  uint64_t lda, const int32_t* __restrict__ rows,
                                                                  const double* __restrict__ signs,
                                                                  double* __restrict__ out, uint64_t ldo) {
    extern __shared__ __align__(16) double srow[]; // n
    const int t = threadIdx.x;
    uint32_t pk[SP4_Q * 2]; // output q: entries (2q, 2q+1) -> pk[2q] lo/hi, (2q+2, 2q+3) -> pk[2q+1]
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
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const double2* src = reinterpret_cast<const double2*>(a + i * lda);
        for (uint64_t c = t; c < n / 2; c += SP4_THREADS)
            reinterpret_cast<double2*>(srow)[c] = __ldcs(src + c);
        __syncthreads();
        double* orow = out + i * ldo;
#pragma unroll
        for (int q = 0; q < SP4_Q; ++q) {
            const uint64_t j = t + static_cast<uint64_t>(q) * SP4_THREADS;
            if (j < n) {
                double s = 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = (pk[2 * q + (u >> 1)] >> (16 * (u & 1))) & 0xffffu;
                    const double x = srow[e & 0x7fffu];
                    s += (e & 0x8000u) ? -x : x; // s_jt = +-1: the reference's s += s_jt A(i, r_jt)
                }
                __stcs(orow + j, s);
            }
        }
        __syncthreads();
    }
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

void rank1_dense_dev(uint64_t n, const double* u, const double* v, double inv_uv, double* out) {
    k_rank1_dense<<<grid_for(n * n, 256), 256, 0, stream()>>>(n, u, v, inv_uv, out);
    RL_LAUNCHED();
}

// out = A H1 H2 (out may alias a); s12 = u1^T u2 (exact integer, host-computed)
void hh2_apply_right_dev(uint64_t n, const double* a, uint64_t lda, const double* u1, const double* u2,
                         double s12, double* out, uint64_t ldo) {
    double* w = ws<double>(WS_SMALL, 2 * n);
    k_hh2_rowdots<<<cdiv(n, 8), 256, 0, stream()>>>(n, a, lda, u1, u2, w, w + n);
    RL_LAUNCHED();
    k_hh2_apply<<<grid_for(n * ((n + 1) / 2), 256), 256, 0, stream()>>>(
        n, a, lda, u1, u2, w, w + n, s12, 2.0 / static_cast<double>(n), out, ldo);
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
        const size_t smem = n * sizeof(double);
        static bool attr[16] = {};
        if (!attr[ctx().device & 15]) {
            RL_CUDA(cudaFuncSetAttribute(k_sparse_right4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SP4_THREADS * SP4_Q * 8));
            attr[ctx().device & 15] = true;
        }
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, ctx().sms));
        k_sparse_right4<<<grid, SP4_THREADS, smem, stream()>>>(n, a, lda, rows, signs, out, ldo);
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

} // namespace rl

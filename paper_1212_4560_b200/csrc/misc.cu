// Small device utilities of the C-ABI: uniform_int draws (random_gen.cpp:59-70),
// packed <-> separate L/U layouts (genp.hpp:14-20), and the K12 peak probes.
#include <vector>

#include "rl_internal.cuh"

namespace rl {

namespace {

// Serial consumption of raw draws with the reference's rejection rule.
__global__ void k_uniform_int_consume(const uint64_t* pool, uint64_t pool_len, uint64_t count, int64_t lo,
                                      uint64_t span, int64_t* out, int* status) {
    if (threadIdx.x != 0 || blockIdx.x != 0)
        return;
    const uint64_t limit = (~0ULL) / span * span;
    uint64_t k = 0;
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t v;
        do {
            if (k >= pool_len) {
                *status = 1;
                return;
            }
            v = pool[k++];
        } while (v >= limit);
        out[i] = lo + static_cast<int64_t>(v % span);
    }
    *status = 0;
}

__global__ void k_unpack_lu(uint64_t n, const double* lu, double* l, double* u) {
    uint64_t total = n * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = e / n, j = e % n;
        double v = lu[e];
        l[e] = (i > j) ? v : (i == j ? 1.0 : 0.0);
        u[e] = (j >= i) ? v : 0.0;
    }
}

__global__ void k_pack_lu(uint64_t n, const double* l, const double* u, double* lu) {
    uint64_t total = n * n;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = e / n, j = e % n;
        lu[e] = (i > j) ? l[e] : u[e];
    }
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__global__ void k_probe_dmma(double* out, int iters) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        acc[i][0] = acc[i][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            dmma(acc[j], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        s += acc[i][0] + acc[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_probe_copy(const double4* __restrict__ in, double4* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

// kind 0 One (max column abs sum), 1 Inf (max row abs sum), 3 Frobenius partial sums
__global__ void k_norm_cols(uint64_t m, uint64_t n, const double* a, double* out) {
    uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (j >= n)
        return;
    double s = 0.0;
    for (uint64_t i = 0; i < m; ++i)
        s += fabs(a[i * n + j]);
    out[j] = s;
}

__global__ void k_norm_rows(uint64_t m, uint64_t n, const double* a, double* out) {
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= m)
        return;
    double s = 0.0;
    for (uint64_t j = 0; j < n; ++j)
        s += fabs(a[i * n + j]);
    out[i] = s;
}

} // namespace


// One / Inf norm partial vectors (host takes the max of n or m values)
void abs_sums_dev(uint64_t m, uint64_t n, const double* a, int rows, double* out) {
    if (rows)
        k_norm_rows<<<cdiv(m, 128), 128, 0, stream()>>>(m, n, a, out);
    else
        k_norm_cols<<<cdiv(n, 128), 128, 0, stream()>>>(m, n, a, out);
    RL_LAUNCHED();
}

void uniform_int_dev(uint64_t seed, uint64_t sid, uint64_t count, int64_t lo, int64_t hi, int64_t* out) {
    const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
    uint64_t slack = 64 + count / 4;
    for (int tries = 0; tries < 6; ++tries, slack *= 4) {
        uint64_t len = count + slack;
        uint64_t* pool = ws<uint64_t>(WS_TMP2, len + 1);
        int* st = reinterpret_cast<int*>(pool + len);
        rng_generate(seed, sid, Draw::RawU64, len, 0.0, 1.0, pool);
        k_uniform_int_consume<<<1, 32, 0, stream()>>>(pool, len, count, lo, span, out, st);
        RL_LAUNCHED();
        int h = 1;
        RL_CUDA(cudaMemcpyAsync(&h, st, sizeof(int), cudaMemcpyDeviceToHost, stream()));
        RL_CUDA(cudaStreamSynchronize(stream()));
        if (h == 0)
            return;
    }
    fail(RL_ERROR, "uniform_int: draw pool exhausted");
}

void unpack_lu_dev(uint64_t n, const double* lu, double* l, double* u) {
    k_unpack_lu<<<cdiv(n * n, 256) > 4736 ? 4736 : cdiv(n * n, 256), 256, 0, stream()>>>(n, lu, l, u);
    RL_LAUNCHED();
}

void pack_lu_dev(uint64_t n, const double* l, const double* u, double* lu) {
    k_pack_lu<<<cdiv(n * n, 256) > 4736 ? 4736 : cdiv(n * n, 256), 256, 0, stream()>>>(n, l, u, lu);
    RL_LAUNCHED();
}

// K12: measured FP64 DMMA peak (register-resident m8n8k4 chains) and HBM copy
// bandwidth (read + write bytes of a 2 GiB device copy), in the caller's process.
rl_status probe_peaks(double* fp64, double* hbm) {
    cudaStream_t st = stream();
    const int sms = ctx().sms;
    double* out = ws<double>(WS_TMP1, static_cast<size_t>(sms) * 8 * 128);
    cudaEvent_t e0, e1;
    RL_CUDA(cudaEventCreate(&e0));
    RL_CUDA(cudaEventCreate(&e1));
    float ms = 0.f;
    if (fp64) {
        const int blocks = sms * 8, threads = 128, iters = 20000;
        k_probe_dmma<<<blocks, threads, 0, st>>>(out, 200);
        RL_LAUNCHED();
        RL_CUDA(cudaEventRecord(e0, st));
        k_probe_dmma<<<blocks, threads, 0, st>>>(out, iters);
        RL_LAUNCHED();
        RL_CUDA(cudaEventRecord(e1, st));
        RL_CUDA(cudaEventSynchronize(e1));
        RL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        double flops = 2.0 * 256 * 8 * static_cast<double>(iters) * blocks * (threads / 32);
        *fp64 = flops / (ms * 1e-3) / 1e12;
    }
    if (hbm) {
        const size_t bytes = 1ULL << 30;
        double* a = ws<double>(WS_RF5, bytes / 8);
        double* b = ws<double>(WS_RF6, bytes / 8);
        RL_CUDA(cudaMemsetAsync(a, 0, bytes, st));
        double best = 0.0;
        for (int r = 0; r < 4; ++r) {
            RL_CUDA(cudaEventRecord(e0, st));
            k_probe_copy<<<sms * 8, 512, 0, st>>>(reinterpret_cast<const double4*>(a),
                                                  reinterpret_cast<double4*>(b), bytes / 32);
            RL_LAUNCHED();
            RL_CUDA(cudaEventRecord(e1, st));
            RL_CUDA(cudaEventSynchronize(e1));
            RL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            best = std::max(best, 2.0 * bytes / (ms * 1e-3) / 1e9);
        }
        *hbm = best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return RL_OK;
}

} // namespace rl

// FP64 pipe probe (dev aid): does DMMA (mma.sync m8n8k4 f64) share the DFMA pipe?
// Each warp runs independent chains; flop/s for DMMA-only, DFMA-only and both interleaved.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int NM, int NF>
__global__ void k_mix(double* out, int iters, double s) {
    double acc[8][2];
    double f[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = s * i;
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = s + i;
    const double a = s * 1.0001, b = s * 0.9999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (NM > 0) {
#pragma unroll
                for (int i = 0; i < NM; ++i) dmma(acc[i], a, b);
            }
            if (NF > 0) {
#pragma unroll
                for (int i = 0; i < NF; ++i) f[i] = fma(f[i], a, b);
            }
        }
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += acc[i][0] + acc[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) r += f[i];
    if (r == 12345.0) out[threadIdx.x] = r;
}

template <int NM, int NF>
void run(const char* name, int blocks, int threads, int iters) {
    double* d;
    cudaMalloc(&d, 8192);
    k_mix<NM, NF><<<blocks, threads>>>(d, 10, 1.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_mix<NM, NF><<<blocks, threads>>>(d, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double warps = double(blocks) * threads / 32;
    double fl_m = warps * iters * 8.0 * NM * 512.0;      // m8n8k4: 256 FMA = 512 flop per warp op
    double fl_f = warps * 32 * iters * 8.0 * NF * 2.0;
    printf("%-28s %8.3f ms  DMMA %6.2f TF/s  DFMA %6.2f TF/s  total %6.2f TF/s\n", name, ms, fl_m / ms / 1e9,
           fl_f / ms / 1e9, (fl_m + fl_f) / ms / 1e9);
    cudaFree(d);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int B = sms * 4, T = 256;
    run<8, 0>("dmma only (8 chains)", B, T, 4000);
    run<0, 16>("dfma only (16 chains)", B, T, 4000);
    run<8, 16>("dmma 8 + dfma 16", B, T, 4000);
    run<4, 16>("dmma 4 + dfma 16", B, T, 4000);
    run<8, 8>("dmma 8 + dfma 8", B, T, 4000);
    run<2, 16>("dmma 2 + dfma 16", B, T, 4000);
    return 0;
}

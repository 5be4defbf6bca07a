// Dependent-latency microbenchmarks (dev aid): cycles per dependent op on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, double seed, int n) {
    __shared__ double sm[1024];
    __shared__ int ism[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + 1e-9 * i; ism[i] = (i * 7 + 1) & 1023; }
    __syncthreads();
    double x = seed, y = seed * 0.5;
    long long t0, t1;
    // 1 DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 0.999999999, 1e-12);
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0);
    // 2 rcp.approx.f64 chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1e-3; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0);
    // 3 IEEE division chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) y = 1.0 / (y + 1e-3);
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0);
    // 4 sqrt chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) y = sqrt(y + 1.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0);
    // 5 LDS pointer chase
    int p = threadIdx.x & 1023;
    t0 = clock64();
    for (int i = 0; i < n; ++i) p = ism[p];
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0);
    // 6 SHFL f64 chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-12;
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0);
    // 7 syncthreads loop (all threads)
    t0 = clock64();
    for (int i = 0; i < n; ++i) { sm[threadIdx.x & 1023] += 1.0; __syncthreads(); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0);
    // 8 DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + 1e-12;
    t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0);
    // 9 rsqrt.approx.f64 chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1.0; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[8] = (t1 - t0);
    // 10 float rcp chain
    float f = (float)y;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { f = __frcp_rn(f + 1.0f); }
    t1 = clock64(); if (threadIdx.x == 0) cyc[9] = (t1 - t0);
    float g = f;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(g)); g = r + 1.0f; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[10] = (t1 - t0);
    out[threadIdx.x] = x + y + p + f + g;
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8 * 16);
    const char* names[] = {"dfma", "rcp.approx.f64", "div.rn.f64", "sqrt.rn.f64", "lds chase", "shfl f64", "syncthreads", "dadd", "rsqrt.approx.f64", "frcp_rn f32", "rcp.approx.f32"};
    for (int nt : {32, 512, 1024}) {
        k_lat<<<1, nt>>>(out, cyc, 1.5, 1000);
        cudaDeviceSynchronize();
        k_lat<<<1, nt>>>(out, cyc, 1.5, 1000);
        long long h[16]; cudaMemcpy(h, cyc, 8 * 11, cudaMemcpyDeviceToHost);
        printf("threads %d:", nt);
        for (int i = 0; i < 11; ++i) printf("  %s %.1f", names[i], h[i] / 1000.0);
        printf("\n");
    }
    return 0;
}

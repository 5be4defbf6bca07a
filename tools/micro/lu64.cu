// Cycle counts of the batched kernel's register LU alone (dev aid): one CTA, REPS LUs back to back.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include
//        -I../../paper_1212_4560_b200/csrc --expt-relaxed-constexpr -o lu64 lu64.cu
#include "../../paper_1212_4560_b200/csrc/genp_batched.cu"
#include <cstdio>

namespace rl {
namespace {
__global__ void __launch_bounds__(64, 1) k_lu64(const double* A, double* out, long long* cyc, int reps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x, tr = t >> 3, tc = t & 7;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 64;" ::"r"(smem_u32(&S.mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t ph = 0;
    double acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        double w[8][8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c)
                w[r][c] = A[(tr + 8 * r) * 64 + tc + 8 * c] + (r == c && tr == tc ? 64.0 : 0.0);
        __syncthreads();
        lu_regs(w, S, tr, tc, ph);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c)
                acc += w[r][c];
    }
    long long t1 = clock64();
    if (t == 0)
        cyc[0] = t1 - t0;
    out[t] = acc;
}
} // namespace
} // namespace rl


namespace rl {
namespace {
template <int F> struct V { static constexpr bool bulk = !(F & 1), wait = !(F & 2), rcp = !(F & 4), crit = !(F & 8), pub = !(F & 16);
  static constexpr int rmode = (F >> 5) & 3; static constexpr bool bar = (F & 128) != 0; };
__device__ __forceinline__ double rcp_nb(double p) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
    double e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    return p == 0.0 ? 0.0 : r;
}
template <int M> __device__ __forceinline__ double rcpv(double p) {
    if (M == 0) return pivot_rcp(p);
    if (M == 1) return rcp_nb(p);
    if (M == 2) return __drcp_rn(p);
    return 1.0 / p;
}
template <int F, int K>
__device__ __forceinline__ void vpub(const double (&w)[8][8], Smem& S, int s, int tr, int tc, uint32_t mb) {
    double* ur = S.pub + (s & 1) * 128 + tc;
    double* uc = S.pub + (s & 1) * 128 + 64 + tr;
    if (V<F>::pub) {
    if (tc == s) {
        if (tr == s) S.rcp[8 * K + s] = V<F>::rcp ? rcpv<V<F>::rmode>(w[K][K]) : w[K][K];
#pragma unroll
        for (int r = K; r < 8; ++r) uc[8 * r] = w[r][K];
    }
    if (tr == s) {
#pragma unroll
        for (int c = K; c < 8; ++c) ur[8 * c] = w[K][c];
    }
    }
    if (!V<F>::bar) mb_arrive(mb);
}
template <int F, int K, int PAR, bool LAST>
__device__ __forceinline__ void vstep(double (&w)[8][8], Smem& S, int s, int tr, int tc, uint32_t mb, uint32_t& ph) {
    constexpr int KC = LAST ? K + 1 : K;
    if (V<F>::bar) __syncthreads(); else if (V<F>::wait) mb_wait(mb, ph); else __syncwarp();
    const double* ur = S.pub + PAR * 128 + tc;
    const double* uc = S.pub + PAR * 128 + 64 + tr;
    const double inv = S.rcp[8 * K + s];
    double m[8];
#pragma unroll
    for (int r = K; r < 8; ++r) m[r] = uc[8 * r] * inv;
    m[K] = tr > s ? m[K] : 0.0;
    const bool cK = tc > s;
    auto u_at = [&](int c) { return c == K ? (cK ? ur[8 * c] : 0.0) : ur[8 * c]; };
    if (KC < 8) {
        if (V<F>::crit) {
#pragma unroll
        for (int c = K; c < 8; ++c) w[KC][c] = fma(-m[KC], u_at(c), w[KC][c]);
        const double ukc = u_at(KC);
#pragma unroll
        for (int r = K; r < 8; ++r) if (r != KC) w[r][KC] = fma(-m[r], ukc, w[r][KC]);
        }
        vpub<F, (KC < 8 ? KC : 7)>(w, S, LAST ? 0 : s + 1, tr, tc, mb);
    }
    if (V<F>::bulk) {
#pragma unroll
    for (int c = K; c < 8; ++c) {
        if (c == KC) continue;
        const double u = u_at(c);
#pragma unroll
        for (int r = K; r < 8; ++r) if (r != KC) w[r][c] = fma(-m[r], u, w[r][c]);
    }
    }
}
template <int F, int K>
__device__ __forceinline__ void vblock(double (&w)[8][8], Smem& S, int tr, int tc, uint32_t mb, uint32_t& ph) {
#pragma unroll 1
    for (int s = 0; s < 6; s += 2) { vstep<F, K, 0, false>(w, S, s, tr, tc, mb, ph); vstep<F, K, 1, false>(w, S, s + 1, tr, tc, mb, ph); }
    vstep<F, K, 0, false>(w, S, 6, tr, tc, mb, ph);
    vstep<F, K, 1, true>(w, S, 7, tr, tc, mb, ph);
}
template <int F>
__global__ void __launch_bounds__(64, 1) k_v(const double* A, double* out, long long* cyc, int reps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x, tr = t >> 3, tc = t & 7;
    if (t == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 64;" ::"r"(smem_u32(&S.mbar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    uint32_t ph = 0; double acc = 0;
    const uint32_t mb = smem_u32(&S.mbar);
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        double w[8][8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) w[r][c] = A[(tr + 8 * r) * 64 + tc + 8 * c] + (r == c && tr == tc ? 64.0 : 0.0);
        __syncthreads();
        vpub<F, 0>(w, S, 0, tr, tc, mb);
        vblock<F,0>(w,S,tr,tc,mb,ph); vblock<F,1>(w,S,tr,tc,mb,ph); vblock<F,2>(w,S,tr,tc,mb,ph); vblock<F,3>(w,S,tr,tc,mb,ph);
        vblock<F,4>(w,S,tr,tc,mb,ph); vblock<F,5>(w,S,tr,tc,mb,ph); vblock<F,6>(w,S,tr,tc,mb,ph); vblock<F,7>(w,S,tr,tc,mb,ph);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc += w[r][c];
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    out[t] = acc;
}
} // namespace
} // namespace rl
template <int F> void runv(const char* name, double* A, double* o, long long* c) {
    cudaFuncSetAttribute(rl::k_v<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(rl::Smem));
    rl::k_v<F><<<1, 64, sizeof(rl::Smem)>>>(A, o, c, 10);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %lld cycles per LU (%lld per step)\n", name, h / 10, h / 640);
}

namespace rl {
namespace {
// variant B: publications laid out [owner][8] (128-bit stores / loads), branch-free rcp by all
// threads, predicated stores; SYNC 0 = bar.sync, 1 = mbarrier arrive/wait
template <int SYNC, int K>
__device__ __forceinline__ void bpub(const double (&w)[8][8], Smem& S, int s, int tr, int tc, uint32_t mb) {
    double* ur = S.pub + (s & 1) * 128 + tc * 8;       // row k: owner (s, tc) writes c = 0..7
    double* uc = S.pub + (s & 1) * 128 + 64 + tr * 8;  // col k: owner (tr, s) writes r = 0..7
    const double inv = rcp_nb(w[K][K]);
    if (tc == s && tr == s) S.rcp[8 * K + s] = inv;
    if (tc == s) {
#pragma unroll
        for (int r = K & ~1; r < 8; r += 2) *reinterpret_cast<double2*>(uc + r) = make_double2(w[r][K], w[r + 1][K]);
    }
    if (tr == s) {
#pragma unroll
        for (int c = K & ~1; c < 8; c += 2) *reinterpret_cast<double2*>(ur + c) = make_double2(w[K][c], w[K][c + 1]);
    }
    if (SYNC == 1) mb_arrive(mb);
}
template <int SYNC, int K, int PAR, bool LAST>
__device__ __forceinline__ void bstep(double (&w)[8][8], Smem& S, int s, int tr, int tc, uint32_t mb, uint32_t& ph) {
    constexpr int KC = LAST ? K + 1 : K;
    if (SYNC == 0) __syncthreads(); else mb_wait(mb, ph);
    const double* ur = S.pub + PAR * 128 + tc * 8;
    const double* uc = S.pub + PAR * 128 + 64 + tr * 8;
    const double inv = S.rcp[8 * K + s];
    double m[8];
#pragma unroll
    for (int r = K & ~1; r < 8; r += 2) { const double2 v = *reinterpret_cast<const double2*>(uc + r); if (r >= K) m[r] = v.x * inv; m[r + 1] = v.y * inv; }
    m[K] = tr > s ? m[K] : 0.0;
    const bool cK = tc > s;
    // pivot-row pairs re-read where used
    auto upair = [&](int c, double& u0, double& u1) {
        const double2 v = *reinterpret_cast<const double2*>(ur + c);
        u0 = (c == K) ? (cK ? v.x : 0.0) : v.x;
        u1 = (c + 1 == K) ? (cK ? v.y : 0.0) : v.y;
    };
    if (KC < 8) {
        double ukc = 0.0;
#pragma unroll
        for (int c = K & ~1; c < 8; c += 2) {
            double u0, u1;
            upair(c, u0, u1);
            if (c >= K) w[KC][c] = fma(-m[KC], u0, w[KC][c]);
            w[KC][c + 1] = fma(-m[KC], u1, w[KC][c + 1]);
            if (c == KC) ukc = u0;
            if (c + 1 == KC) ukc = u1;
        }
#pragma unroll
        for (int r = K; r < 8; ++r) if (r != KC) w[r][KC] = fma(-m[r], ukc, w[r][KC]);
        bpub<SYNC, (KC < 8 ? KC : 7)>(w, S, LAST ? 0 : s + 1, tr, tc, mb);
    }
#pragma unroll
    for (int c = K & ~1; c < 8; c += 2) {
        double u0, u1;
        upair(c, u0, u1);
#pragma unroll
        for (int r = K; r < 8; ++r) {
            if (r == KC) continue;
            if (c >= K && c != KC) w[r][c] = fma(-m[r], u0, w[r][c]);
            if (c + 1 != KC) w[r][c + 1] = fma(-m[r], u1, w[r][c + 1]);
        }
    }
}
template <int SYNC, int K>
__device__ __forceinline__ void bblock(double (&w)[8][8], Smem& S, int tr, int tc, uint32_t mb, uint32_t& ph) {
#pragma unroll 1
    for (int s = 0; s < 6; s += 2) { bstep<SYNC, K, 0, false>(w, S, s, tr, tc, mb, ph); bstep<SYNC, K, 1, false>(w, S, s + 1, tr, tc, mb, ph); }
    bstep<SYNC, K, 0, false>(w, S, 6, tr, tc, mb, ph);
    bstep<SYNC, K, 1, true>(w, S, 7, tr, tc, mb, ph);
}
template <int SYNC, int LB>
__global__ void __launch_bounds__(64, LB) k_b(const double* A, double* out, long long* cyc, int reps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x, tr = t >> 3, tc = t & 7;
    if (t == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 64;" ::"r"(smem_u32(&S.mbar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    uint32_t ph = 0; double acc = 0;
    const uint32_t mb = smem_u32(&S.mbar);
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        double w[8][8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) w[r][c] = A[(tr + 8 * r) * 64 + tc + 8 * c] + (r == c && tr == tc ? 64.0 : 0.0);
        __syncthreads();
        bpub<SYNC, 0>(w, S, 0, tr, tc, mb);
        bblock<SYNC,0>(w,S,tr,tc,mb,ph); bblock<SYNC,1>(w,S,tr,tc,mb,ph); bblock<SYNC,2>(w,S,tr,tc,mb,ph); bblock<SYNC,3>(w,S,tr,tc,mb,ph);
        bblock<SYNC,4>(w,S,tr,tc,mb,ph); bblock<SYNC,5>(w,S,tr,tc,mb,ph); bblock<SYNC,6>(w,S,tr,tc,mb,ph); bblock<SYNC,7>(w,S,tr,tc,mb,ph);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc += w[r][c];
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    out[t] = acc;
}
} // namespace
} // namespace rl
template <int F, int LB> void runb(const char* name, double* A, double* o, long long* c) {
    cudaFuncSetAttribute(rl::k_b<F, LB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(rl::Smem));
    rl::k_b<F, LB><<<1, 64, sizeof(rl::Smem)>>>(A, o, c, 10);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %lld cycles per LU (%lld per step)\n", name, h / 10, h / 640);
}

int main() {
    double *A, *o;
    long long* c;
    cudaMalloc(&A, 4096 * 8);
    cudaMalloc(&o, 64 * 8);
    cudaMalloc(&c, 8);
    cudaMemset(A, 0, 4096 * 8);
    cudaFuncSetAttribute(rl::k_lu64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(rl::Smem));
    for (int reps : {1, 10}) {
        rl::k_lu64<<<1, 64, sizeof(rl::Smem)>>>(A, o, c, reps);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("reps %d: %lld cycles per LU (%lld per pivot step)\n", reps, h / reps, h / reps / 64);
    }
    runb<0, 1>("B2 bar.sync", A, o, c);
    runb<1, 1>("B2 mbarrier", A, o, c);
    runb<0, 6>("B2 bar.sync cap6", A, o, c);
    runb<0, 5>("B2 bar.sync cap5", A, o, c);
    runv<0>("full", A, o, c);
    runv<32>("rcp branch-free", A, o, c);
    runv<64>("rcp __drcp_rn", A, o, c);
    runv<96>("rcp 1/p", A, o, c);
    runv<128>("bar.sync", A, o, c);
    runv<128 | 32>("bar.sync + rcp branch-free", A, o, c);
    runv<1>("no bulk FMA", A, o, c);
    runv<2>("no wait", A, o, c);
    runv<4>("no rcp", A, o, c);
    runv<8>("no critical FMA", A, o, c);
    runv<16>("no publish", A, o, c);
    runv<1 | 8>("no FMA at all", A, o, c);
    runv<1 | 2 | 8>("no FMA, no wait", A, o, c);
    runv<1 | 2 | 4 | 8 | 16>("skeleton", A, o, c);
    return 0;
}

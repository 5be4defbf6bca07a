// Register-resident no-pivot LU of an (8G) x (8G) block on G*G threads (genp.cpp:20-33), shared
// by the batched n = 64 kernel (G = 8, with the right-hand side forward-substituted alongside)
// and the blocked LU's 128 x 128 diagonal block (G = 16).
//
// Thread (tr, tc) = (t / G, t % G) owns w(tr + G r, tc + G c), r, c < 8 (cyclic: every thread
// keeps an equal share of the shrinking trailing matrix until the last block of G pivots).  One
// barrier per pivot step k = G K + s: the owners of row k and column k publish them (owner-major
// 128-bit stores, predicated, double-buffered by step parity), the pivot's owner publishes 1/p;
// every thread forms its multipliers m = w(i,k) (1/p) and updates its entries with one FMA
// each.  The next step's row / column are updated and published first.  Rows / columns at or
// left of the pivot are left unchanged by a zero multiplier / pivot-row entry (fma(-0, u, w) =
// w) instead of per-FMA predicates; the column of multipliers is not written back — column k
// keeps w(i,k) and L = w(i,k) (1/p) is formed once by the caller (the same product the update
// used).  1/p: rcp.approx + two Newton steps (exact to rounding for 2^-1022 <= |p| <= 2^1022;
// 0 -> 0 as the reference's m = 0 for a zero pivot, +-inf -> 0; subnormal pivots give an
// infinite reciprocal where the reference's w / p overflows too).
#pragma once

#include <cstdint>

namespace rl {
namespace reglu {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double pivot_rcp(double p) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
    double e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    e = fma(-p, r, 1.0);
    r = fma(r, e, r);
    return (p == 0.0 || isinf(p)) ? 0.0 : r;
}

__device__ __forceinline__ void st_if(double* dst, double v, bool pred) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.shared.f64 [%0], %1;\n}" ::"r"(smem_addr(dst)),
                 "d"(v), "r"(static_cast<int>(pred))
                 : "memory");
}
__device__ __forceinline__ void st2_if(double* dst, double v0, double v1, bool pred) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n @p st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(
                     smem_addr(dst)),
                 "d"(v0), "d"(v1), "r"(static_cast<int>(pred))
                 : "memory");
}

// Publication buffer per parity: the pivot row owner-major at pitch RP (a quarter-warp's eight
// owners' 128-bit reads hit distinct banks), then the pivot column owner-major at pitch 8.
template <int G>
struct Pub {
    static constexpr int RP = 10, C = G * RP, SIZE = C + 8 * G;
};

// Shared-memory pointers of one factorization: pub = 2 Pub<G>::SIZE doubles, rcp = 8G doubles
// (1/U_kk on exit), pubb = 2 doubles (RHS only); mbar: an mbarrier initialised for G*G arrivals
// (MB only) and the thread's copy of its phase parity.
struct Bufs {
    double* pub;
    double* rcp;
    double* pubb;
    uint64_t* mbar = nullptr;
};

// Step hand-off through an mbarrier (MB): a thread arrives once it has published and then
// issues the bulk of its FMAs; the wait sits at the top of the next step, so the bulk FMAs
// leave the critical path.  Measured slower than bar.sync for both users (G = 8: 281 against
// 252 cycles per step, tools/micro/lu64.cu; G = 16: 31.4 against 30.0 us per 128 x 128 block).
__device__ __forceinline__ void mb_arrive(uint64_t* mb) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(mb)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* mb, uint32_t& ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(smem_addr(mb)), "r"(ph)
                     : "memory");
    ph ^= 1u;
}

// Publication for step k = G K + s (K compile-time, s at run time).
template <int G, bool RHS, bool MB, int K>
__device__ __forceinline__ void publish(const double (&w)[8][8], double bcur, const Bufs& B, int s, int tr, int tc) {
    using PB = Pub<G>;
    double* ur = B.pub + (s & 1) * PB::SIZE + tc * PB::RP;
    double* uc = B.pub + (s & 1) * PB::SIZE + PB::C + tr * 8;
    const bool oc = tc == s, orow = tr == s;
    st_if(B.rcp + G * K + s, pivot_rcp(w[K][K]), oc && orow);
    if (RHS)
        st_if(B.pubb + (s & 1), bcur, static_cast<int>(threadIdx.x) == G * K + s); // b_k by thread k
#pragma unroll
    for (int r = K & ~1; r < 8; r += 2)
        st2_if(uc + r, w[r][K], w[r + 1][K], oc);
#pragma unroll
    for (int c = K & ~1; c < 8; c += 2)
        st2_if(ur + c, w[K][c], w[K][c + 1], orow);
    if (MB)
        mb_arrive(B.mbar);
}

// Pivot step k = G K + s (parity PAR = s & 1; LAST: s = G - 1, the next step opens block K+1).
// RHS: thread t (< 8G) holds b_t in bcur and subtracts m_t b_k (genp.cpp:110-115's order).
template <int G, bool RHS, bool MB, int K, int PAR, bool LAST>
__device__ __forceinline__ void step(double (&w)[8][8], double& bcur, const Bufs& B, uint32_t& ph, int s, int tr,
                                     int tc) {
    using PB = Pub<G>;
    constexpr int KC = LAST ? K + 1 : K;
    if (MB)
        mb_wait(B.mbar, ph);
    else
        __syncthreads();
    const double* ur = B.pub + PAR * PB::SIZE + tc * PB::RP;
    const double* uc = B.pub + PAR * PB::SIZE + PB::C + tr * 8;
    const double inv = B.rcp[G * K + s];
    if (RHS) {
        const int t = threadIdx.x, k = G * K + s;
        const double mt = B.pub[PAR * PB::SIZE + PB::C + (t % G) * 8 + (t / G)] * inv;
        const double f = fma(-mt, B.pubb[PAR], bcur);
        bcur = t > k ? f : bcur;
    }
    double m[8], u[8];
#pragma unroll
    for (int r = K & ~1; r < 8; r += 2) {
        const double2 v = *reinterpret_cast<const double2*>(uc + r);
        if (r >= K)
            m[r] = v.x * inv;
        m[r + 1] = v.y * inv;
    }
    m[K] = tr > s ? m[K] : 0.0;
#pragma unroll
    for (int c = K & ~1; c < 8; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(ur + c);
        if (c >= K)
            u[c] = v.x;
        u[c + 1] = v.y;
    }
    u[K] = tc > s ? u[K] : 0.0;
    if (KC < 8) {
#pragma unroll
        for (int c = K; c < 8; ++c)
            w[KC][c] = fma(-m[KC], u[c], w[KC][c]);
#pragma unroll
        for (int r = K; r < 8; ++r)
            if (r != KC)
                w[r][KC] = fma(-m[r], u[KC], w[r][KC]);
        publish<G, RHS, MB, (KC < 8 ? KC : 7)>(w, bcur, B, LAST ? 0 : s + 1, tr, tc);
    }
#pragma unroll
    for (int c = K; c < 8; ++c) {
        if (c == KC)
            continue;
#pragma unroll
        for (int r = K; r < 8; ++r)
            if (r != KC)
                w[r][c] = fma(-m[r], u[c], w[r][c]);
    }
}

// The G pivot steps of block K; the step index only enters predicates, so one loop body per
// block and parity (the register indices are compile-time) keeps the code small.
template <int G, bool RHS, bool MB, int K>
__device__ __forceinline__ void block(double (&w)[8][8], double& bcur, const Bufs& B, uint32_t& ph, int tr, int tc) {
#pragma unroll 1
    for (int s = 0; s < G - 2; s += 2) {
        step<G, RHS, MB, K, 0, false>(w, bcur, B, ph, s, tr, tc);
        step<G, RHS, MB, K, 1, false>(w, bcur, B, ph, s + 1, tr, tc);
    }
    step<G, RHS, MB, K, 0, false>(w, bcur, B, ph, G - 2, tr, tc);
    step<G, RHS, MB, K, 1, true>(w, bcur, B, ph, G - 1, tr, tc);
}

// The whole factorization: on exit w holds U on and above the diagonal and w(i,k)
// (un-normalised) below; B.rcp[k] = 1/U_kk; bcur (RHS) = (L^-1 b)_t.  Callers fence before
// (the publication buffers free) and after (publications consumed).  MB: ph is the thread's
// copy of B.mbar's phase parity (advanced once per pivot step).
template <int G, bool RHS, bool MB = false>
__device__ __forceinline__ void factor(double (&w)[8][8], double& bcur, const Bufs& B, int tr, int tc,
                                       uint32_t* php = nullptr) {
    uint32_t ph = php ? *php : 0u;
    publish<G, RHS, MB, 0>(w, bcur, B, 0, tr, tc);
    block<G, RHS, MB, 0>(w, bcur, B, ph, tr, tc);
    block<G, RHS, MB, 1>(w, bcur, B, ph, tr, tc);
    block<G, RHS, MB, 2>(w, bcur, B, ph, tr, tc);
    block<G, RHS, MB, 3>(w, bcur, B, ph, tr, tc);
    block<G, RHS, MB, 4>(w, bcur, B, ph, tr, tc);
    block<G, RHS, MB, 5>(w, bcur, B, ph, tr, tc);
    block<G, RHS, MB, 6>(w, bcur, B, ph, tr, tc);
    block<G, RHS, MB, 7>(w, bcur, B, ph, tr, tc);
    if (php)
        *php = ph;
}

} // namespace reglu
} // namespace rl

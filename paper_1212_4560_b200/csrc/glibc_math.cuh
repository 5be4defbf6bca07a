// glibc_math.cuh — the exact operation sequences of glibc 2.39's x86-64 `__log_fma` and
// `__sincos_fma`, restated for the GPU (and for the host, where tests/cpp/test_glibc_math.cpp
// checks them against the installed libm bit for bit).
//
// Why: the reference's Gaussian draw (`/root/reference/proj/src/random_gen.cpp:46-52`,
// Box-Muller) calls `std::log` and `std::sin`/`std::cos`, which GCC merges into one `sincos`
// call; on an FMA+AVX2 host glibc's ifunc resolvers bind `log` and `sincos` to their FMA builds.
// Those are not correctly rounded, so matching the reference's G bit for bit means executing
// the same rounding steps: every multiply/add below is a single IEEE operation in the order the
// FMA build performs it, and every `GLM_FMA` is a fused multiply-add exactly where the FMA build
// has one (read from the libm disassembly, `tools/extract_libm_tables.py` documents the
// addresses). No other contraction is allowed: device code uses the `__d*_rn` intrinsics
// (nvcc never fuses those) and the host build uses -ffp-contract=off.
//
// Algorithms (published glibc sources, restated): log — the table method of sysdeps/ieee754/
// dbl-64/e_log.c (128-entry {1/c, log c} table, degree-5 polynomial in r = z/c − 1, a separate
// degree-11 polynomial with an exact r² split near 1). sincos — sysdeps/ieee754/dbl-64/s_sin.c
// (do_sin / do_cos on the 110-row __sincostab with Taylor corrections, the hp0/hp1 reduction
// for |x| < 2.426, reduce_sincos's 4-part π/2 reduction below 105414350). Box-Muller needs
// 0 ≤ x < 2π only; larger arguments (glibc's __branred) are not restated.
#pragma once
#include <stdint.h>
#include <string.h>

#include "glibc_tables.inc"

#if defined(__CUDACC__)
#define GLM_FN __host__ __device__ __forceinline__
#else
#define GLM_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define GLM_MUL(a, b) __dmul_rn((a), (b))
#define GLM_ADD(a, b) __dadd_rn((a), (b))
#define GLM_SUB(a, b) __dsub_rn((a), (b))
#define GLM_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define GLM_MUL(a, b) ((a) * (b))
#define GLM_ADD(a, b) ((a) + (b))
#define GLM_SUB(a, b) ((a) - (b))
#define GLM_FMA(a, b, c) __builtin_fma((a), (b), (c))
#endif

namespace glm {

#if defined(__CUDACC__)
__device__ const double d_log_data[2 + 5 + 11 + 256] = GLM_LOG_DATA_INIT;
__device__ const double d_sincostab[440] = GLM_SINCOSTAB_INIT;
#endif
static const double h_log_data[2 + 5 + 11 + 256] = GLM_LOG_DATA_INIT;
static const double h_sincostab[440] = GLM_SINCOSTAB_INIT;

GLM_FN double ld(int i) {
#if defined(__CUDA_ARCH__)
    return __ldg(&d_log_data[i]);
#else
    return h_log_data[i];
#endif
}
GLM_FN double sct(int i) {
#if defined(__CUDA_ARCH__)
    return __ldg(&d_sincostab[i]);
#else
    return h_sincostab[i];
#endif
}

GLM_FN uint64_t bits(double x) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
GLM_FN double from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}
GLM_FN double copysign_of(double mag, double sgn) {
    return from_bits((bits(mag) & 0x7fffffffffffffffULL) | (bits(sgn) & 0x8000000000000000ULL));
}
GLM_FN double neg(double x) { return from_bits(bits(x) ^ 0x8000000000000000ULL); }

// __log_data layout (indices into ld()).
enum { kLn2hi = 0, kLn2lo = 1, kA = 2, kB = 7, kTab = 18 };

// log(x) for finite x > 0 (the Box-Muller domain (0, 1]; subnormals included).
GLM_FN double log_fma(double x) {
    uint64_t ix = bits(x);
    if (ix - 0x3fee000000000000ULL < 0x0003090000000000ULL) {
        // 1 - 2^-4 <= x < 1 + 0x1.09p-4: no table, degree-11 polynomial, exact r^2 split.
        if (ix == 0x3ff0000000000000ULL)
            return 0.0;
        const double r = GLM_SUB(x, 1.0);
        const double r2 = GLM_MUL(r, r);
        const double r3 = GLM_MUL(r, r2);
        const double p1 = GLM_FMA(r2, ld(kB + 3), GLM_FMA(r, ld(kB + 2), ld(kB + 1)));
        const double p4 = GLM_FMA(r2, ld(kB + 6), GLM_FMA(r, ld(kB + 5), ld(kB + 4)));
        const double p7 =
            GLM_FMA(r3, ld(kB + 10), GLM_FMA(r2, ld(kB + 9), GLM_FMA(r, ld(kB + 8), ld(kB + 7))));
        const double q = GLM_FMA(GLM_FMA(p7, r3, p4), r3, p1);
        const double rhi = GLM_FMA(-0x1p27, r, GLM_FMA(r, 0x1p27, r));
        const double rhi2 = GLM_MUL(rhi, rhi);
        const double rlo = GLM_SUB(r, rhi);
        const double b0 = ld(kB + 0);
        const double hi = GLM_FMA(rhi2, b0, r);
        double lo = GLM_FMA(rhi2, b0, GLM_SUB(r, hi));
        lo = GLM_FMA(GLM_MUL(b0, rlo), GLM_ADD(r, rhi), lo);
        const double y = GLM_FMA(q, r3, lo);
        return GLM_ADD(hi, y);
    }
    const uint64_t top = ix >> 48;
    if (top - 0x10 > 0x7fdf) {
        if ((ix << 1) == 0)
            return -__builtin_inf();
        if (ix == 0x7ff0000000000000ULL)
            return x;
        if ((top & 0x8000) || (top & 0x7ff0) == 0x7ff0)
            return __builtin_nan("");
        // subnormal: normalise, then continue with the exponent corrected
        ix = bits(GLM_MUL(x, 0x1p52)) - (52ULL << 52);
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ULL;
    const int i = static_cast<int>((tmp >> 45) & 127);
    const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
    const double z = from_bits(ix - (tmp & 0xfff0000000000000ULL));
    const double invc = ld(kTab + 2 * i), logc = ld(kTab + 2 * i + 1);
    const double kd = static_cast<double>(k);
    const double w = GLM_FMA(kd, ld(kLn2hi), logc);
    const double r = GLM_FMA(z, invc, -1.0);
    const double hi = GLM_ADD(r, w);
    const double lo = GLM_FMA(kd, ld(kLn2lo), GLM_ADD(GLM_SUB(w, hi), r));
    const double r2 = GLM_MUL(r, r);
    const double p1 = GLM_FMA(r, ld(kA + 2), ld(kA + 1));
    const double p3 = GLM_FMA(r, ld(kA + 4), ld(kA + 3));
    const double lo2 = GLM_FMA(r2, ld(kA + 0), lo);
    const double q = GLM_FMA(p3, r2, p1);
    const double y = GLM_FMA(GLM_MUL(r, r2), q, lo2);
    return GLM_ADD(y, hi);
}

// s_sin.c constants (usncs.h / s_sin.c), as the FMA build loads them.
constexpr double kSn3 = -0x1.5555555555515p-3, kSn5 = 0x1.11110e829872fp-7;
constexpr double kCs2 = 0x1.0000000000000p-1, kCs4 = -0x1.5555555555535p-5,
                 kCs6 = 0x1.6c16bedd9e239p-10;
constexpr double kS1 = -0x1.5555555555555p-3, kS2 = 0x1.1111111110ecep-7,
                 kS3 = -0x1.a01a019db08b8p-13, kS4 = 0x1.71de27b9a7ed9p-19,
                 kS5 = -0x1.addffc2fcdf59p-26;
constexpr double kBig = 0x1.8p45, kHp0 = 0x1.921fb54442d18p+0, kHp1 = 0x1.1a62633145c07p-54;
constexpr double kToint = 0x1.8p52, kHpinv = 0x1.45f306dc9c883p-1;
constexpr double kMp1 = 0x1.921fb58000000p+0, kMp2 = -0x1.dde973c000000p-27;
constexpr double kPp3 = -0x1.cb3b398000000p-55, kPp4 = -0x1.d747f23e32ed7p-83;

// TAYLOR_SIN(a*a, a, da): ((poly(xx)·a − da/2)·xx + da) + a.
GLM_FN double taylor_sin(double a, double da) {
    const double xx = GLM_MUL(a, a);
    double p = GLM_FMA(xx, kS5, kS4);
    p = GLM_FMA(xx, p, kS3);
    p = GLM_FMA(xx, p, kS2);
    p = GLM_FMA(xx, p, kS1);
    const double t = GLM_FMA(xx, GLM_FMA(p, a, neg(GLM_MUL(da, 0.5))), da);
    return GLM_ADD(a, t);
}

// Table row u = big + |x| and the reduced remainder x'' = |x| − (u − big).
struct Row {
    double sn, ssn, cs, ccs, xr;
};
GLM_FN Row row_of(double ax) {
    const double u = GLM_ADD(ax, kBig);
    const int k4 = static_cast<int>(static_cast<uint32_t>(bits(u))) << 2;
    Row t;
    t.xr = GLM_SUB(ax, GLM_SUB(u, kBig));
    t.sn = sct(k4);
    t.ssn = sct(k4 + 1);
    t.cs = sct(k4 + 2);
    t.ccs = sct(k4 + 3);
    return t;
}

// do_sin's table branch on x'' with the sign-adjusted tail dx; magnitude only.
GLM_FN double sin_tab(const Row& t, double dx) {
    const double xr = t.xr;
    const double xx = GLM_MUL(xr, xr);
    const double s = GLM_ADD(GLM_FMA(GLM_MUL(xr, xx), GLM_FMA(xx, kSn5, kSn3), dx), xr);
    const double pc = GLM_MUL(xx, GLM_FMA(GLM_FMA(xx, kCs6, kCs4), xx, kCs2));
    const double c = GLM_FMA(dx, xr, pc);
    const double cor = GLM_FMA(s, t.cs, GLM_FMA(neg(c), t.sn, GLM_FMA(s, t.ccs, t.ssn)));
    return GLM_ADD(cor, t.sn);
}

// do_cos's table branch on x = x'' + dx (already summed by the caller).
GLM_FN double cos_tab(const Row& t, double x) {
    const double xx = GLM_MUL(x, x);
    const double s = GLM_FMA(GLM_MUL(x, xx), GLM_FMA(xx, kSn5, kSn3), x);
    const double c = GLM_MUL(xx, GLM_FMA(GLM_FMA(xx, kCs6, kCs4), xx, kCs2));
    const double cor =
        GLM_FMA(neg(s), t.sn, GLM_FMA(neg(c), t.cs, GLM_FMA(neg(s), t.ssn, t.ccs)));
    return GLM_ADD(cor, t.cs);
}

// sincos(x) for finite |x| < 105414350 (glibc's reduce_sincos range). Returns false outside.
GLM_FN bool sincos_fma(double x, double* sinx, double* cosx) {
    const uint32_t k = static_cast<uint32_t>(bits(x) >> 32) & 0x7fffffffu;
    const double ax = copysign_of(x, 0.0);
    if (k <= 0x3e3fffffu) {  // |x| < 2^-27
        *sinx = x;
        *cosx = 1.0;
        return true;
    }
    if (k <= 0x3feb5fffu) {  // |x| < 0.855469: do_sin(x, 0), do_cos(x, 0)
        const Row t = row_of(ax);
        if (ax < 0.126) {
            *sinx = taylor_sin(x, 0.0);
        } else {
            const double dx = x > 0.0 ? 0.0 : -0.0;
            *sinx = copysign_of(sin_tab(t, dx), x);
        }
        const double dxc = x >= 0.0 ? 0.0 : -0.0;
        *cosx = cos_tab(t, GLM_ADD(dxc, t.xr));
        return true;
    }
    if (k <= 0x400368fcu) {  // |x| < 2.426265: a + da = π/2 − |x|
        const double y = GLM_SUB(kHp0, ax);
        const double a = GLM_ADD(y, kHp1);
        const double da = GLM_ADD(GLM_SUB(y, a), kHp1);
        const double aa = copysign_of(a, 0.0);
        const Row t = row_of(aa);
        const double dxs = a < 0.0 ? neg(da) : da;
        *sinx = copysign_of(cos_tab(t, GLM_ADD(t.xr, dxs)), x);
        if (aa < 0.126) {
            *cosx = taylor_sin(a, da);
        } else {
            const double dxc = a <= 0.0 ? neg(da) : da;
            *cosx = copysign_of(sin_tab(t, dxc), a);
        }
        return true;
    }
    if (k > 0x419921fau)
        return false;
    // reduce_sincos: x = xn·π/2 + (a + da)
    const double tt = GLM_FMA(x, kHpinv, kToint);
    const double xn = GLM_SUB(tt, kToint);
    const uint32_t n = static_cast<uint32_t>(bits(tt)) & 3u;
    const double y = GLM_FMA(neg(xn), kMp2, GLM_FMA(neg(xn), kMp1, x));
    const double t2 = GLM_FMA(neg(xn), kPp3, y);
    double db = GLM_FMA(neg(kPp3), xn, GLM_SUB(y, t2));
    const double b = GLM_FMA(neg(xn), kPp4, t2);
    db = GLM_ADD(db, GLM_FMA(neg(xn), kPp4, GLM_SUB(t2, b)));
    double a = b, da = db;
    if (n == 1 || n == 2) {
        a = neg(a);
        da = neg(da);
    }
    const double aa = copysign_of(a, 0.0);
    const Row t = row_of(aa);
    double r1;  // do_sin(a, da)
    if (aa < 0.126) {
        r1 = taylor_sin(a, da);
    } else {
        const double dx = a <= 0.0 ? neg(da) : da;
        r1 = copysign_of(sin_tab(t, dx), a);
    }
    const double dxc = a < 0.0 ? neg(da) : da;
    double r2 = cos_tab(t, GLM_ADD(dxc, t.xr));  // do_cos(a, da)
    if (n & 2u)
        r2 = neg(r2);
    if (n & 1u) {
        *cosx = r1;
        *sinx = r2;
    } else {
        *sinx = r1;
        *cosx = r2;
    }
    return true;
}

// Order-free checksum term of one Box-Muller pair q with outputs (g0, g1) given as bits:
// the GPU and host checkers (rng_mt64.cu k_bm_hash, tests/cpp/bm_libm_check.cpp) sum these.
GLM_FN uint64_t pair_hash(uint64_t q, uint64_t g0, uint64_t g1) {
    uint64_t z = g0 ^ ((g1 << 29) | (g1 >> 35)) ^ (q * 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdULL;
    z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ULL;
    return z ^ (z >> 33);
}

}  // namespace glm

// Double-double arithmetic and correctly rounded log / sin / cos for the GPU
// Box-Muller transform.
//
// The reference's Gaussian (random_gen.cpp:41-53) is
//     u1 = 1 - U, u2 = U;  r = sqrt(-2 log u1);  a = (2 pi) u2;  g = r cos a, r sin a
// with glibc's libm.  Every step except log/sin/cos is a single IEEE operation the
// GPU reproduces exactly (sqrt is correctly rounded on sm_100a; products are
// computed with __dmul_rn so nothing is contracted).  log, sin and cos are computed
// here to ~2^-100 relative accuracy and rounded once, i.e. correctly rounded; glibc
// 2.39 is within ~0.52 ulp, so the two agree except on the ~0.16% of entries where
// glibc itself is not correctly rounded.  Tables of log(1+i/64)
// and sin/cos(j/64) as double-doubles come from tools/gen_dd_tables.py.
#pragma once

#include <cuda_runtime.h>

namespace rl {

#include "dd_tables.inc"

struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_add_d(dd a, double b) {
    dd s = two_sum(a.hi, b);
    s.lo = __dadd_rn(s.lo, a.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, p.lo));
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = __fma_rn(a.lo, b, p.lo);
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
    double q1 = __ddiv_rn(a.hi, b.hi);
    dd r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
    double q2 = __ddiv_rn(r.hi, b.hi);
    r = dd_add(r, dd_neg(dd_mul_d(b, q2)));
    double q3 = __ddiv_rn(r.hi, b.hi);
    dd q = quick_two_sum(q1, q2);
    return dd_add_d(q, q3);
}

// log(x) for x in (0, 1], correctly rounded (with overwhelming probability).
__device__ __forceinline__ double cr_log_unit(double x) {
    // (x == 1 needs no special case: m = 1, e = 0, i = 0, f = 0 give exactly 0)
    int e;
    double m = frexp(x, &e); // x = m 2^e, m in [0.5, 1)
    m = __dmul_rn(m, 2.0);   // m in [1, 2)
    e -= 1;
    int i = __double2int_rn(__dmul_rn(__dsub_rn(m, 1.0), 64.0));
    double c = __dadd_rn(1.0, __dmul_rn(static_cast<double>(i), 0.015625)); // exact
    double f = __dsub_rn(m, c);                                             // exact, |f| <= 1/128
    // log(m) = log(c) + 2 atanh(s), s = f / (2c + f)
    dd den = two_sum(__dmul_rn(2.0, c), f);
    // s = f / den to ~2^-104: one Newton correction of the double quotient
    const double s_hi = __ddiv_rn(f, den.hi);
    dd prod = two_prod(s_hi, den.hi);
    const double rem = __dsub_rn(__dsub_rn(f, prod.hi), __fma_rn(s_hi, den.lo, prod.lo));
    dd s = quick_two_sum(s_hi, __ddiv_rn(rem, den.hi));
    dd z = dd_mul(s, s);
    // atanh(s)/s = sum z^k / (2k+1), |z| <= 2^-16: 7 terms reach 2^-112
    const double inv[8] = {1.0, 1.0 / 3, 1.0 / 5, 1.0 / 7, 1.0 / 9, 1.0 / 11, 1.0 / 13, 1.0 / 15};
    // high-order tail in double, low-order terms in double-double
    double tail = inv[7];
    for (int k = 6; k >= 3; --k)
        tail = __fma_rn(tail, z.hi, inv[k]);
    dd p = dd_mul({tail, 0.0}, z);
    p = dd_mul(dd_add(p, {RL_INV5_HI, RL_INV5_LO}), z);
    p = dd_mul(dd_add(p, {RL_INV3_HI, RL_INV3_LO}), z);
    p = dd_add_d(p, 1.0);
    dd lg = dd_mul(dd_mul_d(s, 2.0), p);
    dd ec = two_prod(static_cast<double>(e), RL_LN2_HI);
    ec = dd_add_d(ec, __dmul_rn(static_cast<double>(e), RL_LN2_LO));
    double2 t = kLogTab[i];
    dd acc = dd_add(dd_add({t.x, t.y}, lg), ec);
    return __dadd_rn(acc.hi, acc.lo);
}

// sin and cos of a double, correctly rounded (with overwhelming probability),
// for |a| < 2^20.
__device__ __forceinline__ void cr_sincos(double a, double* sn, double* cs) {
    double kd = rint(__dmul_rn(a, 0.63661977236758138)); // 2/pi
    // r = a - k pi/2 in double-double with a 3-part pi/2 (exact products)
    dd p1 = two_prod(kd, RL_PIO2_1);
    dd r = two_sum(a, -p1.hi);
    r = dd_add_d(r, -p1.lo);
    dd p2 = two_prod(kd, RL_PIO2_2);
    r = dd_add(r, dd_neg(p2));
    r = dd_add_d(r, -__dmul_rn(kd, RL_PIO2_3));
    int q = static_cast<int>(kd) & 3;
    // r = j/64 + d, |d| <= 1/128
    double ar = fabs(r.hi);
    int j = __double2int_rn(__dmul_rn(ar, 64.0));
    double sg = r.hi < 0 ? -1.0 : 1.0;
    dd d = dd_add_d(r, -sg * __dmul_rn(static_cast<double>(j), 0.015625));
    dd d2 = dd_mul(d, d);
    // sin(d) = d (1 - d2/3! + d2^2/5! - ...),  cos(d) = 1 - d2/2! + d2^2/4! - ...
    double ts = -1.0 / 39916800.0, tc = 1.0 / 479001600.0;
    ts = __fma_rn(ts, d2.hi, 1.0 / 362880.0);
    tc = __fma_rn(tc, d2.hi, -1.0 / 3628800.0);
    ts = __fma_rn(ts, d2.hi, -1.0 / 5040.0);
    tc = __fma_rn(tc, d2.hi, 1.0 / 40320.0);
    dd ps = dd_mul({ts, 0.0}, d2);
    dd pc = dd_mul({tc, 0.0}, d2);
    ps = dd_mul(dd_add(ps, {RL_INV120_HI, RL_INV120_LO}), d2);
    pc = dd_mul(dd_add(pc, {-RL_INV720_HI, -RL_INV720_LO}), d2);
    ps = dd_mul(dd_add(ps, {-RL_INV6_HI, -RL_INV6_LO}), d2);
    pc = dd_mul(dd_add(pc, {RL_INV24_HI, RL_INV24_LO}), d2);
    pc = dd_mul(dd_add_d(pc, -0.5), d2);
    ps = dd_add_d(ps, 1.0);
    dd sd = dd_mul(d, ps);   // sin(d)
    dd cd = dd_add_d(pc, 1.0); // cos(d)
    double2 s0 = kSinTab[j], c0 = kCosTab[j];
    dd S0 = {sg * s0.x, sg * s0.y}, C0 = {c0.x, c0.y};
    // sin(r) = sin(r0) cos d + cos(r0) sin d ; cos(r) = cos(r0) cos d - sin(r0) sin d
    dd sr = dd_add(dd_mul(S0, cd), dd_mul(C0, sd));
    dd cr = dd_add(dd_mul(C0, cd), dd_neg(dd_mul(S0, sd)));
    double srd = __dadd_rn(sr.hi, sr.lo), crd = __dadd_rn(cr.hi, cr.lo);
    // quadrant select without branches
    const double a0 = (q & 1) ? crd : srd, a1 = (q & 1) ? srd : crd;
    *sn = (q & 2) ? -a0 : a0;
    *cs = ((q + 1) & 2) ? -a1 : a1;
}

} // namespace rl

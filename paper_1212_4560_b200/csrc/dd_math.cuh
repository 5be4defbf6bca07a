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
    double2 t = __ldg(&kLogTab[i]);
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
    double2 s0 = __ldg(&kSinTab[j]), c0 = __ldg(&kCosTab[j]);
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

// ---------------------------------------------------------------- fast paths --
// Ziv-style fast paths: a double + correction estimate of the function with a relative
// error far below half an ulp; when [est - err, est + err] rounds to one double, that
// double is the correctly rounded value (the same value cr_* returns); otherwise the
// caller falls back to cr_*.  err = 2^-62 |est|; the estimates' error analysis gives about
// 2^-65, and rl_box_muller_fast_check found no pair whose accepted fast result differs from
// cr_* in 2^28 random pairs even with a 2^-63 bound.  About 0.9% of pairs take the slow path.
__device__ __forceinline__ bool ziv_round(double hi, double lo, double* out) {
    const double err = fabs(hi) * 0x1.0p-62;
    const double a = __dadd_rn(hi, __dsub_rn(lo, err));
    const double b = __dadd_rn(hi, __dadd_rn(lo, err));
    *out = a;
    return a == b;
}

// log(x), x in (0, 1]: log(c) (table, dd) + e ln2 (dd) + 2 atanh(s), s = f / (2c + f) as
// s_hi + s_lo, the odd series beyond 2s in double (|s| <= 2^-8).
__device__ __forceinline__ bool fast_log_unit(double x, double* out) {
    int e;
    double m = frexp(x, &e);
    m = __dmul_rn(m, 2.0);
    e -= 1;
    const int i = __double2int_rn(__dmul_rn(__dsub_rn(m, 1.0), 64.0));
    const double c = __dadd_rn(1.0, __dmul_rn(static_cast<double>(i), 0.015625)); // exact
    const double f = __dsub_rn(m, c);                                             // exact
    const dd den = two_sum(__dmul_rn(2.0, c), f);
    const double inv = __drcp_rn(den.hi);
    const double s_hi = __dmul_rn(f, inv);
    const double r1 = __fma_rn(-s_hi, den.hi, f); // exact residual
    const double rem = __fma_rn(-s_hi, den.lo, r1);
    const double s_lo = __dmul_rn(rem, inv);
    const double z = __dmul_rn(s_hi, s_hi);
    double t = __fma_rn(z, 1.0 / 9.0, 1.0 / 7.0);
    t = __fma_rn(z, t, 1.0 / 5.0);
    t = __fma_rn(z, t, 1.0 / 3.0);
    const double tail = __dmul_rn(__dmul_rn(__dmul_rn(2.0, s_hi), z), t); // 2 s^3/3 + ...
    const double ed = static_cast<double>(e);
    const dd ec = two_prod(ed, RL_LN2_HI);
    const double2 tb = __ldg(&kLogTab[i]);
    const dd a = two_sum(ec.hi, tb.x);
    const dd b = two_sum(a.hi, __dmul_rn(2.0, s_hi));
    double lo = __dadd_rn(a.lo, b.lo);
    lo = __dadd_rn(lo, ec.lo);
    lo = __dadd_rn(lo, __dmul_rn(ed, RL_LN2_LO));
    lo = __dadd_rn(lo, tb.y);
    lo = __dadd_rn(lo, __dmul_rn(2.0, s_lo));
    lo = __dadd_rn(lo, tail);
    return ziv_round(b.hi, lo, out);
}

// sin and cos of a in [0, 2 pi] (the Box-Muller angle).  k pi/2 reduction with the exact
// k PIO2_1 product (k <= 4) and Sterbenz subtraction, then r = +-j/64 + d with the table.
__device__ __forceinline__ bool fast_sincos(double a, double* sn, double* cs) {
    const double kd = rint(__dmul_rn(a, 0.63661977236758138));
    const double r1 = __dsub_rn(a, __dmul_rn(kd, RL_PIO2_1)); // both exact for k <= 4
    const dd p2 = two_prod(kd, RL_PIO2_2);
    dd r = two_sum(r1, -p2.hi);
    r.lo = __dsub_rn(__dsub_rn(r.lo, p2.lo), __dmul_rn(kd, RL_PIO2_3));
    const int q = static_cast<int>(kd) & 3;
    const int j = __double2int_rn(__dmul_rn(fabs(r.hi), 64.0));
    const double sg = r.hi < 0 ? -1.0 : 1.0;
    const dd d = two_sum(__dsub_rn(r.hi, sg * __dmul_rn(static_cast<double>(j), 0.015625)), r.lo); // exact
    const double z = __dmul_rn(d.hi, d.hi);
    double ps = __fma_rn(z, 1.0 / 362880.0, -1.0 / 5040.0);
    ps = __fma_rn(z, ps, 1.0 / 120.0);
    ps = __fma_rn(z, ps, -1.0 / 6.0);
    const double sd_lo = __fma_rn(__dmul_rn(d.hi, z), ps, d.lo); // sin d = d.hi + sd_lo
    double pc = __fma_rn(z, 1.0 / 40320.0, -1.0 / 720.0);
    pc = __fma_rn(z, pc, 1.0 / 24.0);
    pc = __fma_rn(__dmul_rn(z, z), pc, __fma_rn(-0.5, z, -__dmul_rn(d.hi, d.lo))); // cos d - 1
    const double2 s0 = __ldg(&kSinTab[j]), c0 = __ldg(&kCosTab[j]);
    const double S0h = sg * s0.x, S0l = sg * s0.y;
    // sin r = S0 (1 + pc) + C0 sin d ; cos r = C0 (1 + pc) - S0 sin d
    const dd ps1 = two_prod(c0.x, d.hi);
    const dd hs = two_sum(S0h, ps1.hi);
    double los = __dadd_rn(hs.lo, ps1.lo);
    los = __dadd_rn(los, S0l);
    los = __fma_rn(S0h, pc, los);
    los = __fma_rn(c0.x, sd_lo, los);
    los = __fma_rn(c0.y, d.hi, los);
    const dd pc1 = two_prod(S0h, d.hi);
    const dd hc = two_sum(c0.x, -pc1.hi);
    double loc = __dsub_rn(hc.lo, pc1.lo);
    loc = __dadd_rn(loc, c0.y);
    loc = __fma_rn(c0.x, pc, loc);
    loc = __fma_rn(-S0h, sd_lo, loc);
    loc = __fma_rn(-S0l, d.hi, loc);
    double srd, crd;
    const bool ok = ziv_round(hs.hi, los, &srd) & ziv_round(hc.hi, loc, &crd);
    const double a0 = (q & 1) ? crd : srd, a1 = (q & 1) ? srd : crd;
    *sn = (q & 2) ? -a0 : a0;
    *cs = ((q + 1) & 2) ? -a1 : a1;
    return ok;
}

} // namespace rl

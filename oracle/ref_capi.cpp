// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrappers over the UNMODIFIED reference library (randla, compiled
// from /root/reference/proj/src/{matrix,random_gen,structured,genp}.cpp by
// oracle/Makefile into oracle/_ref/librandla_ref.so).  Tests use it to pin the
// C restatement (oracle/rl_oracle.c) and to generate golden fixtures; bench.py's
// `--impl reference` arm times it as the CPU baseline ("kind": "reference").
//
// Status codes are the same enum as include/rl_b200.h (rl_status): each maps
// 1:1 onto a randla::Error subclass of proj/include/randla/errors.hpp:9-59.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "randla/errors.hpp"
#include "randla/genp.hpp"
#include "randla/matrix.hpp"
#include "randla/random_gen.hpp"
#include "randla/structured.hpp"
#include "randla/dense_core.hpp"
#include "randla/lowrank.hpp"

using namespace randla;

namespace {
thread_local std::string g_msg;

int code_of(const std::exception& e) {
    g_msg = e.what();
    if (dynamic_cast<const DimensionMismatch*>(&e)) return 1;
    if (dynamic_cast<const InvalidArgument*>(&e)) return 2;
    if (dynamic_cast<const PivotBreakdown*>(&e)) return 3;
    if (dynamic_cast<const RankDeficient*>(&e)) return 4;
    if (dynamic_cast<const Degenerate*>(&e)) return 5;
    if (dynamic_cast<const LengthNotPowerOfTwo*>(&e)) return 6;
    if (dynamic_cast<const IndexOutOfRange*>(&e)) return 7;
    if (dynamic_cast<const NoConvergence*>(&e)) return 8;
    if (dynamic_cast<const ZeroMatrix*>(&e)) return 9;
    if (dynamic_cast<const ConstructionFailed*>(&e)) return 10;
    if (dynamic_cast<const Error*>(&e)) return 11;
    return 99;
}

#define GUARD_BEGIN try {
#define GUARD_END                          \
    }                                      \
    catch (const std::exception& e) {      \
        return code_of(e);                 \
    }                                      \
    return 0;

Matrix mat(std::size_t r, std::size_t c, const double* p) {
    Matrix m(r, c); // non-validating ctor (matrix.cpp:8-11): failed GENP output may be non-finite
    std::memcpy(m.data().data(), p, r * c * sizeof(double));
    return m;
}

void put(const Matrix& m, double* out) {
    std::memcpy(out, m.data().data(), m.data().size() * sizeof(double));
}

rnd::MultiplierKind kind_of(int tag, double mu, double sigma) {
    rnd::MultiplierKind k;
    k.tag = static_cast<rnd::MultiplierTag>(tag);
    k.mu = mu;
    k.sigma = sigma;
    return k;
}
} // namespace

extern "C" {

const char* rlref_last_error(void) { return g_msg.c_str(); }

// kind: 0 uniform01, 1 uniform_pm1, 2 gaussian, 3 sign, 4 uniform_int(lo, hi)
int rlref_draws(uint64_t seed, uint64_t sid, int kind, uint64_t count, int64_t lo, int64_t hi,
                double* out) {
    GUARD_BEGIN
    rnd::Rng r(rnd::RngStream{seed, sid});
    for (uint64_t i = 0; i < count; ++i) {
        switch (kind) {
        case 0: out[i] = r.uniform01(); break;
        case 1: out[i] = r.uniform_pm1(); break;
        case 2: out[i] = r.gaussian(); break;
        case 3: out[i] = r.sign(); break;
        default: out[i] = static_cast<double>(r.uniform_int(lo, hi)); break;
        }
    }
    GUARD_END
}

// Raw int64 draws of uniform_int (exact, no double rounding).
int rlref_uniform_int(uint64_t seed, uint64_t sid, uint64_t count, int64_t lo, int64_t hi,
                      int64_t* out) {
    GUARD_BEGIN
    rnd::Rng r(rnd::RngStream{seed, sid});
    for (uint64_t i = 0; i < count; ++i)
        out[i] = r.uniform_int(lo, hi);
    GUARD_END
}

int rlref_gaussian_matrix(uint64_t m, uint64_t n, double mu, double sigma, uint64_t seed,
                          uint64_t sid, double* out) {
    GUARD_BEGIN
    put(rnd::gaussian_matrix(m, n, mu, sigma, rnd::RngStream{seed, sid}), out);
    GUARD_END
}

int rlref_uniform_matrix(uint64_t m, uint64_t n, uint64_t seed, uint64_t sid, double* out) {
    GUARD_BEGIN
    put(rnd::uniform_matrix(m, n, rnd::RngStream{seed, sid}), out);
    GUARD_END
}

// first_col has m entries, first_row n entries (Toeplitz only; may be null otherwise).
int rlref_random_structured(int tag, double mu, double sigma, uint64_t m, uint64_t n,
                            uint64_t seed, uint64_t sid, double* first_col, double* first_row) {
    GUARD_BEGIN
    auto s = rnd::random_structured(kind_of(tag, mu, sigma), m, n, rnd::RngStream{seed, sid});
    std::memcpy(first_col, s.first_col.data(), s.first_col.size() * sizeof(double));
    if (first_row && !s.first_row.empty())
        std::memcpy(first_row, s.first_row.data(), s.first_row.size() * sizeof(double));
    GUARD_END
}

int rlref_householder_sign(uint64_t n, uint64_t seed, uint64_t sid, double* out) {
    GUARD_BEGIN
    put(rnd::householder_sign(n, rnd::RngStream{seed, sid}), out);
    GUARD_END
}

int rlref_matmul(uint64_t m, uint64_t k, uint64_t n, const double* a, const double* b, double* c) {
    GUARD_BEGIN
    put(mat(m, k, a).multiply(mat(k, n, b)), c);
    GUARD_END
}

int rlref_matvec(uint64_t m, uint64_t n, const double* a, const double* x, double* y) {
    GUARD_BEGIN
    auto v = mat(m, n, a).multiply(std::span<const double>(x, n));
    std::memcpy(y, v.data(), m * sizeof(double));
    GUARD_END
}

// Circulant spec * dense (structured.cpp:178-189), spec given by first column.
int rlref_circulant_multiply_matrix(uint64_t n, const double* first_col, uint64_t cols,
                                    const double* a, double* out) {
    GUARD_BEGIN
    auto spec = structured::StructuredSpec::circulant(std::vector<double>(first_col, first_col + n));
    put(structured::multiply_matrix(spec, mat(n, cols, a)), out);
    GUARD_END
}

int rlref_circ_mul(uint64_t n, const double* first_col, const double* x, double* y) {
    GUARD_BEGIN
    auto spec = structured::StructuredSpec::circulant(std::vector<double>(first_col, first_col + n));
    auto v = structured::circ_mul(spec, std::span<const double>(x, n));
    std::memcpy(y, v.data(), n * sizeof(double));
    GUARD_END
}

int rlref_toeplitz_mul(uint64_t m, uint64_t n, const double* col, const double* row,
                       const double* x, double* y) {
    GUARD_BEGIN
    auto spec = structured::StructuredSpec::toeplitz(std::vector<double>(col, col + m),
                                                     std::vector<double>(row, row + n));
    auto v = structured::toeplitz_mul(spec, std::span<const double>(x, n));
    std::memcpy(y, v.data(), m * sizeof(double));
    GUARD_END
}

int rlref_toeplitz_multiply_matrix(uint64_t m, uint64_t n, const double* col, const double* row, uint64_t cols,
                                   const double* a, double* out) {
    GUARD_BEGIN
    auto spec = structured::StructuredSpec::toeplitz(std::vector<double>(col, col + m),
                                                     std::vector<double>(row, row + n));
    put(structured::multiply_matrix(spec, mat(n, cols, a)), out);
    GUARD_END
}

// Complex interleaved (re, im) in/out; dir 0 forward, 1 inverse.
int rlref_fft(uint64_t n, const double* in, int dir, double* out) {
    GUARD_BEGIN
    std::vector<std::complex<double>> x(n);
    for (uint64_t i = 0; i < n; ++i)
        x[i] = {in[2 * i], in[2 * i + 1]};
    auto y = structured::fft(x, dir ? structured::FftDirection::Inverse
                                    : structured::FftDirection::Forward);
    for (uint64_t i = 0; i < n; ++i) {
        out[2 * i] = y[i].real();
        out[2 * i + 1] = y[i].imag();
    }
    GUARD_END
}

int rlref_genp_factor(uint64_t n, const double* a, double pivot_floor, double* l, double* u,
                      double* pivots, double* pmin_pmax) {
    GUARD_BEGIN
    auto f = genp::genp_factor(mat(n, n, a), pivot_floor);
    put(f.L, l);
    put(f.U, u);
    std::memcpy(pivots, f.pivot_abs.data(), n * sizeof(double));
    pmin_pmax[0] = f.pivot_min;
    pmin_pmax[1] = f.pivot_max;
    GUARD_END
}

int rlref_block_ge(uint64_t n, const double* a, uint64_t block, double* l, double* u,
                   double* pnorms, double* pinv_norms) {
    GUARD_BEGIN
    auto f = genp::block_ge(mat(n, n, a), block);
    put(f.L, l);
    put(f.U, u);
    std::memcpy(pnorms, f.pivot_block_norms.data(), f.pivot_block_norms.size() * sizeof(double));
    std::memcpy(pinv_norms, f.pivot_block_inv_norms.data(),
                f.pivot_block_inv_norms.size() * sizeof(double));
    GUARD_END
}

int rlref_genp_solve(uint64_t n, const double* l, const double* u, const double* b, double* y) {
    GUARD_BEGIN
    genp::GenpFactorization f{mat(n, n, l), mat(n, n, u), {}, 0.0, 0.0};
    auto v = genp::genp_solve(f, std::span<const double>(b, n));
    std::memcpy(y, v.data(), n * sizeof(double));
    GUARD_END
}

// report: residual, raw_residual, pivot_min, pivot_max, raw_pivot_min, raw_pivot_max
int rlref_randomized_genp(uint64_t n, const double* a, const double* b, int tag, double mu,
                          double sigma, int side, int refine, uint64_t seed, uint64_t sid,
                          double* y, double* report) {
    GUARD_BEGIN
    auto r = genp::randomized_genp(mat(n, n, a), std::span<const double>(b, n),
                                   kind_of(tag, mu, sigma), static_cast<genp::MulSide>(side),
                                   refine, rnd::RngStream{seed, sid});
    std::memcpy(y, r.first.data(), n * sizeof(double));
    report[0] = r.second.residual;
    report[1] = r.second.raw_residual;
    report[2] = r.second.pivot_min;
    report[3] = r.second.pivot_max;
    report[4] = r.second.raw_pivot_min;
    report[5] = r.second.raw_pivot_max;
    GUARD_END
}

int rlref_illblock_system(uint64_t n, uint64_t seed, uint64_t sid, double* a, double* b,
                          double* y) {
    GUARD_BEGIN
    auto s = rnd::illblock_system(n, rnd::RngStream{seed, sid});
    put(s.A, a);
    std::memcpy(b, s.b.data(), n * sizeof(double));
    std::memcpy(y, s.y_true.data(), n * sizeof(double));
    GUARD_END
}

int rlref_qr_positive(uint64_t m, uint64_t n, const double* a, double* q, double* r) {
    GUARD_BEGIN
    auto f = dense::qr_positive(mat(m, n, a));
    put(f.Q, q);
    put(f.R, r);
    GUARD_END
}

int rlref_singular_values(uint64_t m, uint64_t n, const double* a, double* sigma) {
    GUARD_BEGIN
    auto f = dense::svd(mat(m, n, a));
    std::memcpy(sigma, f.sigma.data(), f.sigma.size() * sizeof(double));
    GUARD_END
}

// lowrank::proto_lowrank (lowrank.cpp:108-177). approx: m x n; basis: n x rho (up to n x rho_plus
// capacity, `basis_cols` receives its column count); out: rho, ok.
int rlref_proto_lowrank(uint64_t m, uint64_t n, const double* a, uint64_t rho_plus, double tau,
                        double tau_prime, int tag, double mu, double sigma, uint64_t seed, uint64_t sid,
                        uint64_t* rho, double* approx, double* basis, uint64_t* basis_cols,
                        double* residual, int* ok) {
    GUARD_BEGIN
    auto r = lowrank::proto_lowrank(mat(m, n, a), rho_plus, tau, tau_prime, kind_of(tag, mu, sigma),
                                    rnd::RngStream{seed, sid});
    *rho = r.rho;
    put(r.approx, approx);
    put(r.basis, basis);
    *basis_cols = r.basis.cols();
    *residual = r.residual;
    *ok = r.ok ? 1 : 0;
    GUARD_END
}

// lowrank::nrank_search (lowrank.cpp:360-396); basis: n x rho of the wide-side work matrix
// (capacity n x rho_plus).
int rlref_nrank_search(uint64_t m, uint64_t n, const double* a, uint64_t rho_minus, uint64_t rho_plus,
                       double kappa, int policy, uint64_t seed, uint64_t sid, uint64_t* rho, double* basis,
                       uint64_t* basis_rows, uint64_t* basis_cols) {
    GUARD_BEGIN
    auto r = lowrank::nrank_search(mat(m, n, a), rho_minus, rho_plus, kappa,
                                   static_cast<lowrank::SearchPolicy>(policy), rnd::RngStream{seed, sid});
    *rho = r.rho;
    put(r.basis, basis);
    *basis_rows = r.basis.rows();
    *basis_cols = r.basis.cols();
    GUARD_END
}

// lowrank::extremal_sv_estimate (lowrank.cpp:204-348); method 0 = Power, 1 = Lanczos.
int rlref_extremal_sv_estimate(uint64_t m, uint64_t n, const double* a, int method, int iters, uint64_t seed,
                               uint64_t sid, double* sv_max, double* sv_min) {
    GUARD_BEGIN
    auto e = lowrank::extremal_sv_estimate(mat(m, n, a), static_cast<lowrank::SvMethod>(method), iters,
                                           rnd::RngStream{seed, sid});
    *sv_max = e.sv_max;
    *sv_min = e.sv_min;
    GUARD_END
}

// lowrank::cond_probe (lowrank.cpp:350-358).
int rlref_cond_probe(uint64_t m, uint64_t n, const double* b, double kappa, int method, int iters,
                     uint64_t seed, uint64_t sid, int* pass) {
    GUARD_BEGIN
    *pass = lowrank::cond_probe(mat(m, n, b), kappa, static_cast<lowrank::SvMethod>(method), iters,
                                rnd::RngStream{seed, sid}) ? 1 : 0;
    GUARD_END
}

// lowrank::power_transform (lowrank.cpp:179-187): (A A^T)^h A.
int rlref_power_transform(uint64_t m, uint64_t n, const double* a, unsigned h, double* out) {
    GUARD_BEGIN
    put(lowrank::power_transform(mat(m, n, a), h), out);
    GUARD_END
}

// lowrank::sampled_residual_check (lowrank.cpp:189-202).
int rlref_sampled_residual_check(uint64_t m, uint64_t n, const double* a, const double* ahat, uint64_t rho1,
                                 uint64_t rho2, double tau, uint64_t seed, uint64_t sid, int* pass) {
    GUARD_BEGIN
    *pass = lowrank::sampled_residual_check(mat(m, n, a), mat(m, n, ahat), rho1, rho2, tau,
                                            rnd::RngStream{seed, sid}) ? 1 : 0;
    GUARD_END
}

} // extern "C"

extern "C" int rlref_profile_matrix_paper(uint64_t n, uint64_t rho, uint64_t seed, uint64_t sid, double* out) {
    try {
        auto s = randla::rnd::paper_sigma_profile(n, rho);
        auto m = randla::rnd::profile_matrix(n, s, randla::rnd::RngStream{seed, sid});
        std::memcpy(out, m.data().data(), n * n * sizeof(double));
    } catch (const std::exception& e) {
        return code_of(e);
    }
    return 0;
}

extern "C" int rlref_profile_matrix(uint64_t n, const double* sigmas, uint64_t seed, uint64_t sid, double* out) {
    try {
        auto m = randla::rnd::profile_matrix(n, std::span<const double>(sigmas, n), randla::rnd::RngStream{seed, sid});
        std::memcpy(out, m.data().data(), n * n * sizeof(double));
    } catch (const std::exception& e) {
        return code_of(e);
    }
    return 0;
}

extern "C" int rlref_random_orthogonal(uint64_t n, uint64_t seed, uint64_t sid, double* out) {
    try {
        auto m = randla::rnd::random_orthogonal(n, randla::rnd::RngStream{seed, sid});
        std::memcpy(out, m.data().data(), n * n * sizeof(double));
    } catch (const std::exception& e) {
        return code_of(e);
    }
    return 0;
}


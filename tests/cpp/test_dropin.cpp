// The reference's own hot-path test cases (proj/tests/test_genp.cpp, test_random_gen.cpp,
// test_structured.cpp, test_dense_core.cpp, test_lowrank.cpp), re-hosted against the B200
// drop-in (include/randla/*.hpp -> librandla_b200.so -> librl_b200.so).  Same calls, same
// seeds, same tolerances.  Exit status = number of failed checks.
#include <cmath>
#include <cstdio>
#include <vector>

#include "randla/dense_core.hpp"
#include "randla/genp.hpp"
#include "randla/lowrank.hpp"
#include "randla/random_gen.hpp"
#include "randla/structured.hpp"

using namespace randla;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                \
    do {                                                                           \
        if (cond)                                                                  \
            ++g_pass;                                                              \
        else {                                                                     \
            ++g_fail;                                                              \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
        }                                                                          \
    } while (0)
#define CHECK_THROWS_AS(expr, E)                                                   \
    do {                                                                           \
        bool thrown = false;                                                       \
        try {                                                                      \
            (void)(expr);                                                          \
        } catch (const E&) {                                                       \
            thrown = true;                                                         \
        } catch (...) {                                                            \
        }                                                                          \
        CHECK(thrown);                                                             \
    } while (0)

static double rel_diff(const Matrix& a, const Matrix& b) {
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < a.data().size(); ++i) {
        num += (a.data()[i] - b.data()[i]) * (a.data()[i] - b.data()[i]);
        den += b.data()[i] * b.data()[i];
    }
    return std::sqrt(num) / std::max(std::sqrt(den), 1e-300);
}

static Matrix naive(const Matrix& a, const Matrix& b) {
    Matrix c(a.rows(), b.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < b.cols(); ++j) {
            double s = 0.0;
            for (std::size_t k = 0; k < a.cols(); ++k)
                s += a(i, k) * b(k, j);
            c(i, j) = s;
        }
    return c;
}

static double rel_residual(const Matrix& a, const std::vector<double>& y, const std::vector<double>& b) {
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < b.size(); ++i) {
        double s = 0.0;
        for (std::size_t j = 0; j < y.size(); ++j)
            s += a(i, j) * y[j];
        num += (s - b[i]) * (s - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / den);
}

static Matrix diag_dominant(std::size_t n, rnd::RngStream s) {
    Matrix a = rnd::uniform_matrix(n, n, s);
    for (std::size_t i = 0; i < n; ++i)
        a(i, i) = static_cast<double>(n) + 1.0;
    return a;
}

int main() {
    std::fprintf(stderr, "[dropin] random_gen\n");
    // ---- random_gen (test_random_gen.cpp) ----
    {
        rnd::Rng a({7, 3}), b({7, 3}), c({7, 4});
        bool all_equal = true, any_diff = false;
        for (int i = 0; i < 100; ++i) {
            double va = a.uniform01(), vb = b.uniform01(), vc = c.uniform01();
            all_equal = all_equal && va == vb;
            any_diff = any_diff || va != vc;
        }
        CHECK(all_equal);
        CHECK(any_diff);
        rnd::Rng r({7, 5});
        bool ok = true;
        for (int i = 0; i < 1000; ++i) {
            auto v = r.uniform_int(1, 6);
            double s = r.sign();
            ok = ok && v >= 1 && v <= 6 && (s == 1.0 || s == -1.0);
        }
        CHECK(ok);
        CHECK_THROWS_AS(r.uniform_int(3, 2), InvalidArgument);
        Matrix g1 = rnd::gaussian_matrix(4, 4, 0.0, 1.0, {11, 0}), g2 = rnd::gaussian_matrix(4, 4, 0.0, 1.0, {11, 0});
        CHECK(g1.data() == g2.data());
        CHECK_THROWS_AS(rnd::gaussian_matrix(2, 2, 0.0, 0.0, {11, 0}), InvalidArgument);
        Matrix u = rnd::uniform_matrix(500, 500, {11, 1});
        double sum = 0.0;
        bool range = true;
        for (double v : u.data()) {
            range = range && v >= -1.0 && v < 1.0;
            sum += v;
        }
        CHECK(range);
        CHECK(std::fabs(sum / u.data().size()) < 0.01);
        // literal first draws (SURVEY.md §8(c) probe goldens)
        rnd::Rng p({1, 0});
        CHECK(p.uniform01() == 0.20959692852878609);
        CHECK(p.uniform01() == 0.12101183419625183);
        rnd::Rng q({1, 0});
        CHECK(q.gaussian() == 0.49698630815925782);
        CHECK(q.gaussian() == 0.47268287749077509);
        auto spec = rnd::random_structured({rnd::MultiplierTag::CirculantSign}, 8, 8, {1, 0});
        const double want[8] = {1, -1, -1, -1, 1, 1, -1, -1};
        bool same = true;
        for (int i = 0; i < 8; ++i)
            same = same && spec.first_col[i] == want[i];
        CHECK(same);
        Matrix h = rnd::householder_sign(12, {5, 5});
        CHECK(rel_diff(naive(h, h), h) < 1e-12); // idempotent (test_random_gen.cpp:99-109)
    }
    std::fprintf(stderr, "[dropin] structured\n");
    // ---- structured (test_structured.cpp) ----
    {
        auto c = structured::StructuredSpec::circulant({1.0, 2.0, 3.0});
        Matrix d = structured::densify(c);
        CHECK(d(0, 0) == 1.0 && d(1, 0) == 2.0 && d(0, 1) == 3.0);
        auto y = structured::circ_mul(structured::StructuredSpec::circulant({0.0, 1.0, 0.0}), std::vector<double>{1, 2, 3});
        CHECK(std::fabs(y[0] - 3) < 1e-14 && std::fabs(y[1] - 1) < 1e-14 && std::fabs(y[2] - 2) < 1e-14);
        std::vector<std::complex<double>> imp(8, 0.0);
        imp[0] = 1.0;
        auto f = structured::fft(imp, structured::FftDirection::Forward);
        bool ones = true;
        for (auto z : f)
            ones = ones && std::abs(z - 1.0) < 1e-14;
        CHECK(ones);
        CHECK_THROWS_AS(structured::fft(std::vector<std::complex<double>>(6), structured::FftDirection::Forward),
                        LengthNotPowerOfTwo);
        auto spec = rnd::random_structured({rnd::MultiplierTag::CirculantSign}, 64, 64, {9, 1});
        Matrix a = rnd::gaussian_matrix(64, 5, 0.0, 1.0, {9, 2});
        CHECK(rel_diff(structured::multiply_matrix(spec, a), naive(structured::densify(spec), a)) < 1e-10);
        auto t = structured::StructuredSpec::toeplitz({0.0, 5.0}, {0.0, 6.0});
        auto ty = structured::toeplitz_mul(t, std::vector<double>{1.0, 1.0});
        CHECK(std::fabs(ty[0] - 6.0) < 1e-14 && std::fabs(ty[1] - 5.0) < 1e-14);
    }
    std::fprintf(stderr, "[dropin] genp\n");
    // ---- genp (test_genp.cpp) ----
    {
        auto f = genp::genp_factor(Matrix::identity(4));
        CHECK(rel_diff(f.L, Matrix::identity(4)) == 0.0);
        CHECK(rel_diff(f.U, Matrix::identity(4)) == 0.0);
        CHECK(f.pivot_min == 1.0 && f.pivot_max == 1.0);
        CHECK_THROWS_AS(genp::genp_factor(Matrix::from_rows({{0.0, 1.0}, {1.0, 0.0}}), 1e-12), PivotBreakdown);
        Matrix a = diag_dominant(8, {31, 0});
        auto g = genp::genp_factor(a);
        CHECK(rel_diff(naive(g.L, g.U), a) < 1e-13);
        bool shape = true;
        for (std::size_t i = 0; i < 8; ++i) {
            shape = shape && g.L(i, i) == 1.0;
            for (std::size_t j = i + 1; j < 8; ++j)
                shape = shape && g.L(i, j) == 0.0;
            for (std::size_t j = 0; j < i; ++j)
                shape = shape && g.U(i, j) == 0.0;
        }
        CHECK(shape);
        CHECK(g.pivot_abs.size() == 8 && g.pivot_min <= g.pivot_max);
        auto fd = genp::genp_factor(Matrix::diagonal(std::vector<double>{2.0, 4.0}));
        auto y = genp::genp_solve(fd, std::vector<double>{2.0, 8.0});
        CHECK(std::fabs(y[0] - 1.0) < 1e-14 && std::fabs(y[1] - 2.0) < 1e-14);
        Matrix a12 = diag_dominant(12, {31, 1});
        auto bl = genp::block_ge(a12, 1);
        auto sc = genp::genp_factor(a12);
        CHECK(rel_diff(bl.L, sc.L) < 1e-12 && rel_diff(bl.U, sc.U) < 1e-12);
        CHECK(bl.pivot_block_norms.size() == 12);
        Matrix a6 = diag_dominant(6, {31, 2});
        auto b6 = genp::block_ge(a6, 6);
        CHECK(b6.pivot_block_norms.size() == 1 && rel_diff(naive(b6.L, b6.U), a6) < 1e-12);
        // iterative_refine: zero steps is the identity, one step improves
        Matrix a10 = diag_dominant(10, {31, 3});
        std::vector<double> bb(10);
        rnd::Rng r({31, 4});
        for (double& v : bb)
            v = r.uniform_pm1();
        auto f10 = genp::genp_factor(a10);
        auto y10 = genp::genp_solve(f10, bb);
        std::vector<double> bad = y10;
        for (double& v : bad)
            v += 1e-4;
        auto same = genp::iterative_refine(a10, f10, bad, bb, 0);
        CHECK(same == bad);
        auto better = genp::iterative_refine(a10, f10, bad, bb, 1);
        CHECK(rel_residual(a10, better, bb) < 1e-3 * rel_residual(a10, bad, bb));
        auto [yi, rep] = genp::randomized_genp(Matrix::identity(8), std::vector<double>(8, 1.0),
                                               {rnd::MultiplierTag::Gaussian}, genp::MulSide::Left, 0, {31, 5});
        CHECK(rel_residual(Matrix::identity(8), yi, std::vector<double>(8, 1.0)) < 1e-12 && rep.residual < 1e-12);
        CHECK_THROWS_AS(genp::randomized_genp(Matrix::identity(3), std::vector<double>(3, 1.0), {}, genp::MulSide::Right,
                                              3, {1, 1}),
                        InvalidArgument);
        // multi-RHS extension agrees with column-by-column solves
        Matrix B = rnd::gaussian_matrix(10, 3, 0.0, 1.0, {31, 6});
        Matrix X = genp::genp_solve(f10, B);
        bool cols = true;
        for (std::size_t j = 0; j < 3; ++j) {
            auto xj = genp::genp_solve(f10, B.column(j));
            for (std::size_t i = 0; i < 10; ++i)
                cols = cols && std::fabs(xj[i] - X(i, j)) < 1e-13;
        }
        CHECK(cols);
        // batched extension agrees with the per-system calls
        std::vector<Matrix> sys;
        std::vector<std::vector<double>> rhs;
        std::vector<std::uint64_t> ids;
        for (std::uint64_t t = 0; t < 6; ++t) {
            sys.push_back(rnd::gaussian_matrix(64, 64, 0.0, 1.0, {40, t}));
            rhs.push_back(rnd::gaussian_matrix(64, 1, 0.0, 1.0, {41, t}).data());
            ids.push_back(100 + t);
        }
        auto out = genp::randomized_genp_batched(sys, rhs, {rnd::MultiplierTag::CirculantSign}, genp::MulSide::Right,
                                                 0, 42, ids);
        bool agree = true;
        for (std::size_t t = 0; t < 6; ++t) {
            auto [ys, rs] = genp::randomized_genp(sys[t], rhs[t], {rnd::MultiplierTag::CirculantSign},
                                                  genp::MulSide::Right, 0, {42, ids[t]});
            for (std::size_t i = 0; i < 64; ++i)
                agree = agree && std::fabs(ys[i] - out[t].first[i]) <= 1e-8 * (1.0 + std::fabs(ys[i]));
        }
        CHECK(agree);
    }
    std::fprintf(stderr, "[dropin] dense core / lowrank\n");
    // ---- dense core / lowrank (test_dense_core.cpp, test_lowrank.cpp) ----
    {
        auto f = dense::qr_positive(Matrix::from_rows({{2.0, 0.0}, {0.0, 3.0}}));
        CHECK(rel_diff(f.Q, Matrix::identity(2)) < 1e-14);
        auto p = dense::qr_positive(Matrix::from_rows({{0.0, 1.0}, {1.0, 0.0}}));
        CHECK(rel_diff(p.R, Matrix::identity(2)) < 1e-14);
        Matrix rd(4, 2);
        for (std::size_t i = 0; i < 4; ++i) {
            rd(i, 0) = static_cast<double>(i + 1);
            rd(i, 1) = 2.0 * static_cast<double>(i + 1);
        }
        CHECK_THROWS_AS(dense::qr_positive(rd), RankDeficient);
        CHECK(dense::numerical_rank(Matrix::diagonal(std::vector<double>{1.0, 0.5, 1e-10}), 1e-6) == 2);
        CHECK(dense::numerical_rank(Matrix::identity(5), 1e-6) == 5);
        CHECK_THROWS_AS(dense::numerical_rank(Matrix::identity(3), 0.0), InvalidArgument);
        CHECK(std::fabs(dense::norm(Matrix::diagonal(std::vector<double>{3.0, 1.0}), dense::NormKind::Two) - 3.0) < 1e-12);
        CHECK(std::fabs(dense::cond2(Matrix::diagonal(std::vector<double>{1.0, 1e-9}), 1e-6) - 1.0) < 1e-12);
        // a rank-8 matrix: its Gaussian sketch spans the column space, projection recovers A
        Matrix U = rnd::gaussian_matrix(200, 8, 0.0, 1.0, {50, 1});
        Matrix V = rnd::gaussian_matrix(8, 60, 0.0, 1.0, {50, 2});
        Matrix A = U.multiply(V);
        Matrix Y = lowrank::approx_basis(A, 8, {rnd::MultiplierTag::Gaussian}, lowrank::SpaceSide::LeftSpace, {50, 3});
        CHECK(Y.rows() == 200 && Y.cols() == 8);
        Matrix Q = dense::qr_positive(Y).Q;
        CHECK(rel_diff(lowrank::project_onto_basis(A, Q, true, dense::Side::Left), A) < 1e-12);
        CHECK(rel_diff(lowrank::project_onto_basis(A, Y, false, dense::Side::Left), A) < 1e-12);
        Matrix Z = lowrank::approx_basis(A, 8, {rnd::MultiplierTag::Gaussian}, lowrank::SpaceSide::RightSpace, {50, 4});
        CHECK(Z.rows() == 60 && Z.cols() == 8);
        // the rank-search side (test_lowrank.cpp:116-177)
        for (auto method : {lowrank::SvMethod::Power, lowrank::SvMethod::Lanczos}) {
            auto est = lowrank::extremal_sv_estimate(Matrix::diagonal(std::vector<double>{5.0, 1.0}), method, 200,
                                                     rnd::RngStream{41, 15});
            CHECK(std::abs(est.sv_max - 5.0) < 1e-3 * 5.0);
            CHECK(std::abs(est.sv_min - 1.0) < 1e-3);
        }
        CHECK(lowrank::cond_probe(Matrix::identity(8), 1e6, lowrank::SvMethod::Power, 500, rnd::RngStream{41, 20}));
        {
            std::vector<double> sig(8, 1e-10);
            sig[0] = 1.0;
            CHECK(!lowrank::cond_probe(Matrix::diagonal(sig), 1e6, lowrank::SvMethod::Power, 500,
                                       rnd::RngStream{41, 21}));
        }
        CHECK(lowrank::nrank_search(Matrix(8, 8), 0, 8, 1e6, lowrank::SearchPolicy::Binary, rnd::RngStream{41, 28}).rho ==
              0);
        CHECK(lowrank::nrank_search(Matrix::identity(16), 0, 16, 1e6, lowrank::SearchPolicy::Binary,
                                    rnd::RngStream{41, 29})
                  .rho == 16);
        {
            Matrix d2 = Matrix::diagonal(std::vector<double>{2.0, 1.0});
            CHECK(rel_diff(lowrank::power_transform(d2, 0), d2) == 0.0);
            CHECK(rel_diff(lowrank::power_transform(d2, 1), Matrix::diagonal(std::vector<double>{8.0, 1.0})) < 1e-14);
        }
        // proto_lowrank (test_lowrank.cpp:72-91): the zero matrix, and a rank-8 matrix recovered
        auto z = lowrank::proto_lowrank(Matrix(4, 4), 2, 1e-8, 1e-6, {rnd::MultiplierTag::Gaussian, 0.0, 1.0},
                                        {41, 9});
        CHECK(z.ok && z.rho == 0);
        Matrix A2 = rnd::gaussian_matrix(64, 8, 0.0, 1.0, {50, 5}).multiply(rnd::gaussian_matrix(8, 48, 0.0, 1.0, {50, 6}));
        auto pl = lowrank::proto_lowrank(A2, 12, 1e-6, 1e-6, {rnd::MultiplierTag::Gaussian, 0.0, 1.0}, {41, 11});
        CHECK(pl.ok && pl.rho == 8 && pl.residual < 1e-6);
        CHECK(pl.basis.rows() == 48 && pl.basis.cols() == 8);
        CHECK(rel_diff(pl.approx, A2) < 1e-12);
        CHECK_THROWS_AS(lowrank::proto_lowrank(A2, 12, 1e-6, 2.0, {rnd::MultiplierTag::Gaussian, 0.0, 1.0}, {41, 11}),
                        InvalidArgument);
    }
    std::printf("drop-in checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}

// randla::dense (hot-path subset) and randla::lowrank on the B200 C-ABI
// (reference semantics: proj/src/dense_core.cpp:48-186, proj/src/lowrank.cpp:45-106).
#include <algorithm>
#include <limits>

#include "randla/dense_core.hpp"
#include "randla/lowrank.hpp"
#include "rl_b200.h"

namespace randla {

using detail::check;

namespace dense {

double norm(const Matrix& a, NormKind kind) {
    const int k = kind == NormKind::One ? 0 : kind == NormKind::Two ? 1 : kind == NormKind::Inf ? 2 : 3;
    double out = 0.0;
    check(rl_norm(a.rows(), a.cols(), a.data().data(), k, &out));
    return out;
}

QrFactors qr_positive(const Matrix& a) {
    if (a.rows() < a.cols())
        throw InvalidArgument("qr_positive: requires rows >= cols");
    Matrix q(a.rows(), a.cols()), r(a.cols(), a.cols());
    check(rl_qr_positive(a.rows(), a.cols(), a.data().data(), q.data().data(), r.data().data()));
    return QrFactors{std::move(q), std::move(r)};
}

std::vector<double> singular_values(const Matrix& a) {
    std::vector<double> sg(std::min(a.rows(), a.cols()));
    std::uint64_t rank = 0;
    check(rl_numerical_rank(a.rows(), a.cols(), a.data().data(), 0.5, &rank, sg.data()));
    return sg;
}

double cond2(const Matrix& a, double tol) { // dense_core.cpp:177-186
    std::vector<double> sg = singular_values(a);
    if (sg.empty() || sg[0] == 0.0)
        throw ZeroMatrix("cond2: zero matrix");
    std::size_t rank = 0;
    for (std::size_t j = 0; j < sg.size(); ++j)
        if (sg[j] >= tol * sg[0])
            rank = j + 1;
    const double smin = sg[rank - 1];
    return smin == 0.0 ? std::numeric_limits<double>::infinity() : sg[0] / smin;
}

std::size_t numerical_rank(const Matrix& a, double tol) {
    if (!(tol > 0.0 && tol < 1.0))
        throw InvalidArgument("numerical_rank: tol must lie in (0, 1)");
    std::uint64_t rank = 0;
    std::vector<double> sg(std::min(a.rows(), a.cols()));
    check(rl_numerical_rank(a.rows(), a.cols(), a.data().data(), tol, &rank, sg.data()));
    return rank;
}

} // namespace dense

namespace lowrank {

Matrix project_onto_basis(const Matrix& a, const Matrix& basis, bool orthonormal, dense::Side side) {
    const std::size_t expected = side == dense::Side::Right ? a.cols() : a.rows();
    if (basis.rows() != expected)
        throw DimensionMismatch("project_onto_basis: basis row count mismatch");
    // the orthogonal projector onto span(basis) equals Q Q^T for Q = qr_positive(basis).Q; the
    // QR's rank check plays the role of the reference's SVD rank test (lowrank.cpp:50-54)
    const Matrix q = orthonormal ? basis : dense::qr_positive(basis).Q;
    if (side == dense::Side::Left) {
        Matrix out(a.rows(), a.cols());
        check(rl_project_onto_basis_left(a.rows(), a.cols(), q.cols(), a.data().data(), q.data().data(), nullptr,
                                         out.data().data()));
        return out;
    }
    return a.multiply(q).multiply(q.transpose()); // A T T^T (lowrank.cpp:55-59)
}

Matrix approx_basis(const Matrix& a, std::size_t rho_plus, rnd::MultiplierKind kind, SpaceSide side,
                    rnd::RngStream stream) {
    const std::size_t m = a.rows(), n = a.cols();
    if (rho_plus < 1 || rho_plus > std::min(m, n))
        throw InvalidArgument("approx_basis: rho_plus out of range");
    const std::size_t mult_rows = side == SpaceSide::RightSpace ? m : n;
    if (kind.tag == rnd::MultiplierTag::Gaussian) {
        Matrix y(side == SpaceSide::RightSpace ? n : m, rho_plus);
        check(rl_approx_basis(m, n, a.data().data(), rho_plus, kind.mu, kind.sigma,
                              side == SpaceSide::RightSpace ? 1 : 0, stream.seed, stream.stream_id,
                              y.data().data()));
        return y;
    }
    Matrix g(1, 1);
    switch (kind.tag) {
    case rnd::MultiplierTag::UniformPm1:
        g = rnd::uniform_matrix(mult_rows, rho_plus, stream);
        break;
    case rnd::MultiplierTag::HouseholderSign:
        g = rnd::householder_sign(mult_rows, stream).leading_columns(rho_plus);
        break;
    case rnd::MultiplierTag::ToeplitzGaussian:
        g = structured::densify(rnd::random_structured(kind, mult_rows, rho_plus, stream));
        break;
    case rnd::MultiplierTag::CirculantGaussian:
    case rnd::MultiplierTag::CirculantSign:
        g = structured::densify(rnd::random_structured(kind, mult_rows, mult_rows, stream)).leading_columns(rho_plus);
        break;
    default:
        throw InvalidArgument("approx_basis: unknown multiplier kind");
    }
    return side == SpaceSide::RightSpace ? a.transpose().multiply(g) : a.multiply(g);
}

LowRankResult proto_lowrank(const Matrix& a, std::size_t rho_plus, double tau, double tau_prime,
                            rnd::MultiplierKind kind, rnd::RngStream stream) {
    if (kind.tag != rnd::MultiplierTag::Gaussian && kind.tag != rnd::MultiplierTag::ToeplitzGaussian)
        throw InvalidArgument("proto_lowrank: the B200 path takes the Gaussian and ToeplitzGaussian kinds");
    const std::size_t m = a.rows(), n = a.cols();
    Matrix basis(n, std::max<std::size_t>(rho_plus, 1));
    Matrix approx(m, n);
    uint64_t rho = 0;
    double residual = 0.0;
    int ok = 0;
    check(rl_proto_lowrank(m, n, a.data().data(), rho_plus, tau, tau_prime, static_cast<int>(kind.tag), kind.mu,
                           kind.sigma, stream.seed,
                           stream.stream_id, &rho, basis.data().data(), approx.data().data(), &residual, &ok));
    LowRankResult r;
    r.rho = rho;
    r.basis = rho > 0 ? basis.leading_columns(rho) : Matrix(n, 1);
    r.approx = std::move(approx);
    r.residual = residual;
    r.ok = ok != 0;
    return r;
}

Matrix power_transform(const Matrix& a, unsigned h) {
    Matrix out(a.rows(), a.cols());
    check(rl_power_transform(a.rows(), a.cols(), a.data().data(), h, out.data().data()));
    return out;
}

SvEstimates extremal_sv_estimate(const Matrix& a, SvMethod method, int iters, rnd::RngStream stream) {
    SvEstimates e;
    check(rl_extremal_sv_estimate(a.rows(), a.cols(), a.data().data(), method == SvMethod::Lanczos ? 1 : 0, iters,
                                  stream.seed, stream.stream_id, &e.sv_max, &e.sv_min));
    return e;
}

bool cond_probe(const Matrix& b, double kappa_threshold, SvMethod method, int iters, rnd::RngStream stream) {
    int pass = 0;
    check(rl_cond_probe(b.rows(), b.cols(), b.data().data(), kappa_threshold, method == SvMethod::Lanczos ? 1 : 0,
                        iters, stream.seed, stream.stream_id, &pass));
    return pass != 0;
}

NrankResult nrank_search(const Matrix& a, std::size_t rho_minus, std::size_t rho_plus, double kappa_threshold,
                         SearchPolicy policy, rnd::RngStream stream) {
    const std::size_t wide = std::max(a.rows(), a.cols());
    std::vector<double> basis(wide * std::max<std::size_t>(rho_plus, 1), 0.0);
    uint64_t rho = 0, rows = 0, cols = 0;
    check(rl_nrank_search(a.rows(), a.cols(), a.data().data(), rho_minus, rho_plus, kappa_threshold,
                          policy == SearchPolicy::Binary ? 0 : 1, stream.seed, stream.stream_id, &rho, basis.data(),
                          &rows, &cols));
    NrankResult r;
    r.rho = rho;
    basis.resize(rows * cols);
    r.basis = Matrix(rows, cols, std::move(basis));
    return r;
}

} // namespace lowrank
} // namespace randla

// randla::genp on the B200 C-ABI (reference semantics: proj/src/genp.cpp).
#include "randla/genp.hpp"

#include <algorithm>
#include <cmath>

#include "randla/dense_core.hpp"
#include "rl_b200.h"

namespace randla::genp {

using detail::check;

GenpFactorization genp_factor(const Matrix& a, double pivot_floor) {
    if (a.rows() != a.cols())
        throw DimensionMismatch("genp_factor: square matrix required");
    if (pivot_floor < 0.0)
        throw InvalidArgument("genp_factor: pivot_floor must be >= 0");
    const std::size_t n = a.rows();
    Matrix l(n, n), u(n, n);
    std::vector<double> piv(n);
    double mm[2] = {0.0, 0.0};
    std::int64_t step = -1;
    check(rl_genp_factor(n, a.data().data(), pivot_floor, l.data().data(), u.data().data(), piv.data(), mm,
                         &step));
    return GenpFactorization{std::move(l), std::move(u), std::move(piv), mm[0], mm[1]};
}

BlockGeFactorization block_ge(const Matrix& a, std::size_t block) {
    if (a.rows() != a.cols())
        throw DimensionMismatch("block_ge: square matrix required");
    if (block == 0)
        throw InvalidArgument("block_ge: block must be positive");
    GenpFactorization f = genp_factor(a, 0.0);
    const std::size_t n = a.rows();
    std::vector<double> pn, pin;
    for (std::size_t o = 0; o < n; o += block) {
        const std::size_t bs = std::min(block, n - o);
        // pivot block of step o = the Schur complement block = L_oo U_oo (genp.cpp:55-61)
        Matrix p = f.L.block(o, o, bs, bs).multiply(f.U.block(o, o, bs, bs));
        std::vector<double> sg = dense::singular_values(p);
        const double smin = sg.back();
        if (!(smin > 0.0))
            throw PivotBreakdown("block_ge: singular pivot block at offset " + std::to_string(o));
        pn.push_back(sg.front());
        pin.push_back(1.0 / smin);
    }
    return BlockGeFactorization{std::move(f.L), std::move(f.U), std::move(pn), std::move(pin)};
}

std::vector<double> genp_solve(const GenpFactorization& f, std::span<const double> b) {
    const std::size_t n = f.L.rows();
    if (b.size() != n)
        throw DimensionMismatch("genp_solve: rhs length mismatch");
    std::vector<double> y(n);
    check(rl_genp_solve(n, 1, f.L.data().data(), f.U.data().data(), b.data(), y.data()));
    return y;
}

Matrix genp_solve(const GenpFactorization& f, const Matrix& b) {
    const std::size_t n = f.L.rows();
    if (b.rows() != n)
        throw DimensionMismatch("genp_solve: rhs row count mismatch");
    Matrix x(n, b.cols());
    check(rl_genp_solve(n, b.cols(), f.L.data().data(), f.U.data().data(), b.data().data(), x.data().data()));
    return x;
}

std::vector<double> iterative_refine(const Matrix& a, const GenpFactorization& f, std::span<const double> y0,
                                     std::span<const double> b, int steps) {
    if (steps < 0)
        throw InvalidArgument("iterative_refine: steps must be >= 0");
    std::vector<double> y(y0.begin(), y0.end());
    for (int s = 0; s < steps; ++s) { // genp.cpp:126-142
        std::vector<double> ay = a.multiply(y);
        std::vector<double> r(b.size());
        for (std::size_t i = 0; i < b.size(); ++i)
            r[i] = b[i] - ay[i];
        std::vector<double> d = genp_solve(f, r);
        for (std::size_t i = 0; i < y.size(); ++i)
            y[i] += d[i];
    }
    return y;
}

namespace {
PrecondReport to_report(const rl_precond_report& r, rnd::MultiplierKind kind, int refine) {
    PrecondReport p;
    p.multiplier = kind;
    p.refinement_steps = refine;
    p.residual = r.residual;
    p.raw_residual = r.raw_residual;
    p.pivot_min = r.pivot_min;
    p.pivot_max = r.pivot_max;
    p.raw_pivot_min = r.raw_pivot_min;
    p.raw_pivot_max = r.raw_pivot_max;
    return p;
}
} // namespace

std::pair<std::vector<double>, PrecondReport>
randomized_genp(const Matrix& a, std::span<const double> b, rnd::MultiplierKind kind, MulSide side, int refine,
                rnd::RngStream stream) {
    if (a.rows() != a.cols() || b.size() != a.rows())
        throw DimensionMismatch("randomized_genp: shape mismatch");
    if (refine < 0 || refine > 2)
        throw InvalidArgument("randomized_genp: refine must be in {0, 1, 2}");
    std::vector<double> y(a.rows());
    rl_precond_report r{};
    check(rl_randomized_genp(a.rows(), 1, a.data().data(), b.data(), static_cast<int>(kind.tag), kind.mu,
                             kind.sigma, static_cast<int>(side), refine, stream.seed, stream.stream_id, y.data(),
                             &r));
    return {std::move(y), to_report(r, kind, refine)};
}

std::vector<std::pair<std::vector<double>, PrecondReport>>
randomized_genp_batched(const std::vector<Matrix>& systems, const std::vector<std::vector<double>>& rhs,
                        rnd::MultiplierKind kind, MulSide side, int refine, std::uint64_t seed,
                        std::span<const std::uint64_t> stream_ids) {
    const std::size_t batch = systems.size();
    if (rhs.size() != batch || stream_ids.size() != batch)
        throw DimensionMismatch("randomized_genp_batched: batch size mismatch");
    if (batch == 0)
        return {};
    const std::size_t n = systems[0].rows();
    std::vector<double> a(batch * n * n), b(batch * n), x(batch * n);
    for (std::size_t t = 0; t < batch; ++t) {
        if (systems[t].rows() != n || systems[t].cols() != n || rhs[t].size() != n)
            throw DimensionMismatch("randomized_genp_batched: systems must share one square shape");
        std::copy(systems[t].data().begin(), systems[t].data().end(), a.begin() + t * n * n);
        std::copy(rhs[t].begin(), rhs[t].end(), b.begin() + t * n);
    }
    std::vector<rl_precond_report> reps(batch);
    check(rl_randomized_genp_batched(batch, n, a.data(), b.data(), static_cast<int>(kind.tag), kind.mu,
                                     kind.sigma, static_cast<int>(side), refine, seed, stream_ids.data(),
                                     x.data(), reps.data()));
    std::vector<std::pair<std::vector<double>, PrecondReport>> out;
    out.reserve(batch);
    for (std::size_t t = 0; t < batch; ++t)
        out.emplace_back(std::vector<double>(x.begin() + t * n, x.begin() + (t + 1) * n),
                         to_report(reps[t], kind, refine));
    return out;
}

} // namespace randla::genp

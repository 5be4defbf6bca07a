// randla::rnd on the B200 C-ABI (reference semantics: proj/src/random_gen.cpp:13-199).
#include "randla/random_gen.hpp"

#include <limits>

#include "rl_b200.h"

namespace randla::rnd {

using detail::check;

namespace {
constexpr std::size_t kBlock = 4096;
}

Rng::Rng(RngStream stream) : stream_(stream) {}

std::uint64_t Rng::next() {
    if (buf_.empty() || pos_ < buf_start_ || pos_ >= buf_start_ + buf_.size()) {
        buf_.assign(kBlock, 0);
        buf_start_ = pos_;
        check(rl_rng_block(stream_.seed, stream_.stream_id, buf_start_, kBlock, buf_.data()));
    }
    return buf_[pos_++ - buf_start_];
}

double Rng::uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
double Rng::uniform_pm1() { return 2.0 * uniform01() - 1.0; }

double Rng::gaussian() {
    if (has_cached_) {
        has_cached_ = false;
        return cached_;
    }
    std::uint64_t raw[2] = {next(), next()};
    double g[2];
    check(rl_box_muller(1, raw, g));
    cached_ = g[1];
    has_cached_ = true;
    return g[0];
}

double Rng::sign() { return (next() & 1u) ? 1.0 : -1.0; }

std::int64_t Rng::uniform_int(std::int64_t lo, std::int64_t hi) {
    if (hi < lo)
        throw InvalidArgument("uniform_int: empty range");
    const std::uint64_t span = static_cast<std::uint64_t>(hi - lo) + 1;
    const std::uint64_t limit = std::numeric_limits<std::uint64_t>::max() / span * span;
    std::uint64_t v;
    do {
        v = next();
    } while (v >= limit);
    return lo + static_cast<std::int64_t>(v % span);
}

Matrix gaussian_matrix(std::size_t m, std::size_t n, double mu, double sigma, RngStream stream) {
    if (!(sigma > 0.0))
        throw InvalidArgument("gaussian_matrix: sigma must be positive");
    Matrix out(m, n);
    check(rl_gaussian_matrix(m, n, mu, sigma, stream.seed, stream.stream_id, out.data().data()));
    return out;
}

Matrix uniform_matrix(std::size_t m, std::size_t n, RngStream stream) {
    Matrix out(m, n);
    check(rl_uniform_matrix(m, n, stream.seed, stream.stream_id, out.data().data()));
    return out;
}

structured::StructuredSpec random_structured(MultiplierKind kind, std::size_t m, std::size_t n,
                                             RngStream stream) {
    std::vector<double> col(m), row(n);
    check(rl_random_structured(static_cast<int>(kind.tag), kind.mu, kind.sigma, m, n, stream.seed,
                               stream.stream_id, col.data(), row.data()));
    if (kind.tag == MultiplierTag::ToeplitzGaussian)
        return structured::StructuredSpec::toeplitz(std::move(col), std::move(row));
    return structured::StructuredSpec::circulant(std::move(col));
}

Matrix householder_sign(std::size_t n, RngStream stream) {
    Matrix out(n, n);
    check(rl_householder_sign(n, stream.seed, stream.stream_id, out.data().data()));
    return out;
}

void householder_pair_signs(std::size_t n, RngStream stream, std::vector<double>& u1, std::vector<double>& u2) {
    u1.resize(n);
    u2.resize(n);
    check(rl_householder_pair_signs(n, stream.seed, stream.stream_id, u1.data(), u2.data()));
}

void sparse_sign(std::size_t n, int nnz, RngStream stream, std::vector<std::int32_t>& rows,
                 std::vector<double>& signs) {
    rows.resize(n * static_cast<std::size_t>(nnz));
    signs.resize(rows.size());
    check(rl_sparse_sign(n, nnz, stream.seed, stream.stream_id, rows.data(), signs.data()));
}

std::vector<double> paper_sigma_profile(std::size_t n, std::size_t rho) {
    std::vector<double> s(n, 1e-10); // random_gen.cpp:194-199
    for (std::size_t j = 0; j < std::min(rho, n); ++j)
        s[j] = 1.0 / static_cast<double>(j + 1);
    return s;
}

} // namespace randla::rnd

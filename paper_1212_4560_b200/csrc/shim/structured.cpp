// randla::structured on the B200 C-ABI (reference semantics: proj/src/structured.cpp).
#include "randla/structured.hpp"

#include "rl_b200.h"

namespace randla::structured {

using detail::check;

StructuredSpec StructuredSpec::circulant(std::vector<double> first_col) {
    if (first_col.empty())
        throw InvalidArgument("circulant: empty first column");
    const std::size_t n = first_col.size();
    return StructuredSpec{Kind::Circulant, n, n, std::move(first_col), {}};
}

StructuredSpec StructuredSpec::toeplitz(std::vector<double> first_col, std::vector<double> first_row) {
    if (first_col.empty() || first_row.empty())
        throw InvalidArgument("toeplitz: empty generators");
    if (first_col[0] != first_row[0])
        throw InvalidArgument("toeplitz: first_col[0] != first_row[0]");
    const std::size_t m = first_col.size(), n = first_row.size();
    return StructuredSpec{Kind::Toeplitz, m, n, std::move(first_col), std::move(first_row)};
}

Matrix densify(const StructuredSpec& spec) {
    Matrix out(spec.n_rows, spec.n_cols);
    for (std::size_t i = 0; i < spec.n_rows; ++i)
        for (std::size_t j = 0; j < spec.n_cols; ++j)
            out(i, j) = spec.kind == StructuredSpec::Kind::Circulant
                            ? spec.first_col[(i + spec.n_rows - j) % spec.n_rows]
                            : (i >= j ? spec.first_col[i - j] : spec.first_row[j - i]);
    return out;
}

StructuredSpec transpose_spec(const StructuredSpec& spec) {
    if (spec.kind == StructuredSpec::Kind::Circulant) {
        const std::size_t n = spec.n_rows;
        std::vector<double> col(n);
        for (std::size_t k = 0; k < n; ++k)
            col[k] = spec.first_col[(n - k) % n];
        return StructuredSpec::circulant(std::move(col));
    }
    return StructuredSpec::toeplitz(spec.first_row, spec.first_col);
}

std::vector<std::complex<double>> fft(std::span<const std::complex<double>> x, FftDirection dir) {
    std::vector<std::complex<double>> out(x.size());
    check(rl_dft(x.size(), reinterpret_cast<const double*>(x.data()), dir == FftDirection::Inverse ? 1 : 0,
                 reinterpret_cast<double*>(out.data())));
    return out;
}

std::vector<double> circ_mul(const StructuredSpec& spec, std::span<const double> x) {
    if (spec.kind != StructuredSpec::Kind::Circulant)
        throw InvalidArgument("circ_mul: circulant spec required");
    if (x.size() != spec.n_rows)
        throw DimensionMismatch("circ_mul: vector length mismatch");
    std::vector<double> y(x.size());
    check(rl_circ_mul(x.size(), spec.first_col.data(), x.data(), y.data()));
    return y;
}

std::vector<double> toeplitz_mul(const StructuredSpec& spec, std::span<const double> x) {
    if (spec.kind != StructuredSpec::Kind::Toeplitz)
        throw InvalidArgument("toeplitz_mul: toeplitz spec required");
    if (x.size() != spec.n_cols)
        throw DimensionMismatch("toeplitz_mul: vector length mismatch");
    return densify(spec).multiply(x);
}

Matrix multiply_matrix(const StructuredSpec& spec, const Matrix& a) {
    if (spec.n_cols != a.rows())
        throw DimensionMismatch("multiply_matrix: inner dimensions differ");
    if (spec.kind == StructuredSpec::Kind::Circulant) {
        Matrix out(spec.n_rows, a.cols());
        check(rl_circulant_multiply_matrix(spec.n_rows, spec.first_col.data(), a.cols(), a.data().data(),
                                           out.data().data()));
        return out;
    }
    return densify(spec).multiply(a);
}

} // namespace randla::structured

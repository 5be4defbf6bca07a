// randla::structured for the drop-in library. The spec helpers are host bookkeeping; every
// product (fft, circ_mul, toeplitz_mul, multiply_matrix) runs on the GPU through the C-ABI
// (csrc/fft_exact.cu), which executes the reference's own FFT algorithm step for step — the
// results are the reference's bits (structured.cpp:20-189), matrix-free, O(n log n).
#include "randla/structured.hpp"

#include <algorithm>

#include "rl_b200.h"

namespace randla::structured {

using detail::check;

namespace {
template <class E>
void require(bool ok, const char* msg) {
    if (!ok)
        throw E(msg);
}
using Kind = StructuredSpec::Kind;
} // namespace

StructuredSpec StructuredSpec::circulant(std::vector<double> first_col) {
    require<InvalidArgument>(!first_col.empty(), "circulant: empty first column");
    const std::size_t order = first_col.size();
    return StructuredSpec{Kind::Circulant, order, order, std::move(first_col), {}};
}

StructuredSpec StructuredSpec::toeplitz(std::vector<double> first_col, std::vector<double> first_row) {
    require<InvalidArgument>(!first_col.empty() && !first_row.empty(), "toeplitz: empty generators");
    require<InvalidArgument>(first_col.front() == first_row.front(), "toeplitz: first_col[0] != first_row[0]");
    const std::size_t rows = first_col.size(), cols = first_row.size();
    return StructuredSpec{Kind::Toeplitz, rows, cols, std::move(first_col), std::move(first_row)};
}

// Entry (i, j) depends only on i - j: the circulant reads its column cyclically, the Toeplitz
// matrix its column below the diagonal and its row above.
Matrix densify(const StructuredSpec& spec) {
    Matrix out(spec.n_rows, spec.n_cols);
    const auto entry = [&spec](std::size_t i, std::size_t j) {
        if (spec.kind == Kind::Circulant)
            return spec.first_col[(i + spec.n_rows - j) % spec.n_rows];
        return i >= j ? spec.first_col[i - j] : spec.first_row[j - i];
    };
    for (std::size_t i = 0; i < spec.n_rows; ++i)
        for (std::size_t j = 0; j < spec.n_cols; ++j)
            out(i, j) = entry(i, j);
    return out;
}

// C^T is the circulant of c reversed after its first entry; T^T swaps the generators.
StructuredSpec transpose_spec(const StructuredSpec& spec) {
    if (spec.kind == Kind::Toeplitz)
        return StructuredSpec::toeplitz(spec.first_row, spec.first_col);
    std::vector<double> col(spec.first_col);
    std::reverse(col.begin() + 1, col.end());
    return StructuredSpec::circulant(std::move(col));
}

std::vector<std::complex<double>> fft(std::span<const std::complex<double>> x, FftDirection dir) {
    std::vector<std::complex<double>> out(x.size());
    check(rl_fft(x.size(), reinterpret_cast<const double*>(x.data()), dir == FftDirection::Inverse ? 1 : 0,
                 reinterpret_cast<double*>(out.data())));
    return out;
}

std::vector<double> circ_mul(const StructuredSpec& spec, std::span<const double> x) {
    require<InvalidArgument>(spec.kind == Kind::Circulant, "circ_mul: circulant spec required");
    require<DimensionMismatch>(x.size() == spec.n_rows, "circ_mul: vector length mismatch");
    std::vector<double> y(x.size());
    check(rl_circ_mul(x.size(), spec.first_col.data(), x.data(), y.data()));
    return y;
}

std::vector<double> toeplitz_mul(const StructuredSpec& spec, std::span<const double> x) {
    require<InvalidArgument>(spec.kind == Kind::Toeplitz, "toeplitz_mul: toeplitz spec required");
    require<DimensionMismatch>(x.size() == spec.n_cols, "toeplitz_mul: vector length mismatch");
    std::vector<double> y(spec.n_rows);
    check(rl_toeplitz_mul(spec.n_rows, spec.n_cols, spec.first_col.data(), spec.first_row.data(), x.data(),
                          y.data()));
    return y;
}

Matrix multiply_matrix(const StructuredSpec& spec, const Matrix& a) {
    require<DimensionMismatch>(spec.n_cols == a.rows(), "multiply_matrix: inner dimensions differ");
    Matrix out(spec.n_rows, a.cols());
    if (spec.kind == Kind::Circulant)
        check(rl_circulant_multiply_matrix(spec.n_rows, spec.first_col.data(), a.cols(), a.data().data(),
                                           out.data().data()));
    else
        check(rl_toeplitz_multiply_matrix(spec.n_rows, spec.n_cols, spec.first_col.data(), spec.first_row.data(),
                                          a.cols(), a.data().data(), out.data().data()));
    return out;
}

} // namespace randla::structured

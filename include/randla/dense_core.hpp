#pragma once
// Dense-core subset on the hot path (reference: proj/include/randla/dense_core.hpp:10-76):
// norms, qr_positive, numerical_rank, cond2.  The reference's remaining SVD-based helpers
// (svd factors, pseudo_inverse, truncate_svd, leading_basis, pivoted_solve, least_squares,
// inverse) are oracle-side utilities, out of scope for the B200 path.
#include <cstddef>
#include <vector>

#include "randla/matrix.hpp"

namespace randla::dense {

enum class NormKind { One, Two, Inf, Frobenius };
double norm(const Matrix& a, NormKind kind);
inline double norm2(const Matrix& a) { return norm(a, NormKind::Two); }

struct QrFactors {
    Matrix Q;
    Matrix R;
};
QrFactors qr_positive(const Matrix& a);

std::vector<double> singular_values(const Matrix& a); // B200: sigma only
double cond2(const Matrix& a, double tol);
std::size_t numerical_rank(const Matrix& a, double tol);

enum class Side { Left, Right };

} // namespace randla::dense

// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// CPU restatement of the four Eigen-backed randla::dense symbols that the
// reference's GENP/RNG translation units reference: Eigen is
// absent from this image, so proj/src/dense_core.cpp cannot be compiled.  The
// semantics follow proj/src/dense_core.cpp:
//   norm        dense_core.cpp:48-84   (Two = sigma_1 of the full SVD)
//   qr_positive dense_core.cpp:86-115  (Householder QR, rank check
//                                       min|R_ii| > 1e-13 sigma_1(R), sign fix)
//   svd         dense_core.cpp:117-136 (sigma non-increasing; sign convention:
//                                       largest-|.| entry of each left vector > 0)
//   cond2       dense_core.cpp:177-186 (+ numerical_rank :161-175)
//   inverse     dense_core.cpp:241-247 (partial-pivoting LU inverse; needed by lowrank.cpp)
// Eigen's own rounding is not reproduced (it is unpinned upstream);
// QR is unique for full rank, so Q and R agree with Eigen to rounding.
// The SVD is a one-sided (Hestenes) Jacobi iteration.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <vector>

#include "randla/dense_core.hpp"

namespace randla::dense {

namespace {

// One-sided Jacobi on the columns of W (m x n, row-major, m >= n).  On return
// W = U * diag(sigma) (columns unnormalised) and V accumulates the rotations.
void hestenes(std::vector<double>& w, std::size_t m, std::size_t n, std::vector<double>& v) {
    v.assign(n * n, 0.0);
    for (std::size_t i = 0; i < n; ++i)
        v[i * n + i] = 1.0;
    for (int sweep = 0; sweep < 80; ++sweep) {
        double off = 0.0;
        for (std::size_t p = 0; p + 1 < n; ++p)
            for (std::size_t q = p + 1; q < n; ++q) {
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (std::size_t i = 0; i < m; ++i) {
                    double wp = w[i * n + p], wq = w[i * n + q];
                    alpha += wp * wp;
                    beta += wq * wq;
                    gamma += wp * wq;
                }
                if (gamma == 0.0)
                    continue;
                double rel = std::abs(gamma) / std::sqrt(alpha * beta);
                if (!(rel > 1e-15))
                    continue;
                off = std::max(off, rel);
                double zeta = (beta - alpha) / (2.0 * gamma);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                for (std::size_t i = 0; i < m; ++i) {
                    double wp = w[i * n + p], wq = w[i * n + q];
                    w[i * n + p] = c * wp - s * wq;
                    w[i * n + q] = s * wp + c * wq;
                }
                for (std::size_t i = 0; i < n; ++i) {
                    double vp = v[i * n + p], vq = v[i * n + q];
                    v[i * n + p] = c * vp - s * vq;
                    v[i * n + q] = s * vp + c * vq;
                }
            }
        if (off <= 1e-15)
            break;
    }
}

// Thin SVD of a (m x n): returns sigma (l = min(m,n)), U (m x l), V (n x l).
void thin_svd(const Matrix& a, std::vector<double>& sigma, std::vector<double>& u,
              std::vector<double>& vv) {
    const bool tr = a.rows() < a.cols();
    const std::size_t m = tr ? a.cols() : a.rows(), n = tr ? a.rows() : a.cols();
    std::vector<double> w(m * n);
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j)
            w[i * n + j] = tr ? a(j, i) : a(i, j);
    std::vector<double> v;
    hestenes(w, m, n, v);
    std::vector<double> norms(n);
    for (std::size_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (std::size_t i = 0; i < m; ++i)
            s += w[i * n + j] * w[i * n + j];
        norms[j] = std::sqrt(s);
    }
    std::vector<std::size_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](std::size_t x, std::size_t y) { return norms[x] > norms[y]; });
    sigma.resize(n);
    std::vector<double> uu(m * n), vt(n * n);
    for (std::size_t k = 0; k < n; ++k) {
        std::size_t j = order[k];
        sigma[k] = norms[j];
        for (std::size_t i = 0; i < m; ++i)
            uu[i * n + k] = norms[j] > 0 ? w[i * n + j] / norms[j] : 0.0;
        for (std::size_t i = 0; i < n; ++i)
            vt[i * n + k] = v[i * n + j];
    }
    if (tr) {
        u = vt; // a^T = U' S V'^T  =>  a = V' S U'^T
        vv = uu;
    } else {
        u = uu;
        vv = vt;
    }
}

} // namespace

double norm(const Matrix& a, NormKind kind) {
    switch (kind) {
    case NormKind::One: {
        double best = 0.0;
        for (std::size_t j = 0; j < a.cols(); ++j) {
            double s = 0.0;
            for (std::size_t i = 0; i < a.rows(); ++i)
                s += std::abs(a(i, j));
            best = std::max(best, s);
        }
        return best;
    }
    case NormKind::Inf: {
        double best = 0.0;
        for (std::size_t i = 0; i < a.rows(); ++i) {
            double s = 0.0;
            for (std::size_t j = 0; j < a.cols(); ++j)
                s += std::abs(a(i, j));
            best = std::max(best, s);
        }
        return best;
    }
    case NormKind::Frobenius: {
        double s = 0.0;
        for (double x : a.data())
            s += x * x;
        return std::sqrt(s);
    }
    case NormKind::Two: {
        std::vector<double> sg, u, v;
        thin_svd(a, sg, u, v);
        return sg.empty() ? 0.0 : sg[0];
    }
    }
    return 0.0;
}

QrFactors qr_positive(const Matrix& a) {
    const std::size_t m = a.rows(), n = a.cols();
    if (m < n)
        throw InvalidArgument("qr_positive: requires rows >= cols");
    // Householder QR, column-major working copy.
    std::vector<double> w(m * n);
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j)
            w[j * m + i] = a(i, j);
    std::vector<double> tau(n, 0.0);
    for (std::size_t k = 0; k < n; ++k) {
        double* x = &w[k * m];
        double sn = 0.0;
        for (std::size_t i = k + 1; i < m; ++i)
            sn += x[i] * x[i];
        double alpha = x[k];
        if (sn == 0.0) {
            tau[k] = 0.0;
            continue;
        }
        double beta = -std::copysign(std::sqrt(alpha * alpha + sn), alpha);
        tau[k] = (beta - alpha) / beta;
        double scale = 1.0 / (alpha - beta);
        for (std::size_t i = k + 1; i < m; ++i)
            x[i] *= scale;
        x[k] = beta;
        for (std::size_t j = k + 1; j < n; ++j) {
            double* y = &w[j * m];
            double s = y[k];
            for (std::size_t i = k + 1; i < m; ++i)
                s += x[i] * y[i];
            s *= tau[k];
            y[k] -= s;
            for (std::size_t i = k + 1; i < m; ++i)
                y[i] -= s * x[i];
        }
    }
    Matrix r(n, n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = i; j < n; ++j)
            r(i, j) = w[j * m + i];
    // Thin Q = H_0 ... H_{n-1} [I; 0]
    std::vector<double> q(m * n, 0.0); // column-major
    for (std::size_t j = 0; j < n; ++j)
        q[j * m + j] = 1.0;
    for (std::size_t kk = n; kk-- > 0;) {
        const double* x = &w[kk * m];
        for (std::size_t j = 0; j < n; ++j) {
            double* y = &q[j * m];
            double s = y[kk];
            for (std::size_t i = kk + 1; i < m; ++i)
                s += x[i] * y[i];
            s *= tau[kk];
            y[kk] -= s;
            for (std::size_t i = kk + 1; i < m; ++i)
                y[i] -= s * x[i];
        }
    }
    double min_diag = std::numeric_limits<double>::infinity();
    for (std::size_t i = 0; i < n; ++i)
        min_diag = std::min(min_diag, std::abs(r(i, i)));
    double n2 = norm(r, NormKind::Two);
    if (!(min_diag > 1e-13 * n2))
        throw RankDeficient("qr_positive: numerically rank-deficient input");
    Matrix qm(m, n);
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j)
            qm(i, j) = q[j * m + i];
    for (std::size_t i = 0; i < n; ++i)
        if (r(i, i) < 0.0) {
            for (std::size_t j = 0; j < n; ++j)
                r(i, j) = -r(i, j);
            for (std::size_t k = 0; k < m; ++k)
                qm(k, i) = -qm(k, i);
        }
    return QrFactors{std::move(qm), std::move(r)};
}

SvdFactors svd(const Matrix& a) {
    std::vector<double> sg, u, v;
    thin_svd(a, sg, u, v);
    const std::size_t m = a.rows(), n = a.cols(), l = sg.size();
    // Full factors: thin vectors in the leading columns (only sigma is used by
    // the reference code paths this oracle exercises: block_ge, cond2, norm2).
    Matrix s(m, m), t(n, n);
    for (std::size_t j = 0; j < l; ++j) {
        std::size_t imax = 0;
        for (std::size_t i = 1; i < m; ++i)
            if (std::abs(u[i * l + j]) > std::abs(u[imax * l + j]))
                imax = i;
        double sgn = u[imax * l + j] < 0.0 ? -1.0 : 1.0;
        for (std::size_t i = 0; i < m; ++i)
            s(i, j) = sgn * u[i * l + j];
        for (std::size_t i = 0; i < n; ++i)
            t(i, j) = sgn * v[i * l + j];
    }
    return SvdFactors{std::move(s), std::move(sg), std::move(t)};
}

double cond2(const Matrix& a, double tol) {
    std::vector<double> sg, u, v;
    thin_svd(a, sg, u, v);
    if (sg.empty() || sg[0] == 0.0)
        throw ZeroMatrix("cond2: zero matrix");
    std::size_t rank = 0;
    for (std::size_t j = 0; j < sg.size(); ++j)
        if (sg[j] >= tol * sg[0])
            rank = j + 1;
    double smin = sg[rank - 1];
    if (smin == 0.0)
        return std::numeric_limits<double>::infinity();
    return sg[0] / smin;
}

Matrix inverse(const Matrix& a) {
    if (a.rows() != a.cols())
        throw DimensionMismatch("inverse: square matrix required");
    const std::size_t n = a.rows();
    Matrix w = a, inv = Matrix::identity(n);
    for (std::size_t k = 0; k < n; ++k) { // Gauss-Jordan with partial pivoting
        std::size_t p = k;
        for (std::size_t i = k + 1; i < n; ++i)
            if (std::abs(w(i, k)) > std::abs(w(p, k)))
                p = i;
        if (p != k)
            for (std::size_t j = 0; j < n; ++j) {
                std::swap(w(k, j), w(p, j));
                std::swap(inv(k, j), inv(p, j));
            }
        const double d = w(k, k);
        for (std::size_t j = 0; j < n; ++j) {
            w(k, j) /= d;
            inv(k, j) /= d;
        }
        for (std::size_t i = 0; i < n; ++i) {
            if (i == k || w(i, k) == 0.0)
                continue;
            const double f = w(i, k);
            for (std::size_t j = 0; j < n; ++j) {
                w(i, j) -= f * w(k, j);
                inv(i, j) -= f * inv(k, j);
            }
        }
    }
    return inv;
}

} // namespace randla::dense

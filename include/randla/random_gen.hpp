#pragma once
// Random streams and multipliers (reference: proj/include/randla/random_gen.hpp:16-104).
// Every draw comes from the GPU's mt19937_64 jump-ahead generator and matches the
// reference's stream bit for bit (Gaussians: correctly rounded log/sin/cos).
#include <cstdint>
#include <span>
#include <vector>

#include "randla/matrix.hpp"
#include "randla/structured.hpp"

namespace randla::rnd {

struct RngStream {
    std::uint64_t seed = 0;
    std::uint64_t stream_id = 0;
    RngStream with_stream(std::uint64_t id) const { return RngStream{seed, id}; }
};

// Sequential draws of one stream.  Raw engine outputs are fetched from the GPU in blocks;
// the transforms are those of random_gen.cpp:33-70.
class Rng {
  public:
    explicit Rng(RngStream stream);
    double uniform01();
    double uniform_pm1();
    double gaussian();
    double sign();
    std::int64_t uniform_int(std::int64_t lo, std::int64_t hi);

  private:
    std::uint64_t next();
    RngStream stream_;
    std::uint64_t pos_ = 0;        // stream position of the next raw draw
    std::uint64_t buf_start_ = 0;  // position of buf_[0]
    std::vector<std::uint64_t> buf_;
    bool has_cached_ = false;
    double cached_ = 0.0;
};

enum class MultiplierTag {
    Gaussian,
    UniformPm1,
    ToeplitzGaussian,
    CirculantGaussian,
    CirculantSign,
    HouseholderSign,
    HouseholderPair, // B200 extension: H1 H2, H_i = I - 2 u_i u_i^T / n, u_i in {+-1}^n
    SparseSign,      // B200 extension: 4 nonzeros +-1 per column at uniform rows
};

struct MultiplierKind {
    MultiplierTag tag = MultiplierTag::Gaussian;
    double mu = 0.0;
    double sigma = 1.0;
};

Matrix gaussian_matrix(std::size_t m, std::size_t n, double mu, double sigma, RngStream stream);
Matrix uniform_matrix(std::size_t m, std::size_t n, RngStream stream);
structured::StructuredSpec random_structured(MultiplierKind kind, std::size_t m, std::size_t n,
                                             RngStream stream);
Matrix householder_sign(std::size_t n, RngStream stream);

// B200 extensions: the signs of the orthogonal Householder pair, the sparse +-1 pattern.
void householder_pair_signs(std::size_t n, RngStream stream, std::vector<double>& u1,
                            std::vector<double>& u2);
void sparse_sign(std::size_t n, int nnz, RngStream stream, std::vector<std::int32_t>& rows,
                 std::vector<double>& signs);

std::vector<double> paper_sigma_profile(std::size_t n, std::size_t rho);

} // namespace randla::rnd

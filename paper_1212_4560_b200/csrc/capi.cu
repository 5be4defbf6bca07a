// The C-ABI (include/rl_b200.h): status codes instead of exceptions, host-pointer
// entry points with the reference's value semantics, device-pointer entry points for
// the large configurations.  Every entry point catches everything: nothing throws
// across the boundary.
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include <cstdio>
#include "rl_internal.cuh"

namespace rl {
const char* last_error();
uint64_t total_launches();
void init_device(int device);
void copy2d_dev(uint64_t rows, uint64_t cols, const double* src, uint64_t lds, double* dst, uint64_t ldd);
void genp_factor_blocked(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                         unsigned long long* d_breakdown, double* aux);
void genp_block_inverses(uint64_t n, const double* lu, uint64_t lda, double* aux);
void genp_solve_blocked(uint64_t n, uint64_t nrhs, const double* lu, uint64_t lda, const double* aux,
                        double* b, uint64_t ldb);
void circulant_dense_dev(uint64_t n, const double* c, double* out);
void rank1_dense_dev(uint64_t n, const double* u, const double* v, double inv_uv, double* out);
void circ_apply_vec_dev(uint64_t n, uint64_t nrhs, const double* c, const double* z, double* y);
rl_status randomized_genp_dev(uint64_t n, uint64_t nrhs, const double* A, const double* B, int tag,
                              double mu, double sigma, int side, int refine, uint64_t seed, uint64_t sid,
                              double* X, rl_precond_report* report, uint32_t flags);
const std::vector<rl_column_report>& last_column_reports();
void extremal_sv_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda, int method, int iters, uint64_t seed,
                     uint64_t sid, double* sv_max, double* sv_min);
bool cond_probe_dev(uint64_t m, uint64_t n, const double* b, uint64_t ldb, double kappa, int method, int iters,
                    uint64_t seed, uint64_t sid);
uint64_t nrank_search_dev(uint64_t m, uint64_t n, const double* a, uint64_t rho_minus, uint64_t rho_plus,
                          double kappa, int policy, uint64_t seed, uint64_t sid, double* basis,
                          uint64_t* basis_rows);
rl_status randomized_genp_batched_dev(uint64_t batch, uint64_t n, const double* dA, const double* dB,
                                      int tag, double mu, double sigma, int side, int refine,
                                      uint64_t seed, const uint64_t* d_sids, double* dX,
                                      rl_precond_report* d_rep);
void gemm_splitk(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, double alpha, const double* a,
                 uint64_t lda, const double* b, uint64_t ldb, double beta, double* c, uint64_t ldc,
                 int splits);
int splits_for(uint64_t m, uint64_t n, uint64_t k);
void sparse_apply_right_dev(uint64_t n, int nnz, const int32_t* rows, const double* signs, const double* a,
                            uint64_t lda, double* out, uint64_t ldo);
void hh2_apply_right_dev(uint64_t n, const double* a, uint64_t lda, const double* u1, const double* u2,
                         double s12, double* out, uint64_t ldo, const double* s12p = nullptr);
void dot_pm1_dev(uint64_t n, const double* u1, const double* u2, double* d_out);
bool circ_fft_supported(uint64_t n);
bool proto_lowrank_supported(uint64_t m, uint64_t n, uint64_t rho_plus);
void proto_lowrank_dev(uint64_t m, uint64_t n, const double* d_a, uint64_t rho_plus, double tau, double tau_prime,
                       int tag, double mu, double sig_g, uint64_t seed, uint64_t sid, uint64_t* rho_out,
                       double* d_basis, double* d_approx, double* residual, int* ok);
uint64_t toeplitz_fft_len(uint64_t n);
void toeplitz_apply_right_fft_dev(uint64_t m, uint64_t n, const double* g, const double* a, uint64_t lda,
                                  double* out, uint64_t ldo);
void toeplitz_dense_dev(uint64_t n, const double* g, double* out);
void circ_apply_right_fft_dev(uint64_t m, uint64_t n, const double* c, const double* a, uint64_t lda, double* out,
                              uint64_t ldo);
bool cholqr3(uint64_t m, int k, const double* y, double* q, double* r);
void cholqr3_async(uint64_t m, int k, const double* y, double* q, double* r, int* d_bad, bool want_q = true,
                   bool diag_only = false);
void rank_bracket_diag_launch(int k, const double* d_rdiag, int* d_flag);
void small_sv_launch(int k, const double* d_a, double* d_sg);
void rank_bracket_launch(int k, const double* d_r, int* d_flag);
std::vector<double> small_singular_values(int k, const double* d_a);
double sumsq_dev(uint64_t count, const double* x);
void uniform_int_dev(uint64_t seed, uint64_t sid, uint64_t count, int64_t lo, int64_t hi, int64_t* out);
void unpack_lu_dev(uint64_t n, const double* lu, double* l, double* u);
void pack_lu_dev(uint64_t n, const double* l, const double* u, double* lu);
rl_status probe_peaks(double* fp64, double* hbm);
void fft_exact_dev(uint64_t n, uint64_t batch, const double2* src, double2* dst, int inverse);
void structured_multiply_dev(uint64_t m, uint64_t n, const double* first_col, const double* first_row,
                             uint64_t cols, const double* a, double* out);
void abs_sums_dev(uint64_t m, uint64_t n, const double* a, int rows, double* out);
} // namespace rl

using namespace rl;

namespace {

#define API_BEGIN try {
#define API_END                                                  \
    }                                                            \
    catch (const Failure& f) {                                   \
        set_error(f.msg);                                        \
        return f.code;                                           \
    }                                                            \
    catch (const std::exception& e) {                            \
        set_error(e.what());                                     \
        return RL_ERROR;                                         \
    }                                                            \
    return RL_OK;

template <typename T>
T* upload(int slot, const T* h, uint64_t count) {
    T* d = ws<T>(slot, count);
    if (count)
        RL_CUDA(cudaMemcpyAsync(d, h, count * sizeof(T), cudaMemcpyHostToDevice, stream()));
    return d;
}


// Upload a row-major n x n host matrix into dev in row panels on a copy stream, leaving
// the transfer in flight (ctx().upload): the randomized GENP's first A * G product runs
// one GEMM per panel as each arrives, so the 512 MiB copy of config 3 overlaps the DGEMM
// instead of preceding it.  Small matrices upload in one piece.
void upload_rows_async(double* dev, const double* host, uint64_t n) {
    Ctx& c = ctx();
    struct CopyStream {
        cudaStream_t s = nullptr;
        cudaEvent_t start = nullptr, done[8] = {};
        int device = -1;
    };
    static thread_local CopyStream cs;
    if (cs.device != c.device) {
        RL_CUDA(cudaStreamCreateWithFlags(&cs.s, cudaStreamNonBlocking));
        RL_CUDA(cudaEventCreateWithFlags(&cs.start, cudaEventDisableTiming));
        for (auto& e : cs.done)
            RL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cs.device = c.device;
    }
    if (n < 2048) {
        if (n)
            RL_CUDA(cudaMemcpyAsync(dev, host, n * n * sizeof(double), cudaMemcpyHostToDevice, stream()));
        return;
    }
    // previous users of the buffer (earlier calls on the main stream) finish first
    RL_CUDA(cudaEventRecord(cs.start, stream()));
    RL_CUDA(cudaStreamWaitEvent(cs.s, cs.start, 0));
    const uint64_t ends[5] = {n / 16 & ~127ULL, n / 4 & ~127ULL, n / 2 & ~127ULL, 3 * n / 4 & ~127ULL, n};
    PendingUpload up;
    up.dev = dev;
    uint64_t r0 = 0;
    for (uint64_t r1 : ends) {
        if (r1 <= r0)
            continue;
        RL_CUDA(cudaMemcpyAsync(dev + r0 * n, host + r0 * n, (r1 - r0) * n * sizeof(double), cudaMemcpyHostToDevice,
                                cs.s));
        RL_CUDA(cudaEventRecord(cs.done[up.npanels], cs.s));
        up.done[up.npanels] = cs.done[up.npanels];
        up.row_end[up.npanels++] = r1;
        r0 = r1;
    }
    c.upload = up;
}

template <typename T>
void download(T* h, const T* d, uint64_t count) {
    if (count)
        RL_CUDA(cudaMemcpyAsync(h, d, count * sizeof(T), cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
}

void require_positive(uint64_t r, uint64_t c, const char* what) {
    if (r == 0 || c == 0)
        fail(RL_INVALID_ARGUMENT, std::string(what) + ": dimensions must be positive");
}

void minmax_fold(const double* p, uint64_t n, double* mn, double* mx) {
    double a = n ? p[0] : 0.0, b = a;
    for (uint64_t i = 0; i < n; ++i) {
        a = (p[i] < a) ? p[i] : a;
        b = (b < p[i]) ? p[i] : b;
    }
    *mn = a;
    *mx = b;
}

} // namespace

extern "C" {

const char* rl_last_error(void) { return last_error(); }

rl_status rl_init(int device) {
    API_BEGIN
    ensure_device();
    init_device(device);
    API_END
}

rl_status rl_set_stream(void* s) {
    API_BEGIN
    Ctx& c = ctx();
    // NULL selects the legacy default stream (what torch reports for its default stream)
    c.stream = s ? static_cast<cudaStream_t>(s) : cudaStreamLegacy;
    API_END
}

void* rl_get_stream(void) {
    try {
        return ctx().stream;
    } catch (...) {
        return nullptr;
    }
}

rl_status rl_synchronize(void) {
    API_BEGIN
    RL_CUDA(cudaStreamSynchronize(stream()));
    API_END
}

uint64_t rl_launch_count(void) { return total_launches(); }

// ------------------------------------------------------------ random_gen ----
rl_status rl_rng_draws(uint64_t seed, uint64_t sid, int kind, uint64_t count, int64_t lo, int64_t hi,
                       double* out) {
    API_BEGIN
    if (count == 0)
        return RL_OK;
    if (kind == RL_DRAW_UNIFORM_INT) {
        if (hi < lo)
            fail(RL_INVALID_ARGUMENT, "uniform_int: empty range");
        int64_t* d = ws<int64_t>(WS_H0, count);
        uniform_int_dev(seed, sid, count, lo, hi, d);
        std::vector<int64_t> h(count);
        download(h.data(), d, count);
        for (uint64_t i = 0; i < count; ++i)
            out[i] = static_cast<double>(h[i]);
        return RL_OK;
    }
    Draw k = kind == RL_DRAW_UNIFORM01     ? Draw::Uniform01
             : kind == RL_DRAW_UNIFORM_PM1 ? Draw::UniformPm1
             : kind == RL_DRAW_GAUSSIAN    ? Draw::Gaussian
             : kind == RL_DRAW_SIGN        ? Draw::Sign
                                           : (fail(RL_INVALID_ARGUMENT, "rng_draws: bad kind"), Draw::Sign);
    double* d = ws<double>(WS_H0, count);
    rng_generate(seed, sid, k, count, 0.0, 1.0, d);
    download(out, d, count);
    API_END
}

rl_status rl_raw_u64(uint64_t seed, uint64_t sid, uint64_t count, uint64_t* out) {
    API_BEGIN
    uint64_t* d = ws<uint64_t>(WS_H0, count);
    rng_generate(seed, sid, Draw::RawU64, count, 0.0, 1.0, d);
    download(out, d, count);
    API_END
}

rl_status rl_dev_gaussian_matrix(uint64_t m, uint64_t n, double mu, double sigma, uint64_t seed,
                                 uint64_t sid, double* d_out) {
    API_BEGIN
    if (!(sigma > 0.0))
        fail(RL_INVALID_ARGUMENT, "gaussian_matrix: sigma must be positive");
    require_positive(m, n, "gaussian_matrix");
    rng_generate(seed, sid, Draw::Gaussian, m * n, mu, sigma, d_out);
    API_END
}

rl_status rl_gaussian_matrix(uint64_t m, uint64_t n, double mu, double sigma, uint64_t seed,
                             uint64_t sid, double* out) {
    API_BEGIN
    if (!(sigma > 0.0))
        fail(RL_INVALID_ARGUMENT, "gaussian_matrix: sigma must be positive");
    require_positive(m, n, "gaussian_matrix");
    double* d = ws<double>(WS_H0, m * n);
    rng_generate(seed, sid, Draw::Gaussian, m * n, mu, sigma, d);
    download(out, d, m * n);
    API_END
}

rl_status rl_dev_uniform_matrix(uint64_t m, uint64_t n, uint64_t seed, uint64_t sid, double* d_out) {
    API_BEGIN
    require_positive(m, n, "uniform_matrix");
    rng_generate(seed, sid, Draw::UniformPm1, m * n, 0.0, 1.0, d_out);
    API_END
}

rl_status rl_uniform_matrix(uint64_t m, uint64_t n, uint64_t seed, uint64_t sid, double* out) {
    API_BEGIN
    require_positive(m, n, "uniform_matrix");
    double* d = ws<double>(WS_H0, m * n);
    rng_generate(seed, sid, Draw::UniformPm1, m * n, 0.0, 1.0, d);
    download(out, d, m * n);
    API_END
}

rl_status rl_random_structured(int tag, double mu, double sigma, uint64_t m, uint64_t n, uint64_t seed,
                               uint64_t sid, double* first_col, double* first_row) {
    API_BEGIN
    switch (tag) {
    case RL_TOEPLITZ_GAUSSIAN: { // random_gen.cpp:94-103: col[0], col[1..m-1], row[1..n-1]
        require_positive(m, n, "random_structured");
        uint64_t cnt = m + n - 1;
        double* d = ws<double>(WS_H0, cnt);
        rng_generate(seed, sid, Draw::Gaussian, cnt, mu, sigma, d);
        std::vector<double> h(cnt);
        download(h.data(), d, cnt);
        for (uint64_t i = 0; i < m; ++i)
            first_col[i] = h[i];
        if (first_row) {
            first_row[0] = h[0];
            for (uint64_t j = 1; j < n; ++j)
                first_row[j] = h[m + j - 1];
        }
        return RL_OK;
    }
    case RL_CIRCULANT_GAUSSIAN:
    case RL_CIRCULANT_SIGN: {
        if (m != n)
            fail(RL_DIMENSION_MISMATCH, "random_structured: circulant requires m == n");
        require_positive(m, n, "random_structured");
        double* d = ws<double>(WS_H0, n);
        if (tag == RL_CIRCULANT_SIGN)
            rng_generate(seed, sid, Draw::Sign, n, 0.0, 1.0, d);
        else
            rng_generate(seed, sid, Draw::Gaussian, n, mu, sigma, d);
        download(first_col, d, n);
        return RL_OK;
    }
    default:
        fail(RL_INVALID_ARGUMENT, "random_structured: kind is not structured");
    }
    API_END
}

rl_status rl_householder_sign(uint64_t n, uint64_t seed, uint64_t sid, double* out) {
    API_BEGIN
    require_positive(n, n, "householder_sign");
    // random_gen.cpp:125-143: resample (u, v) while u^T v == 0, at most 64 times
    double* uv = ws<double>(WS_H0, 2 * n * 64);
    rng_generate(seed, sid, Draw::Sign, 2 * n * 64, 0.0, 1.0, uv);
    std::vector<double> h(2 * n * 64);
    download(h.data(), uv, 2 * n * 64);
    for (int r = 0; r < 64; ++r) {
        double s = 0.0;
        for (uint64_t i = 0; i < n; ++i)
            s += h[2 * n * r + i] * h[2 * n * r + n + i];
        if (s == 0.0)
            continue;
        double* d = ws<double>(WS_H1, n * n);
        rank1_dense_dev(n, uv + 2 * n * r, uv + 2 * n * r + n, 1.0 / s, d);
        download(out, d, n * n);
        return RL_OK;
    }
    fail(RL_DEGENERATE, "householder_sign: u^T v == 0 after 64 resamples");
    API_END
}

rl_status rl_householder_pair_signs(uint64_t n, uint64_t seed, uint64_t sid, double* u1, double* u2) {
    API_BEGIN
    require_positive(n, n, "householder_pair");
    double* d = ws<double>(WS_H0, 2 * n);
    rng_generate(seed, sid, Draw::Sign, 2 * n, 0.0, 1.0, d);
    download(u1, d, n);
    download(u2, d + n, n);
    API_END
}

rl_status rl_sparse_sign(uint64_t n, int nnz, uint64_t seed, uint64_t sid, int32_t* rows, double* signs) {
    API_BEGIN
    if (nnz < 1 || nnz > 8 || static_cast<uint64_t>(nnz) > n)
        fail(RL_INVALID_ARGUMENT, "sparse_sign: need 1 <= nnz <= min(8, n)");
    int32_t* dr = ws<int32_t>(WS_H0, n * nnz);
    double* ds = ws<double>(WS_H1, n * nnz);
    rng_sparse_sign(seed, sid, n, nnz, dr, ds);
    download(rows, dr, n * nnz);
    download(signs, ds, n * nnz);
    API_END
}

rl_status rl_sparse_apply_right(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                                const double* a, double* out) {
    API_BEGIN
    require_positive(n, n, "sparse_apply_right");
    if (nnz < 1 || nnz > 8 || static_cast<uint64_t>(nnz) > n)
        fail(RL_INVALID_ARGUMENT, "sparse_apply_right: need 1 <= nnz <= min(8, n)");
    for (uint64_t e = 0; e < n * nnz; ++e)
        if (rows[e] < 0 || static_cast<uint64_t>(rows[e]) >= n)
            fail(RL_INVALID_ARGUMENT, "sparse_apply_right: row index out of range");
    int32_t* dr = ws<int32_t>(WS_H2, n * nnz);
    RL_CUDA(cudaMemcpyAsync(dr, rows, n * nnz * sizeof(int32_t), cudaMemcpyHostToDevice, stream()));
    double* ds = upload(WS_H3, signs, n * nnz);
    double* da = upload(WS_H0, a, n * n);
    double* dout = ws<double>(WS_H1, n * n);
    sparse_apply_right_dev(n, nnz, dr, ds, da, n, dout, n);
    download(out, dout, n * n);
    API_END
}

rl_status rl_dev_sparse_apply_right(uint64_t n, int nnz, const int32_t* d_rows, const double* d_signs,
                                    const double* d_a, double* d_out) {
    API_BEGIN
    require_positive(n, n, "sparse_apply_right");
    if (nnz < 1 || nnz > 8 || static_cast<uint64_t>(nnz) > n)
        fail(RL_INVALID_ARGUMENT, "sparse_apply_right: need 1 <= nnz <= min(8, n)");
    sparse_apply_right_dev(n, nnz, d_rows, d_signs, d_a, n, d_out, n);
    API_END
}

rl_status rl_dev_householder_pair_apply_right(uint64_t n, const double* d_u1, const double* d_u2,
                                              const double* d_a, double* d_out) {
    API_BEGIN
    require_positive(n, n, "householder_pair_apply_right");
    // s12 = u1^T u2 on the device (an exact integer for +-1 entries, as randomized_genp's draw has it)
    double* s12p = ws<double>(WS_FLAGS, 2);
    dot_pm1_dev(n, d_u1, d_u2, s12p);
    hh2_apply_right_dev(n, d_a, n, d_u1, d_u2, 0.0, d_out, n, s12p);
    API_END
}

rl_status rl_dev_circulant_apply_right(uint64_t m, uint64_t n, const double* d_c, const double* d_a,
                                       double* d_out) {
    API_BEGIN
    require_positive(m, n, "circulant_apply_right");
    if (d_a == d_out)
        fail(RL_INVALID_ARGUMENT, "circulant_apply_right: out must not alias a");
    if (circ_fft_supported(n)) {
        circ_apply_right_fft_dev(m, n, d_c, d_a, n, d_out, n);
    } else {
        double* dense = ws<double>(WS_TMP2, n * n);
        circulant_dense_dev(n, d_c, dense);
        gemm(false, false, m, n, n, 1.0, d_a, n, dense, n, 0.0, d_out, n);
    }
    API_END
}

rl_status rl_dev_toeplitz_apply_right(uint64_t m, uint64_t n, const double* d_g, const double* d_a,
                                      double* d_out) {
    API_BEGIN
    require_positive(m, n, "toeplitz_apply_right");
    if (d_a == d_out)
        fail(RL_INVALID_ARGUMENT, "toeplitz_apply_right: out must not alias a");
    if (toeplitz_fft_len(n) != 0) {
        toeplitz_apply_right_fft_dev(m, n, d_g, d_a, n, d_out, n);
    } else {
        double* dense = ws<double>(WS_TMP2, n * n);
        toeplitz_dense_dev(n, d_g, dense);
        gemm(false, false, m, n, n, 1.0, d_a, n, dense, n, 0.0, d_out, n);
    }
    API_END
}

rl_status rl_proto_lowrank(uint64_t m, uint64_t n, const double* a, uint64_t rho_plus, double tau,
                           double tau_prime, int tag, double mu, double sigma, uint64_t seed, uint64_t sid,
                           uint64_t* rho, double* basis, double* approx, double* residual, int* ok) {
    API_BEGIN
    require_positive(m, n, "proto_lowrank");
    if (!(tau_prime > 0.0 && tau_prime < 1.0))
        fail(RL_INVALID_ARGUMENT, "proto_lowrank: tau_prime must lie in (0, 1)");
    if (tau > 0.0 && !(tau < 1.0))
        fail(RL_INVALID_ARGUMENT, "proto_lowrank: tau must lie in (0, 1) or <= 0 for auto");
    // lowrank.cpp:116-125: ||A|| = 0 is accepted (rho 0, empty basis) before approx_basis checks
    // rho_plus or the kind
    bool all_zero = true;
    for (uint64_t i = 0; i < m * n && all_zero; ++i)
        all_zero = a[i] == 0.0;
    if (all_zero) {
        *rho = 0;
        *residual = 0.0;
        *ok = 1;
        std::memset(basis, 0, n * std::max<uint64_t>(rho_plus, 1) * sizeof(double));
        std::memset(approx, 0, m * n * sizeof(double));
        return RL_OK;
    }
    if (tag != RL_GAUSSIAN && tag != RL_TOEPLITZ_GAUSSIAN)
        fail(RL_INVALID_ARGUMENT, "proto_lowrank: the B200 path takes the Gaussian and ToeplitzGaussian kinds");
    if (rho_plus < 1 || rho_plus > std::min(m, n))
        fail(RL_INVALID_ARGUMENT, "approx_basis: rho_plus out of range");
    if (tag == RL_GAUSSIAN && !(sigma > 0.0))
        fail(RL_INVALID_ARGUMENT, "gaussian_matrix: sigma must be positive");
    if (!proto_lowrank_supported(m, n, rho_plus) && (rho_plus > 64 || rho_plus > n))
        fail(RL_TOO_LARGE, "proto_lowrank: beyond 64 x 256 the B200 path takes rho_plus <= min(64, n)");
    double* da = upload(WS_H0, a, m * n);
    double* db = ws<double>(WS_H1, n * rho_plus);
    double* dx = ws<double>(WS_H2, m * n);
    proto_lowrank_dev(m, n, da, rho_plus, tau, tau_prime, tag, mu, sigma, seed, sid, rho, db, dx, residual, ok);
    download(basis, db, n * rho_plus);
    download(approx, dx, m * n);
    API_END
}

// --------------------------------------------------------------- matrix ----
rl_status rl_matmul(uint64_t m, uint64_t k, uint64_t n, const double* a, const double* b, double* c) {
    API_BEGIN
    require_positive(m, k, "multiply");
    require_positive(k, n, "multiply");
    double* da = upload(WS_H0, a, m * k);
    double* db = upload(WS_H1, b, k * n);
    double* dc = ws<double>(WS_H2, m * n);
    gemm(false, false, m, n, k, 1.0, da, k, db, n, 0.0, dc, n);
    download(c, dc, m * n);
    API_END
}

rl_status rl_dev_gemm(int ta, int tb, uint64_t m, uint64_t n, uint64_t k, double alpha, const double* a,
                      uint64_t lda, const double* b, uint64_t ldb, double beta, double* c, uint64_t ldc) {
    API_BEGIN
    // small outputs over a long K (Q^T A of a row block, a Gram): one split-K launch + reduction
    gemm_splitk(ta != 0, tb != 0, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, splits_for(m, n, k));
    API_END
}

// ------------------------------------------------------------ structured ----
rl_status rl_circ_mul(uint64_t n, const double* c, const double* x, double* y) {
    return rl_circulant_multiply_matrix(n, c, 1, x, y);
}

rl_status rl_circulant_multiply_matrix(uint64_t n, const double* c, uint64_t cols, const double* a,
                                       double* out) {
    API_BEGIN
    require_positive(n, cols, "multiply_matrix");
    double* dc = upload(WS_H0, c, n);
    double* da = upload(WS_H1, a, n * cols);
    double* dout = ws<double>(WS_H2, n * cols);
    structured_multiply_dev(n, n, dc, nullptr, cols, da, dout);
    download(out, dout, n * cols);
    API_END
}

rl_status rl_toeplitz_mul(uint64_t m, uint64_t n, const double* col, const double* row, const double* x,
                          double* y) {
    return rl_toeplitz_multiply_matrix(m, n, col, row, 1, x, y);
}

rl_status rl_toeplitz_multiply_matrix(uint64_t m, uint64_t n, const double* col, const double* row, uint64_t cols,
                                      const double* a, double* out) {
    API_BEGIN
    require_positive(m, n, "toeplitz_mul");
    require_positive(cols, 1, "multiply_matrix");
    double* dc = upload(WS_H0, col, m);
    double* dr = upload(WS_H3, row, n);
    double* da = upload(WS_H1, a, n * cols);
    double* dout = ws<double>(WS_H2, m * cols);
    structured_multiply_dev(m, n, dc, dr, cols, da, dout);
    download(out, dout, m * cols);
    API_END
}

// ------------------------------------------------------------------ genp ----
rl_status rl_dev_genp_factor(uint64_t n, double* d_a, uint64_t lda, double pivot_floor, double* d_pivots,
                             int64_t* breakdown_step) {
    API_BEGIN
    if (pivot_floor < 0.0)
        fail(RL_INVALID_ARGUMENT, "genp_factor: pivot_floor must be >= 0");
    unsigned long long* brk = ws<unsigned long long>(WS_H3, 1);
    RL_CUDA(cudaMemsetAsync(brk, 0xff, 8, stream()));
    genp_factor_blocked(n, d_a, lda, pivot_floor, d_pivots, brk, nullptr);
    long long hb = -1;
    download(&hb, reinterpret_cast<long long*>(brk), 1);
    if (breakdown_step)
        *breakdown_step = hb;
    if (hb >= 0)
        fail(RL_PIVOT_BREAKDOWN, "genp_factor: pivot below floor at step " + std::to_string(hb));
    API_END
}

rl_status rl_genp_factor(uint64_t n, const double* a, double pivot_floor, double* l, double* u,
                         double* pivots, double* pmin_pmax, int64_t* breakdown_step) {
    API_BEGIN
    require_positive(n, n, "genp_factor");
    if (pivot_floor < 0.0)
        fail(RL_INVALID_ARGUMENT, "genp_factor: pivot_floor must be >= 0");
    double* da = upload(WS_H0, a, n * n);
    double* dp = ws<double>(WS_H1, n);
    unsigned long long* brk = ws<unsigned long long>(WS_H3, 1);
    RL_CUDA(cudaMemsetAsync(brk, 0xff, 8, stream()));
    genp_factor_blocked(n, da, n, pivot_floor, dp, brk, nullptr);
    long long hb = -1;
    download(&hb, reinterpret_cast<long long*>(brk), 1);
    if (breakdown_step)
        *breakdown_step = hb;
    if (hb >= 0)
        fail(RL_PIVOT_BREAKDOWN, "genp_factor: pivot below floor at step " + std::to_string(hb));
    double* dl = ws<double>(WS_H2, 2 * n * n);
    unpack_lu_dev(n, da, dl, dl + n * n);
    download(l, dl, n * n);
    download(u, dl + n * n, n * n);
    std::vector<double> hp(n);
    download(hp.data(), dp, n);
    if (pivots)
        std::memcpy(pivots, hp.data(), n * sizeof(double));
    if (pmin_pmax)
        minmax_fold(hp.data(), n, &pmin_pmax[0], &pmin_pmax[1]);
    API_END
}

rl_status rl_dev_genp_solve_packed(uint64_t n, uint64_t nrhs, const double* d_lu, uint64_t lda, double* d_b) {
    API_BEGIN
    double* aux = ws<double>(WS_LU_AUX, ((n + 127) / 128) * 2 * 128 * 128);
    genp_block_inverses(n, d_lu, lda, aux);
    genp_solve_blocked(n, nrhs, d_lu, lda, aux, d_b, nrhs);
    API_END
}

rl_status rl_genp_solve(uint64_t n, uint64_t nrhs, const double* l, const double* u, const double* b,
                        double* x) {
    API_BEGIN
    require_positive(n, nrhs, "genp_solve");
    double* dl = upload(WS_H0, l, n * n);
    double* du = upload(WS_H1, u, n * n);
    double* db = upload(WS_H2, b, n * nrhs);
    double* dlu = ws<double>(WS_H3, n * n);
    pack_lu_dev(n, dl, du, dlu);
    double* aux = ws<double>(WS_LU_AUX, ((n + 127) / 128) * 2 * 128 * 128);
    genp_block_inverses(n, dlu, n, aux);
    genp_solve_blocked(n, nrhs, dlu, n, aux, db, nrhs);
    download(x, db, n * nrhs);
    API_END
}

rl_status rl_dev_randomized_genp_ex(uint64_t n, uint64_t nrhs, const double* d_a, const double* d_b, int tag,
                                    double mu, double sigma, int side, int refine, uint64_t seed,
                                    uint64_t sid, double* d_x, rl_precond_report* report, uint32_t flags) {
    API_BEGIN
    require_positive(n, nrhs, "randomized_genp");
    rl_status s = randomized_genp_dev(n, nrhs, d_a, d_b, tag, mu, sigma, side, refine, seed, sid, d_x, report,
                                      flags);
    if (s != RL_OK)
        return s;
    API_END
}

rl_status rl_dev_randomized_genp(uint64_t n, uint64_t nrhs, const double* d_a, const double* d_b, int tag,
                                 double mu, double sigma, int side, int refine, uint64_t seed, uint64_t sid,
                                 double* d_x, rl_precond_report* report) {
    return rl_dev_randomized_genp_ex(n, nrhs, d_a, d_b, tag, mu, sigma, side, refine, seed, sid, d_x, report, 0);
}

rl_status rl_randomized_genp(uint64_t n, uint64_t nrhs, const double* a, const double* b, int tag, double mu,
                             double sigma, int side, int refine, uint64_t seed, uint64_t sid, double* x,
                             rl_precond_report* report) {
    return rl_randomized_genp_ex(n, nrhs, a, b, tag, mu, sigma, side, refine, seed, sid, x, report, 0);
}

rl_status rl_randomized_genp_ex(uint64_t n, uint64_t nrhs, const double* a, const double* b, int tag, double mu,
                                double sigma, int side, int refine, uint64_t seed, uint64_t sid, double* x,
                                rl_precond_report* report, uint32_t flags) {
    API_BEGIN
    require_positive(n, nrhs, "randomized_genp");
    double* db = upload(WS_H1, b, n * nrhs);
    double* da = ws<double>(WS_H0, n * n);
    upload_rows_async(da, a, n);
    double* dx = ws<double>(WS_H2, n * nrhs);
    rl_status s;
    try {
        s = randomized_genp_dev(n, nrhs, da, db, tag, mu, sigma, side, refine, seed, sid, dx, report, flags);
    } catch (...) {
        wait_upload(da);
        throw;
    }
    wait_upload(da);
    if (s != RL_OK)
        return s;
    download(x, dx, n * nrhs);
    API_END
}

rl_status rl_last_column_reports(uint64_t nrhs, rl_column_report* out) {
    API_BEGIN
    const std::vector<rl_column_report>& c = last_column_reports();
    if (c.size() != nrhs)
        fail(RL_INVALID_ARGUMENT, "last_column_reports: no randomized_genp call with this nrhs on this thread");
    std::memcpy(out, c.data(), nrhs * sizeof(rl_column_report));
    API_END
}

rl_status rl_dev_randomized_genp_batched(uint64_t batch, uint64_t n, const double* d_a, const double* d_b,
                                         int tag, double mu, double sigma, int side, int refine, uint64_t seed,
                                         const uint64_t* d_sids, double* d_x, rl_precond_report* d_reports) {
    API_BEGIN
    if (batch == 0)
        return RL_OK;
    rl_precond_report* rep = d_reports ? d_reports : ws<rl_precond_report>(WS_H3, batch);
    rl_status s = randomized_genp_batched_dev(batch, n, d_a, d_b, tag, mu, sigma, side, refine, seed, d_sids,
                                              d_x, rep);
    if (s != RL_OK) {
        set_error("randomized_genp (batched): pivot breakdown on every attempt");
        return s;
    }
    API_END
}

rl_status rl_randomized_genp_batched(uint64_t batch, uint64_t n, const double* a, const double* b, int tag,
                                     double mu, double sigma, int side, int refine, uint64_t seed,
                                     const uint64_t* sids, double* x, rl_precond_report* reports) {
    API_BEGIN
    if (batch == 0)
        return RL_OK;
    require_positive(n, n, "randomized_genp");
    double* da = upload(WS_H0, a, batch * n * n);
    double* db = upload(WS_H1, b, batch * n);
    uint64_t* ds = upload(WS_H2, sids, batch);
    double* dx = ws<double>(WS_IN_A, batch * n);
    rl_precond_report* dr = ws<rl_precond_report>(WS_IN_B, batch);
    rl_status s = randomized_genp_batched_dev(batch, n, da, db, tag, mu, sigma, side, refine, seed, ds, dx, dr);
    if (s != RL_OK) {
        set_error("randomized_genp (batched): pivot breakdown on every attempt");
        return s;
    }
    download(x, dx, batch * n);
    if (reports)
        download(reports, dr, batch);
    API_END
}

// ------------------------------------------------------- lowrank / dense ----
rl_status rl_approx_basis(uint64_t m, uint64_t n, const double* a, uint64_t rho, double mu, double sigma,
                          int space, uint64_t seed, uint64_t sid, double* y) {
    API_BEGIN
    require_positive(m, n, "approx_basis");
    if (rho < 1 || rho > std::min(m, n))
        fail(RL_INVALID_ARGUMENT, "approx_basis: rho_plus out of range");
    if (!(sigma > 0.0))
        fail(RL_INVALID_ARGUMENT, "gaussian_matrix: sigma must be positive");
    double* da = upload(WS_H0, a, m * n);
    const uint64_t rows = space == 0 ? n : m; // H is n x rho (LeftSpace), G is m x rho (RightSpace)
    double* dh = ws<double>(WS_H1, rows * rho);
    rng_generate(seed, sid, Draw::Gaussian, rows * rho, mu, sigma, dh);
    const uint64_t out_rows = space == 0 ? m : n;
    double* dy = ws<double>(WS_H2, out_rows * rho);
    if (space == 0)
        gemm(false, false, m, rho, n, 1.0, da, n, dh, rho, 0.0, dy, rho);
    else
        gemm_splitk(true, false, n, rho, m, 1.0, da, n, dh, rho, 0.0, dy, rho, splits_for(n, rho, m));
    download(y, dy, out_rows * rho);
    API_END
}

namespace {
// dense::qr_positive on device data (dense_core.cpp:86-115): shifted CholeskyQR3, then the
// reference's rank check min |R_ii| > 1e-13 sigma_1(R).  Returns R on the host too.
std::vector<double> qr_positive_dev(uint64_t m, uint64_t n, const double* dy, double* dq, double* dr) {
    if (m < n)
        fail(RL_INVALID_ARGUMENT, "qr_positive: requires rows >= cols");
    if (n > 128)
        fail(RL_TOO_LARGE, "qr_positive: more than 128 columns");
    int* flags = ws<int>(WS_FLAGS, 4);
    RL_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(int), stream()));
    cholqr3_async(m, static_cast<int>(n), dy, dq, dr, flags);
    rank_bracket_launch(static_cast<int>(n), dr, flags + 1);
    std::vector<double> hr(n * n);
    download(hr.data(), dr, n * n); // synchronises
    int hf[2];
    download(hf, flags, 2);
    if (hf[0])
        fail(RL_RANK_DEFICIENT, "qr_positive: numerically rank-deficient input");
    bool ok = hf[1] == 0;
    if (hf[1] == 2) { // between the Frobenius bounds: sigma_1(R) itself
        std::vector<double> sg = small_singular_values(static_cast<int>(n), dr);
        double min_diag = std::numeric_limits<double>::infinity();
        for (uint64_t i = 0; i < n; ++i)
            min_diag = std::min(min_diag, std::fabs(hr[i * n + i]));
        ok = min_diag > 1e-13 * sg[0];
    }
    if (!ok)
        fail(RL_RANK_DEFICIENT, "qr_positive: numerically rank-deficient input");
    return hr;
}
} // namespace

rl_status rl_qr_positive(uint64_t m, uint64_t n, const double* a, double* q, double* r) {
    API_BEGIN
    require_positive(m, n, "qr_positive");
    double* da = upload(WS_H0, a, m * n);
    double* dq = ws<double>(WS_H1, m * n);
    double* dr = ws<double>(WS_H2, n * n);
    std::vector<double> hr = qr_positive_dev(m, n, da, dq, dr);
    download(q, dq, m * n);
    std::memcpy(r, hr.data(), n * n * sizeof(double));
    API_END
}

rl_status rl_dev_qr_positive(uint64_t m, uint64_t n, const double* d_y, double* d_q, double* d_r) {
    API_BEGIN
    require_positive(m, n, "qr_positive");
    qr_positive_dev(m, n, d_y, d_q, d_r);
    API_END
}

rl_status rl_project_onto_basis_left(uint64_t m, uint64_t n, uint64_t k, const double* a, const double* q,
                                     double* sta, double* out) {
    API_BEGIN
    require_positive(m, n, "project_onto_basis");
    require_positive(k, k, "project_onto_basis");
    double* da = upload(WS_H0, a, m * n);
    double* dq = upload(WS_H1, q, m * k);
    double* ds = ws<double>(WS_H2, k * n);
    gemm_splitk(true, false, k, n, m, 1.0, dq, k, da, n, 0.0, ds, n, splits_for(k, n, m));
    if (sta)
        download(sta, ds, k * n);
    if (out) {
        double* dout = ws<double>(WS_H3, m * n);
        gemm(false, false, m, n, k, 1.0, dq, k, ds, n, 0.0, dout, n);
        download(out, dout, m * n);
    }
    API_END
}

namespace {
// dense::numerical_rank (dense_core.cpp:161-175) of device data: rank and the min(m, n)
// singular values (non-increasing).  da is not modified.
uint64_t numerical_rank_dev(uint64_t m, uint64_t n, const double* da, double tol, std::vector<double>& sg) {
    if (!(tol > 0.0 && tol < 1.0))
        fail(RL_INVALID_ARGUMENT, "numerical_rank: tol must lie in (0, 1)");
    require_positive(m, n, "numerical_rank");
    const uint64_t l = std::min(m, n);
    if (std::max(m, n) <= 128) {
        // pad to square: zero rows/columns add zero singular values only
        const uint64_t k = std::max(m, n);
        double* sq = ws<double>(WS_H1, k * k);
        RL_CUDA(cudaMemsetAsync(sq, 0, k * k * 8, stream()));
        copy2d_dev(m, n, da, n, sq, k);
        sg = small_singular_values(static_cast<int>(k), sq);
        sg.resize(l);
    } else if (l <= 128) {
        // sigma(A) = sigma(R) for the thin QR of A (m >= n) or of A^T
        const uint64_t rows = std::max(m, n), cols = l;
        double* t = ws<double>(WS_H1, rows * cols);
        if (m >= n)
            copy2d_dev(m, n, da, n, t, n);
        else
            transpose_dev(m, n, da, n, t, m);
        double fro2 = sumsq_dev(rows * cols, t);
        if (fro2 == 0.0) {
            sg.assign(l, 0.0);
        } else {
            double* dq = ws<double>(WS_H2, rows * cols);
            double* dr = ws<double>(WS_H3, cols * cols);
            if (!cholqr3(rows, static_cast<int>(cols), t, dq, dr))
                fail(RL_NO_CONVERGENCE, "numerical_rank: QR of a numerically rank-deficient matrix");
            sg = small_singular_values(static_cast<int>(cols), dr);
        }
    } else {
        fail(RL_TOO_LARGE, "numerical_rank: min(m, n) > 128 is not supported on this path");
    }
    uint64_t r = 0;
    if (!sg.empty() && sg[0] != 0.0)
        for (uint64_t j = 0; j < l; ++j)
            if (sg[j] >= tol * sg[0])
                r = j + 1;
    return r;
}
} // namespace

rl_status rl_numerical_rank(uint64_t m, uint64_t n, const double* a, double tol, uint64_t* rank, double* sigma) {
    API_BEGIN
    if (!(tol > 0.0 && tol < 1.0))
        fail(RL_INVALID_ARGUMENT, "numerical_rank: tol must lie in (0, 1)");
    require_positive(m, n, "numerical_rank");
    double* da = upload(WS_H0, a, m * n);
    std::vector<double> sg;
    *rank = numerical_rank_dev(m, n, da, tol, sg);
    if (sigma)
        std::memcpy(sigma, sg.data(), sg.size() * sizeof(double));
    API_END
}

rl_status rl_dev_numerical_rank(uint64_t m, uint64_t n, const double* d_a, double tol, uint64_t* rank,
                                double* sigma) {
    API_BEGIN
    std::vector<double> sg;
    *rank = numerical_rank_dev(m, n, d_a, tol, sg);
    if (sigma)
        std::memcpy(sigma, sg.data(), sg.size() * sizeof(double));
    API_END
}

rl_status rl_dev_range_finder(uint64_t m, uint64_t n, const double* d_a, uint64_t rho, uint64_t seed,
                              uint64_t sid, double rank_tol, double* d_q, double* d_b, double* sigma_host,
                              uint64_t* rank, double* resid_fro) {
    API_BEGIN
    require_positive(m, n, "range_finder");
    if (rho < 1 || rho > std::min<uint64_t>(std::min(m, n), 128))
        fail(RL_INVALID_ARGUMENT, "range_finder: rho_plus out of range");
    // Y = A H, H = gaussian_matrix(n, rho) (lowrank.cpp:67-84, LeftSpace)
    double* dh = ws<double>(WS_RF1, n * rho);
    rng_generate(seed, sid, Draw::Gaussian, n * rho, 0.0, 1.0, dh);
    double* dy = ws<double>(WS_RF2, m * rho);
    // both GEMM operands K-major: H^T (rho x n) and, below, Q^T (rho x m) let the TMA kernel
    // load the 72-wide operand as one box per 16 k (same k order, same bits as the N-/M-major
    // forms)
    double* dht = ws<double>(WS_RF7, n * rho);
    transpose_dev(n, rho, dh, rho, dht, n);
    gemm_splitk(false, true, m, rho, n, 1.0, d_a, n, dht, n, 0.0, dy, rho, splits_for(m, rho, n));
    // [Q, R] = qr_positive(Y), its rank test bracketed on the device (k_rank_bracket)
    double* dr = ws<double>(WS_RF3, rho * rho);
    int* flags = ws<int>(WS_FLAGS, 4);
    RL_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(int), stream()));
    // only the rank test needs R here: diag(R) and ||R||_F = ||Y||_F (no R_acc products)
    cholqr3_async(m, static_cast<int>(rho), dy, d_q, dr, flags, true, true);
    rank_bracket_diag_launch(static_cast<int>(rho), dr, flags + 1);
    // B = Q^T A (lowrank.cpp:61-64 `sta`)
    double* dqt = ws<double>(WS_RF8, m * rho);
    transpose_dev(m, rho, d_q, rho, dqt, m);
    gemm_splitk(false, false, rho, n, m, 1.0, dqt, m, d_a, n, 0.0, d_b, n, splits_for(rho, n, m));
    // sigma(B) from R of B^T
    double* bt = ws<double>(WS_RF1, n * rho);
    transpose_dev(rho, n, d_b, n, bt, rho);
    double* qb = ws<double>(WS_RF2, n * rho);
    double* rb = ws<double>(WS_RF3B, rho * rho);
    cholqr3_async(n, static_cast<int>(rho), bt, qb, rb, flags + 2, false); // R only: sigma(B) = sigma(R)
    double* dsg = ws<double>(WS_RF5B, 128 + 1);
    small_sv_launch(static_cast<int>(rho), rb, dsg);
    // one synchronisation: the flags and sigma together
    int hf[3];
    std::vector<double> sg(129);
    download(hf, flags, 3);
    download(sg.data(), dsg, 129);
    static const bool trace = getenv("RL_JACOBI_TRACE") != nullptr;
    if (trace)
        fprintf(stderr, "[rl] range finder sigma(B): %.0f sweeps\n", sg[128]);
    if (sg[128] < 0)
        fail(RL_NO_CONVERGENCE, "range_finder: Jacobi sweeps for sigma(B) did not settle");
    sg.resize(rho);
    if (hf[0])
        fail(RL_RANK_DEFICIENT, "qr_positive: numerically rank-deficient sketch");
    if (hf[1] != 0) {
        bool ok = false;
        if (hf[1] == 2) { // rare: sigma_1(R) itself — Y is rebuilt and R formed in full
            rng_generate(seed, sid, Draw::Gaussian, n * rho, 0.0, 1.0, dh);
            transpose_dev(n, rho, dh, rho, dht, n); // the same product as the first Y
            gemm_splitk(false, true, m, rho, n, 1.0, d_a, n, dht, n, 0.0, dy, rho, splits_for(m, rho, n));
            double* qtmp = ws<double>(WS_OUT, m * rho);
            if (!cholqr3(m, static_cast<int>(rho), dy, qtmp, dr))
                fail(RL_RANK_DEFICIENT, "qr_positive: numerically rank-deficient sketch");
            std::vector<double> hr(rho * rho), sr = small_singular_values(static_cast<int>(rho), dr);
            download(hr.data(), dr, rho * rho);
            double min_diag = std::numeric_limits<double>::infinity();
            for (uint64_t i = 0; i < rho; ++i)
                min_diag = std::min(min_diag, std::fabs(hr[i * rho + i]));
            ok = min_diag > 1e-13 * sr[0];
        }
        if (!ok)
            fail(RL_RANK_DEFICIENT, "qr_positive: numerically rank-deficient sketch");
    }
    if (hf[2])
        fail(RL_NO_CONVERGENCE, "range_finder: QR of B^T failed");
    if (sigma_host)
        std::memcpy(sigma_host, sg.data(), rho * sizeof(double));
    uint64_t r = 0;
    if (sg[0] != 0.0)
        for (uint64_t j = 0; j < rho; ++j)
            if (sg[j] >= rank_tol * sg[0])
                r = j + 1;
    if (rank)
        *rank = r;
    if (resid_fro) {
        // ||A - Q B||_F / ||A||_F with E formed explicitly
        double* e = ws<double>(WS_OUT, m * n);
        copy2d_dev(m, n, d_a, n, e, n);
        gemm(false, false, m, n, rho, -1.0, d_q, rho, d_b, n, 1.0, e, n);
        *resid_fro = std::sqrt(sumsq_dev(m * n, e) / sumsq_dev(m * n, d_a));
    }
    RL_CUDA(cudaStreamSynchronize(stream()));
    API_END
}

rl_status rl_rng_block(uint64_t seed, uint64_t sid, uint64_t offset, uint64_t count, uint64_t* raw) {
    API_BEGIN
    uint64_t* d = ws<uint64_t>(WS_H0, count);
    rng_generate_at(seed, sid, Draw::RawU64, offset, count, 0.0, 1.0, d);
    download(raw, d, count);
    API_END
}

rl_status rl_box_muller(uint64_t npairs, const uint64_t* raw, double* out) {
    API_BEGIN
    uint64_t* d = upload(WS_H0, raw, 2 * npairs);
    double* o = ws<double>(WS_H1, 2 * npairs);
    box_muller_pairs_dev(d, npairs, o);
    download(out, o, 2 * npairs);
    API_END
}

rl_status rl_box_muller_hash(uint64_t seed, uint64_t npairs, uint64_t chunk, uint64_t* hashes) {
    API_BEGIN
    if (chunk == 0)
        fail(RL_INVALID_ARGUMENT, "box_muller_hash: chunk must be positive");
    const uint64_t nchunks = (npairs + chunk - 1) / chunk;
    unsigned long long* dh = ws<unsigned long long>(WS_H1, nchunks ? nchunks : 1);
    box_muller_hash_dev(seed, npairs, chunk, dh);
    download(reinterpret_cast<unsigned long long*>(hashes), dh, nchunks);
    API_END
}

rl_status rl_fft(uint64_t n, const double* in, int inverse, double* out) {
    API_BEGIN
    if (n == 0 || (n & (n - 1)))
        fail(RL_LENGTH_NOT_POW2, "fft: length must be a power of two");
    double* d = upload(WS_H0, in, 2 * n);
    double* o = ws<double>(WS_H1, 2 * n);
    fft_exact_dev(n, 1, reinterpret_cast<const double2*>(d), reinterpret_cast<double2*>(o), inverse);
    download(out, o, 2 * n);
    API_END
}

rl_status rl_norm(uint64_t m, uint64_t n, const double* a, int kind, double* out) {
    API_BEGIN
    require_positive(m, n, "norm");
    double* d = upload(WS_H0, a, m * n);
    if (kind == 3) {
        *out = std::sqrt(sumsq_dev(m * n, d));
    } else if (kind == 0 || kind == 2) {
        const uint64_t cnt = kind == 2 ? m : n;
        double* v = ws<double>(WS_H1, cnt);
        abs_sums_dev(m, n, d, kind == 2, v);
        std::vector<double> h(cnt);
        download(h.data(), v, cnt);
        double best = 0.0;
        for (double x : h)
            best = std::max(best, x);
        *out = best;
    } else {
        uint64_t r = 0;
        std::vector<double> sg(std::min(m, n));
        rl_status st = rl_numerical_rank(m, n, a, 0.5, &r, sg.data());
        if (st != RL_OK)
            return st;
        *out = sg.empty() ? 0.0 : sg[0];
    }
    API_END
}

// ------------------------------------------------------------ rank search ----
rl_status rl_extremal_sv_estimate(uint64_t m, uint64_t n, const double* a, int method, int iters, uint64_t seed,
                                  uint64_t sid, double* sv_max, double* sv_min) {
    API_BEGIN
    require_positive(m, n, "extremal_sv_estimate");
    if (method != 0 && method != 1)
        fail(RL_INVALID_ARGUMENT, "extremal_sv_estimate: method must be Power (0) or Lanczos (1)");
    double* da = upload(WS_H0, a, m * n);
    extremal_sv_dev(m, n, da, n, method, iters, seed, sid, sv_max, sv_min);
    API_END
}

rl_status rl_cond_probe(uint64_t m, uint64_t n, const double* b, double kappa, int method, int iters, uint64_t seed,
                        uint64_t sid, int* pass) {
    API_BEGIN
    require_positive(m, n, "cond_probe");
    double* db = upload(WS_H0, b, m * n);
    *pass = cond_probe_dev(m, n, db, n, kappa, method, iters, seed, sid) ? 1 : 0;
    API_END
}

rl_status rl_nrank_search(uint64_t m, uint64_t n, const double* a, uint64_t rho_minus, uint64_t rho_plus,
                          double kappa, int policy, uint64_t seed, uint64_t sid, uint64_t* rho, double* basis,
                          uint64_t* basis_rows, uint64_t* basis_cols) {
    API_BEGIN
    require_positive(m, n, "nrank_search");
    double* da = upload(WS_H0, a, m * n);
    double* db = ws<double>(WS_H1, std::max(m, n) * std::max<uint64_t>(rho_plus, 1));
    uint64_t rows = 0;
    const uint64_t r = nrank_search_dev(m, n, da, rho_minus, rho_plus, kappa, policy, seed, sid, db, &rows);
    *rho = r;
    *basis_rows = rows;
    *basis_cols = r > 0 ? r : 1; // the reference's Matrix(n, 1) when rho = 0
    if (r > 0)
        download(basis, db, rows * r);
    else
        std::memset(basis, 0, rows * sizeof(double));
    API_END
}

rl_status rl_power_transform(uint64_t m, uint64_t n, const double* a, unsigned h, double* out) {
    API_BEGIN
    require_positive(m, n, "power_transform");
    double* da = upload(WS_H0, a, m * n);
    double* cur = ws<double>(WS_H2, m * n);
    copy2d_dev(m, n, da, n, cur, n);
    if (h > 0) { // (A A^T)^h A (lowrank.cpp:179-187)
        double* aat = ws<double>(WS_H1, m * m);
        double* nxt = ws<double>(WS_H3, m * n);
        gemm(false, true, m, m, n, 1.0, da, n, da, n, 0.0, aat, m);
        for (unsigned i = 0; i < h; ++i) {
            gemm(false, false, m, n, m, 1.0, aat, m, cur, n, 0.0, nxt, n);
            std::swap(cur, nxt);
        }
    }
    download(out, cur, m * n);
    API_END
}

rl_status rl_probe_peaks(double* fp64_tflops, double* hbm_gbs) {
    API_BEGIN
    return probe_peaks(fp64_tflops, hbm_gbs);
    API_END
}

} // extern "C"

/* rl_b200.h — C-ABI of the B200-native randomized-multiplier GENP / range finder.
 *
 * This is the thin layer the C++ drop-in (include/randla/*.hpp, the reference's
 * own API) calls, and what any FFI (ctypes, cgo, JNI, ...) would bind: plain
 * pointers and sizes, row-major storage with leading dimension = cols (the
 * reference's layout, proj/include/randla/matrix.hpp:28), status codes instead
 * of exceptions.  Every entry point names the reference interface it replaces.
 *
 *  - rl_*      : HOST pointers in/out; the call copies to the GPU, runs the CUDA
 *                path, copies back and synchronises (the reference's value
 *                semantics).
 *  - rl_dev_*  : DEVICE pointers; enqueued on the calling thread's stream
 *                (rl_set_stream), no host synchronisation unless stated.
 *
 * Thread safety: every entry point is reentrant.  Each calling thread gets its
 * own CUDA stream and workspace; results never depend on scheduling (no
 * atomics-order-dependent sums), as the reference's parallel_trials requires
 * (proj/src/bench.cpp:63-93, tests/test_bench.cpp:57-73).
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns RL_NO_DEVICE.
 */
#ifndef RL_B200_H
#define RL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 1:1 with the randla::Error hierarchy, proj/include/randla/errors.hpp:9-59. */
typedef enum {
    RL_OK = 0,
    RL_DIMENSION_MISMATCH = 1,   /* randla::DimensionMismatch */
    RL_INVALID_ARGUMENT = 2,     /* randla::InvalidArgument */
    RL_PIVOT_BREAKDOWN = 3,      /* randla::PivotBreakdown */
    RL_RANK_DEFICIENT = 4,       /* randla::RankDeficient */
    RL_DEGENERATE = 5,           /* randla::Degenerate */
    RL_LENGTH_NOT_POW2 = 6,      /* randla::LengthNotPowerOfTwo */
    RL_INDEX_OUT_OF_RANGE = 7,   /* randla::IndexOutOfRange */
    RL_NO_CONVERGENCE = 8,       /* randla::NoConvergence */
    RL_ZERO_MATRIX = 9,          /* randla::ZeroMatrix */
    RL_CONSTRUCTION_FAILED = 10, /* randla::ConstructionFailed */
    RL_ERROR = 11,               /* randla::Error (e.g. structured.cpp:44-45) */
    RL_TOO_LARGE = 12,           /* randla::TooLarge */
    RL_CUDA_ERROR = 20,          /* CUDA runtime failure (message in rl_last_error) */
    RL_NO_DEVICE = 21            /* no CUDA device: there is no CPU fallback */
} rl_status;

/* rnd::MultiplierTag (random_gen.hpp:46-53) + two additive extensions. */
typedef enum {
    RL_GAUSSIAN = 0,
    RL_UNIFORM_PM1 = 1,
    RL_TOEPLITZ_GAUSSIAN = 2,
    RL_CIRCULANT_GAUSSIAN = 3,
    RL_CIRCULANT_SIGN = 4,
    RL_HOUSEHOLDER_SIGN = 5,
    RL_HOUSEHOLDER_PAIR = 6, /* NEW: H1 H2, H_i = I - 2 u_i u_i^T / n, u_i in {+-1}^n */
    RL_SPARSE_SIGN = 7       /* NEW: 4 nonzeros +-1 per column at uniform rows */
} rl_multiplier_tag;

/* genp::MulSide (genp.hpp:49) */
typedef enum { RL_LEFT = 0, RL_RIGHT = 1, RL_BOTH = 2 } rl_mul_side;

/* genp::PrecondReport (genp.hpp:51-60) + which attempt was kept. */
typedef struct {
    double residual;      /* ||A y - b|| / ||b|| after the preconditioned solve (max over RHS) */
    double raw_residual;  /* same for plain GENP on A (the failure arm) */
    double pivot_min;
    double pivot_max;
    double raw_pivot_min;
    double raw_pivot_max;
    int32_t attempt;        /* index of the returned attempt (0..7) */
    int32_t attempts_drawn; /* multipliers drawn (1 + redraws) */
} rl_precond_report;

/* RNG draw kinds for rl_rng_draws (rnd::Rng methods, random_gen.cpp:33-70). */
typedef enum { RL_DRAW_UNIFORM01 = 0, RL_DRAW_UNIFORM_PM1 = 1, RL_DRAW_GAUSSIAN = 2,
               RL_DRAW_SIGN = 3, RL_DRAW_UNIFORM_INT = 4 } rl_draw_kind;

/* ----------------------------------------------------------- runtime ---- */
const char* rl_last_error(void);                 /* thread-local message of the last failure */
rl_status rl_init(int device);                   /* select device, load jump tables */
rl_status rl_set_stream(void* cuda_stream);      /* stream for this thread's rl_dev_* calls; NULL = legacy default */
void* rl_get_stream(void);
rl_status rl_synchronize(void);
/* Number of this library's kernel launches on the calling thread so far. */
uint64_t rl_launch_count(void);

/* ------------------------------------- random_gen.hpp (random_gen.cpp) ---- */
/* rnd::Rng draws (random_gen.cpp:22-70): count draws of one kind from stream (seed, stream_id). */
rl_status rl_rng_draws(uint64_t seed, uint64_t stream_id, int kind, uint64_t count, int64_t lo,
                       int64_t hi, double* out);
/* Raw tempered mt19937_64 outputs after Rng's discard(8) (random_gen.cpp:29-30). */
rl_status rl_raw_u64(uint64_t seed, uint64_t stream_id, uint64_t count, uint64_t* out);
/* rnd::gaussian_matrix (random_gen.cpp:72-80) */
rl_status rl_gaussian_matrix(uint64_t m, uint64_t n, double mu, double sigma, uint64_t seed,
                             uint64_t stream_id, double* out);
rl_status rl_dev_gaussian_matrix(uint64_t m, uint64_t n, double mu, double sigma, uint64_t seed,
                                 uint64_t stream_id, double* d_out);
/* rnd::uniform_matrix (random_gen.cpp:82-88) */
rl_status rl_uniform_matrix(uint64_t m, uint64_t n, uint64_t seed, uint64_t stream_id, double* out);
rl_status rl_dev_uniform_matrix(uint64_t m, uint64_t n, uint64_t seed, uint64_t stream_id,
                                double* d_out);
/* rnd::random_structured (random_gen.cpp:90-123): first_col (m) and, for Toeplitz, first_row (n). */
rl_status rl_random_structured(int tag, double mu, double sigma, uint64_t m, uint64_t n,
                               uint64_t seed, uint64_t stream_id, double* first_col,
                               double* first_row);
/* rnd::householder_sign (random_gen.cpp:125-143): dense I - u v^T/(u^T v). */
rl_status rl_householder_sign(uint64_t n, uint64_t seed, uint64_t stream_id, double* out);
/* NEW: signs u1, u2 of the orthogonal Householder pair. */
rl_status rl_householder_pair_signs(uint64_t n, uint64_t seed, uint64_t stream_id, double* u1,
                                    double* u2);
/* NEW: sparse +-1 multiplier, rows[n][nnz], signs[n][nnz] per column. */
rl_status rl_sparse_sign(uint64_t n, int nnz, uint64_t seed, uint64_t stream_id, int32_t* rows,
                         double* signs);
/* NEW: out = A S for the sparse +-1 S above (A, out n x n row-major): the multiplier stage of
 * randomized_genp's Right side with RL_SPARSE_SIGN (genp.cpp:175-180 applies M on the right). */
rl_status rl_sparse_apply_right(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                                const double* a, double* out);
/* Device-pointer variants of the two matrix-free right multipliers (calling thread's stream):
 * out = A S (sparse +-1, d_rows/d_signs n x nnz) and out = A H1 H2 (Householder pair,
 * H_i = I - (2/n) u_i u_i^T, d_u1/d_u2 n signs).  out may alias a only for the pair. */
rl_status rl_dev_sparse_apply_right(uint64_t n, int nnz, const int32_t* d_rows, const double* d_signs,
                                    const double* d_a, double* d_out);
rl_status rl_dev_householder_pair_apply_right(uint64_t n, const double* d_u1, const double* d_u2,
                                              const double* d_a, double* d_out);
/* out = A C for the circulant C(i,j) = c[(i-j) mod n] (structured::circulant, structured.cpp:54-68;
 * randomized_genp's Right side with CirculantSign / CirculantGaussian, genp.cpp:175-180):
 * A, out m x n row-major on the device, out != a.  Power-of-two 64 <= n <= 8192 go through the
 * FFT (matrix-free, O(m n log n)); other n through a dense product. */
rl_status rl_dev_circulant_apply_right(uint64_t m, uint64_t n, const double* d_c, const double* d_a,
                                       double* d_out);
/* out = A T for the n x n Toeplitz T(i,j) = col[i-j] (i >= j), row[j-i] (j > i) (structured::toeplitz,
 * structured.cpp:61-68; toeplitz_mul's circulant embedding, :156-176): d_g = col[0..n-1] followed by
 * row[1..n-1] (random_structured's draw order).  FFT of the embedding for next_pow2(2n-1) <= 8192,
 * a dense product otherwise; out != a. */
/* lowrank::proto_lowrank (lowrank.cpp:108-177) for the Gaussian and ToeplitzGaussian kinds
 * (RightSpace sketches A^T G on stream stream_id + 104729 a, a = 0..3): host pointers, a m x n; basis n x rho_plus
 * (its first *rho columns are the orthonormal basis), approx m x n; small matrices only
 * (min(m, n) <= 64, max(m, n) <= 256, rho_plus <= 64; RL_TOO_LARGE otherwise). */
rl_status rl_proto_lowrank(uint64_t m, uint64_t n, const double* a, uint64_t rho_plus, double tau,
                           double tau_prime, int tag, double mu, double sigma, uint64_t seed, uint64_t stream_id,
                           uint64_t* rho, double* basis, double* approx, double* residual, int* ok);
rl_status rl_dev_toeplitz_apply_right(uint64_t m, uint64_t n, const double* d_g, const double* d_a,
                                      double* d_out);

/* -------------------------------------------- matrix.hpp (matrix.cpp) ---- */
/* Matrix::multiply(const Matrix&) (matrix.cpp:86-102): C(m x n) = A(m x k) B(k x n). */
rl_status rl_matmul(uint64_t m, uint64_t k, uint64_t n, const double* a, const double* b, double* c);
/* Device GEMM, row-major: C = alpha op(A) op(B) + beta C; trans = 0 (N) or 1 (T). */
rl_status rl_dev_gemm(int trans_a, int trans_b, uint64_t m, uint64_t n, uint64_t k, double alpha,
                      const double* d_a, uint64_t lda, const double* d_b, uint64_t ldb, double beta,
                      double* d_c, uint64_t ldc);

/* ------------------------------------ structured.hpp (structured.cpp) ---- */
/* The structured products are the reference's FFT algorithms executed step for step on the GPU
 * (csrc/fft_exact.cu): the same bits as the reference, O(n log n), matrix-free. A column whose
 * imaginary residue fails take_real's test (structured.cpp:39-50) returns RL_ERROR
 * ("structured product: imaginary residue exceeds tolerance", randla::Error).
 * structured::circ_mul (structured.cpp:132-154): y = C x, C circulant with first column c. */
rl_status rl_circ_mul(uint64_t n, const double* c, const double* x, double* y);
/* structured::multiply_matrix for a circulant spec (structured.cpp:178-189): out = C A, A n x cols. */
rl_status rl_circulant_multiply_matrix(uint64_t n, const double* c, uint64_t cols, const double* a,
                                       double* out);
/* structured::toeplitz_mul (structured.cpp:156-176): y = T x, T m x n with first column col (m)
 * and first row row (n), col[0] == row[0]. */
rl_status rl_toeplitz_mul(uint64_t m, uint64_t n, const double* col, const double* row, const double* x,
                          double* y);
/* structured::multiply_matrix for a Toeplitz spec: out = T A, A n x cols, out m x cols. */
rl_status rl_toeplitz_multiply_matrix(uint64_t m, uint64_t n, const double* col, const double* row, uint64_t cols,
                                      const double* a, double* out);

/* ---------------------------------------------------- genp.hpp (genp.cpp) ---- */
/* genp::genp_factor (genp.cpp:11-41): separate unit-lower L and upper U, |pivots|,
 * pmin_pmax[2].  On PivotBreakdown, *breakdown_step (may be NULL) = first step k. */
rl_status rl_genp_factor(uint64_t n, const double* a, double pivot_floor, double* l, double* u,
                         double* pivots, double* pmin_pmax, int64_t* breakdown_step);
/* Device, in place, packed (L strictly below the diagonal, U on/above), blocked. */
rl_status rl_dev_genp_factor(uint64_t n, double* d_a, uint64_t lda, double pivot_floor,
                             double* d_pivots, int64_t* breakdown_step);
/* genp::genp_solve (genp.cpp:106-124), extended to nrhs right-hand sides:
 * B (n x nrhs, row-major) -> X. */
rl_status rl_genp_solve(uint64_t n, uint64_t nrhs, const double* l, const double* u,
                        const double* b, double* x);
rl_status rl_dev_genp_solve_packed(uint64_t n, uint64_t nrhs, const double* d_lu, uint64_t lda,
                                   double* d_b);
/* genp::randomized_genp (genp.cpp:207-291), extended to nrhs right-hand sides
 * (nrhs = 1 is the reference call).  B is n x nrhs row-major; report may be NULL. */
rl_status rl_randomized_genp(uint64_t n, uint64_t nrhs, const double* a, const double* b, int tag,
                             double mu, double sigma, int side, int refine, uint64_t seed,
                             uint64_t stream_id, double* x, rl_precond_report* report);
rl_status rl_randomized_genp_ex(uint64_t n, uint64_t nrhs, const double* a, const double* b,
                                int tag, double mu, double sigma, int side, int refine,
                                uint64_t seed, uint64_t stream_id, double* x,
                                rl_precond_report* report, uint32_t flags);
rl_status rl_dev_randomized_genp(uint64_t n, uint64_t nrhs, const double* d_a, const double* d_b,
                                 int tag, double mu, double sigma, int side, int refine,
                                 uint64_t seed, uint64_t stream_id, double* d_x,
                                 rl_precond_report* report);
/* Same with flags: bit 0 = skip the raw-GENP contrast arm (report.raw_* left 0).
 * The benchmark's config-3 step uses it: the configuration times the preconditioned
 * pipeline (A G, GENP, solves, x = G y) only. */
#define RL_FLAG_SKIP_RAW_ARM 1u
rl_status rl_dev_randomized_genp_ex(uint64_t n, uint64_t nrhs, const double* d_a, const double* d_b,
                                    int tag, double mu, double sigma, int side, int refine,
                                    uint64_t seed, uint64_t stream_id, double* d_x,
                                    rl_precond_report* report, uint32_t flags);
/* Per-right-hand-side outcome of the calling thread's last randomized_genp call: column j is
 * the reference call randomized_genp(a, B[:, j], ...) (genp.cpp:207-291) — the first attempt
 * whose residual <= 1e-7, else its best — so `attempt` is that call's accepted draw and
 * `attempts_drawn` how many draws that call would make. Fails with RL_INVALID_ARGUMENT when
 * nrhs differs from the last call's. */
typedef struct {
    double residual, pivot_min, pivot_max;
    int32_t attempt, attempts_drawn;
} rl_column_report;
rl_status rl_last_column_reports(uint64_t nrhs, rl_column_report* out);
/* Batched randomized_genp: `batch` independent systems A[t] (n x n), b[t] (n), each
 * with stream (seed, stream_ids[t]) — semantically the loop bench::table1_genp runs
 * (bench.cpp:117-133).  Host pointers; reports may be NULL. */
rl_status rl_randomized_genp_batched(uint64_t batch, uint64_t n, const double* a, const double* b,
                                     int tag, double mu, double sigma, int side, int refine,
                                     uint64_t seed, const uint64_t* stream_ids, double* x,
                                     rl_precond_report* reports);
rl_status rl_dev_randomized_genp_batched(uint64_t batch, uint64_t n, const double* d_a,
                                         const double* d_b, int tag, double mu, double sigma,
                                         int side, int refine, uint64_t seed,
                                         const uint64_t* d_stream_ids, double* d_x,
                                         rl_precond_report* d_reports);

/* ------------------------- lowrank.hpp / dense_core.hpp (lowrank.cpp, dense_core.cpp) ---- */
/* lowrank::approx_basis, Gaussian kind (lowrank.cpp:67-84): LeftSpace (space=0) Y = A H,
 * H = gaussian_matrix(n, rho_plus); RightSpace (space=1) Y = A^T G, G = gaussian_matrix(m, rho_plus). */
rl_status rl_approx_basis(uint64_t m, uint64_t n, const double* a, uint64_t rho_plus, double mu,
                          double sigma, int space, uint64_t seed, uint64_t stream_id, double* y);
/* dense::qr_positive (dense_core.cpp:86-115): thin Q (m x n), R (n x n), diag(R) > 0. */
rl_status rl_qr_positive(uint64_t m, uint64_t n, const double* a, double* q, double* r);
/* lowrank::project_onto_basis, orthonormal, Side::Left (lowrank.cpp:61-64):
 * sta = Q^T A (k x n), out = Q sta (m x n); either output may be NULL. */
rl_status rl_project_onto_basis_left(uint64_t m, uint64_t n, uint64_t k, const double* a,
                                     const double* q, double* sta, double* out);
/* dense::numerical_rank (dense_core.cpp:161-175) + the singular values (min(m,n)). */
rl_status rl_numerical_rank(uint64_t m, uint64_t n, const double* a, double tol, uint64_t* rank,
                            double* sigma);
/* Device-data variants of the two above (the sharded range finder's per-rank pieces):
 * d_y, d_q m x n, d_r n x n (n <= 128); d_a m x n with min(m, n) <= 128; sigma on the host. */
rl_status rl_dev_qr_positive(uint64_t m, uint64_t n, const double* d_y, double* d_q, double* d_r);
rl_status rl_dev_numerical_rank(uint64_t m, uint64_t n, const double* d_a, double tol, uint64_t* rank,
                                double* sigma);
/* The fused range finder on device data: Y = A H, [Q,R] = qr_positive(Y),
 * B = Q^T A, sigma(B), rank at tol, ||A - Q B||_F / ||A||_F.  d_q (m x k), d_b (k x n). */
rl_status rl_dev_range_finder(uint64_t m, uint64_t n, const double* d_a, uint64_t rho_plus,
                              uint64_t seed, uint64_t stream_id, double rank_tol, double* d_q,
                              double* d_b, double* sigma_host, uint64_t* rank, double* resid_fro);

/* ------------------------------------------ support for the C++ drop-in ---- */
/* Raw draws [offset, offset+count) of stream (seed, stream_id) (rnd::Rng's engine outputs
 * after discard(8)); lets the C++ Rng buffer its sequential draws from the GPU. */
rl_status rl_rng_block(uint64_t seed, uint64_t stream_id, uint64_t offset, uint64_t count,
                       uint64_t* raw);
/* Box-Muller of npairs consecutive raw pairs (random_gen.cpp:46-52): out[2q] = r cos a,
 * out[2q+1] = r sin a. */
rl_status rl_box_muller(uint64_t npairs, const uint64_t* raw, double* out);
/* Checksums of the GPU Box-Muller over npairs splitmix64 pairs (pair q: raw words
 * splitmix64 of seed + 2q, twice): hashes[c] = wrapping sum over q in chunk c of
 * pair_hash(q, bits(g0), bits(g1)) (csrc/glibc_math.cuh). Lets a host program check 2^30 pairs
 * against its own libm without moving the outputs (tests/cpp/bm_libm_check.cpp). */
rl_status rl_box_muller_hash(uint64_t seed, uint64_t npairs, uint64_t chunk, uint64_t* hashes);
/* structured::fft (structured.cpp:96-130), bit for bit: complex interleaved (re, im), n a power
 * of two (else RL_LENGTH_NOT_POW2), inverse scaled by 1/n. O(n log n) on the GPU. */
rl_status rl_fft(uint64_t n, const double* in, int inverse, double* out);
/* dense::norm (dense_core.cpp:48-84): kind 0 One, 1 Two, 2 Inf, 3 Frobenius. */
rl_status rl_norm(uint64_t m, uint64_t n, const double* a, int kind, double* out);

/* ----------------------------- lowrank.hpp rank search (lowrank.cpp:179-396) ---- */
/* lowrank::extremal_sv_estimate (lowrank.cpp:204-348): method 0 Power, 1 Lanczos; the start
 * vectors are the stream's Gaussians. RL_NO_CONVERGENCE as the reference's NoConvergence. */
rl_status rl_extremal_sv_estimate(uint64_t m, uint64_t n, const double* a, int method, int iters, uint64_t seed,
                                  uint64_t stream_id, double* sv_max, double* sv_min);
/* lowrank::cond_probe (lowrank.cpp:350-358): *pass = 1 when sv_max / sv_min <= kappa. */
rl_status rl_cond_probe(uint64_t m, uint64_t n, const double* b, double kappa, int method, int iters, uint64_t seed,
                        uint64_t stream_id, int* pass);
/* lowrank::nrank_search (lowrank.cpp:360-396): policy 0 Binary, 1 LinearDown. basis (capacity
 * max(m, n) x rho_plus) receives the sketch at the final rank, *basis_rows x *basis_cols (the
 * reference's n x 1 zero matrix when rho = 0). */
rl_status rl_nrank_search(uint64_t m, uint64_t n, const double* a, uint64_t rho_minus, uint64_t rho_plus,
                          double kappa, int policy, uint64_t seed, uint64_t stream_id, uint64_t* rho, double* basis,
                          uint64_t* basis_rows, uint64_t* basis_cols);
/* lowrank::power_transform (lowrank.cpp:179-187): (A A^T)^h A. */
rl_status rl_power_transform(uint64_t m, uint64_t n, const double* a, unsigned h, double* out);

/* -------------------------------------------------------- probes (K12) ---- */
/* Measured peaks on the current device: FP64 DMMA TFLOP/s and HBM copy GB/s. */
rl_status rl_probe_peaks(double* fp64_tflops, double* hbm_gbs);

#ifdef __cplusplus
}
#endif
#endif /* RL_B200_H */

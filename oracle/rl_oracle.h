/* TEST INFRASTRUCTURE ONLY — the CPU oracle.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline, never as the product path.
 *
 * Plain-C restatement of the reference hot path (randla, /root/reference/proj),
 * function by function with the reference file:line it follows.  Pinned against
 * the reference itself (oracle/_ref/librandla_ref.so, compiled from the untouched
 * reference sources by oracle/Makefile) and against tests/golden/ fixtures made by
 * tests/golden/make_golden.py.  The two NEW multipliers (Householder pair, sparse
 * +-1) have no reference implementation; their protocol is defined here on top of
 * the reference's pinned Rng draws.
 */
#ifndef RL_ORACLE_H
#define RL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t mt[312];
    int idx;
    int has_cached;
    double cached;
} rlo_rng;

/* Row-parallel worker threads for the full-size parity runs (default 1; bit-identical). */
void rlo_set_threads(int t);

void rlo_rng_init(rlo_rng* r, uint64_t seed, uint64_t sid);
uint64_t rlo_next_u64(rlo_rng* r);
double rlo_uniform01(rlo_rng* r);
double rlo_uniform_pm1(rlo_rng* r);
double rlo_gaussian(rlo_rng* r);
double rlo_sign(rlo_rng* r);
int64_t rlo_uniform_int(rlo_rng* r, int64_t lo, int64_t hi);

/* Raw tempered outputs after the constructor's discard(8). */
void rlo_raw_u64(uint64_t seed, uint64_t sid, uint64_t count, uint64_t* out);
int rlo_gaussian_matrix(uint64_t m, uint64_t n, double mu, double sigma, uint64_t seed,
                        uint64_t sid, double* out);
void rlo_uniform_matrix(uint64_t m, uint64_t n, uint64_t seed, uint64_t sid, double* out);
void rlo_sign_vector(uint64_t n, uint64_t seed, uint64_t sid, double* out);
void rlo_householder_pair_signs(uint64_t n, uint64_t seed, uint64_t sid, double* u1, double* u2);
int rlo_sparse_pm1(uint64_t n, int nnz, uint64_t seed, uint64_t sid, int32_t* rows, double* signs);

void rlo_matmul(uint64_t m, uint64_t k, uint64_t n, const double* a, const double* b, double* c);
void rlo_matvec(uint64_t m, uint64_t n, const double* a, const double* x, double* y);
void rlo_transpose(uint64_t m, uint64_t n, const double* a, double* t);

/* In-place packed GENP (unit L strictly below the diagonal, U on/above).
 * Returns 0, or -(k+1) when |pivot_k| < floor.  pivots may be NULL. */
int rlo_genp_factor(uint64_t n, double* w, double pivot_floor, double* pivots);
void rlo_genp_solve(uint64_t n, const double* lu, const double* b, double* y);
double rlo_relative_residual(uint64_t n, const double* a, const double* y, const double* b);

int rlo_fft(uint64_t n, double* re, double* im, int inverse);
int rlo_circ_mul(uint64_t n, const double* c, const double* x, double* y);
void rlo_svd_left(uint64_t m, uint64_t n, const double* a, double* sigma, double* u);
int rlo_proto_lowrank(uint64_t m, uint64_t n, const double* a, uint64_t rho_plus, double tau, double tau_prime,
                      int tag, double mu, double sig_g, uint64_t seed, uint64_t sid, uint64_t* rho_out,
                      double* basis, double* approx, double* residual, int* ok);
int rlo_toeplitz_mul(uint64_t m, uint64_t n, const double* col, const double* row, const double* x, double* y);
int rlo_circ_apply_left(uint64_t n, const double* c, uint64_t cols, const double* a, double* out);
int rlo_circ_apply_right(uint64_t n, const double* c, const double* a, double* out);

void rlo_hh2_apply_right(uint64_t n, const double* u1, const double* u2, const double* a, double* out);
void rlo_hh2_apply_vec(uint64_t n, const double* u1, const double* u2, const double* y, double* x);
void rlo_sparse_apply_right(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                            const double* a, double* out);
void rlo_sparse_apply_vec(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                          const double* y, double* x);

/* report[6] = residual, raw_residual, pivot_min, pivot_max, raw_pivot_min, raw_pivot_max;
 * extra[2] (may be NULL) = accepted attempt index, attempts drawn. */
int rlo_randomized_genp(uint64_t n, const double* a, const double* b, int tag, double mu,
                        double sigma, int side, int refine, uint64_t seed, uint64_t sid, double* y,
                        double* report, int* extra);
/* randomized_genp for nrhs columns sharing the draws (per column bit-identical to the single
 * call); B, Y row-major n x nrhs, reports nrhs x 6, extras nrhs x 2. */
int rlo_randomized_genp_multi(uint64_t n, uint64_t nrhs, const double* a, const double* B, int tag, double mu,
                              double sigma, int side, int refine, uint64_t seed, uint64_t sid, int skip_raw,
                              double* Y, double* reports, int* extras);

int rlo_qr_positive(uint64_t m, uint64_t n, const double* a, double* q, double* r);
void rlo_singular_values(uint64_t m, uint64_t n, const double* a, double* sigma);
uint64_t rlo_numerical_rank(uint64_t l, const double* sigma, double tol);

#ifdef __cplusplus
}
#endif
#endif

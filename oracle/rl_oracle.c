/* TEST INFRASTRUCTURE ONLY — CPU oracle (see rl_oracle.h).  Never the product
 * path: the product (paper_1212_4560_b200/, libs under paper_1212_4560_b200/lib)
 * never links or loads this file.
 *
 * Compiled with -O3 -ffp-contract=off and no -march, like the reference's
 * Release build (proj/CMakeLists.txt:6-8), so a*b+c is never fused and results
 * are bit-identical to oracle/_ref/librandla_ref.so on the same inputs
 * (tests/test_oracle.py checks this).
 */
#define _POSIX_C_SOURCE 200809L
#include "rl_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

/* Optional row-parallelism for the full-size parity runs (tools/fullsize_parity.py):
 * rows of the product and of each elimination step are independent, so the threaded
 * results are bit-identical to the sequential ones. */
#include <pthread.h>
static int g_threads = 1;
void rlo_set_threads(int t) { g_threads = t < 1 ? 1 : (t > 256 ? 256 : t); }

typedef void (*row_fn)(uint64_t lo, uint64_t hi, void* arg);
struct par_job {
    row_fn fn;
    void* arg;
    uint64_t lo, hi;
};
static void* par_entry(void* p) {
    struct par_job* j = (struct par_job*)p;
    j->fn(j->lo, j->hi, j->arg);
    return NULL;
}
static void par_rows(uint64_t m, row_fn fn, void* arg) {
    pthread_t th[256];
    struct par_job jobs[256];
    int t = g_threads;
    for (int i = 0; i < t; ++i) {
        jobs[i].fn = fn;
        jobs[i].arg = arg;
        jobs[i].lo = m * (uint64_t)i / (uint64_t)t;
        jobs[i].hi = m * (uint64_t)(i + 1) / (uint64_t)t;
        pthread_create(&th[i], NULL, par_entry, &jobs[i]);
    }
    for (int i = 0; i < t; ++i)
        pthread_join(th[i], NULL);
}

struct mm_args {
    uint64_t k, n;
    const double *a, *b;
    double* c;
};
static void matmul_rows(uint64_t lo, uint64_t hi, void* p) {
    struct mm_args* g = (struct mm_args*)p;
    for (uint64_t i = lo; i < hi; ++i)
        for (uint64_t kk = 0; kk < g->k; ++kk) {
            double av = g->a[i * g->k + kk];
            if (av == 0.0)
                continue;
            const double* rr = g->b + kk * g->n;
            double* orow = g->c + i * g->n;
            for (uint64_t j = 0; j < g->n; ++j)
                orow[j] += av * rr[j];
        }
}

/* threaded elimination: each worker owns the rows i == tid (mod t); two barriers per step */
struct ge_shared {
    uint64_t n;
    double* w;
    double floor;
    double* pivots;
    pthread_barrier_t bar;
    volatile int stop;
    int t;
};
struct ge_job {
    struct ge_shared* s;
    int tid;
};
static void* ge_worker(void* p) {
    struct ge_job* j = (struct ge_job*)p;
    struct ge_shared* s = j->s;
    const uint64_t n = s->n;
    double* w = s->w;
    for (uint64_t k = 0; k < n; ++k) {
        double pv = w[k * n + k];
        if (j->tid == 0) {
            if (s->pivots)
                s->pivots[k] = fabs(pv);
            if (fabs(pv) < s->floor)
                s->stop = (int)(k + 1);
        }
        pthread_barrier_wait(&s->bar);
        if (s->stop)
            return NULL;
        uint64_t first = k + 1 + (uint64_t)((j->tid - (int)((k + 1) % (uint64_t)s->t) + s->t) % s->t);
        for (uint64_t i = first; i < n; i += (uint64_t)s->t) {
            double mlt = (pv == 0.0) ? 0.0 : w[i * n + k] / pv;
            w[i * n + k] = mlt;
            if (mlt != 0.0)
                for (uint64_t jj = k + 1; jj < n; ++jj)
                    w[i * n + jj] -= mlt * w[k * n + jj];
        }
        pthread_barrier_wait(&s->bar);
    }
    return NULL;
}

/* ---------------------------------------------------------------- RNG ---- */

/* random_gen.cpp:13-18 */
static uint64_t splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* std::mt19937_64 (ISO C++ [rand.eng.mers] with the mt19937_64 parameters). */
#define MT_N 312
#define MT_M 156
static void mt_seed(rlo_rng* r, uint64_t v) {
    r->mt[0] = v;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

static void mt_twist(rlo_rng* r) {
    for (int i = 0; i < MT_N; ++i) {
        uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % MT_N] & 0x7FFFFFFFULL);
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    r->idx = 0;
}

uint64_t rlo_next_u64(rlo_rng* r) {
    if (r->idx >= MT_N)
        mt_twist(r);
    uint64_t z = r->mt[r->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* random_gen.cpp:22-31 */
void rlo_rng_init(rlo_rng* r, uint64_t seed, uint64_t sid) {
    uint64_t s = seed;
    uint64_t a = splitmix64(&s);
    s ^= sid * 0xda942042e4dd58b5ULL + 0x2545f4914f6cdd1dULL;
    uint64_t b = splitmix64(&s);
    mt_seed(r, a ^ (b << 1));
    for (int i = 0; i < 8; ++i)
        (void)rlo_next_u64(r);
    r->has_cached = 0;
    r->cached = 0.0;
}

/* random_gen.cpp:33-35 */
double rlo_uniform01(rlo_rng* r) { return (double)(rlo_next_u64(r) >> 11) * 0x1.0p-53; }
/* random_gen.cpp:37-39 */
double rlo_uniform_pm1(rlo_rng* r) { return 2.0 * rlo_uniform01(r) - 1.0; }

/* random_gen.cpp:41-53 (Box-Muller, cos first, sin cached) */
double rlo_gaussian(rlo_rng* r) {
    if (r->has_cached) {
        r->has_cached = 0;
        return r->cached;
    }
    double u1 = 1.0 - rlo_uniform01(r);
    double u2 = rlo_uniform01(r);
    double rr = sqrt(-2.0 * log(u1));
    double a = 2.0 * kPi * u2;
    r->cached = rr * sin(a);
    r->has_cached = 1;
    return rr * cos(a);
}

/* random_gen.cpp:55-57 */
double rlo_sign(rlo_rng* r) { return (rlo_next_u64(r) & 1u) ? 1.0 : -1.0; }

/* random_gen.cpp:59-70 (hi >= lo is the caller's responsibility here) */
int64_t rlo_uniform_int(rlo_rng* r, int64_t lo, int64_t hi) {
    uint64_t span = (uint64_t)(hi - lo) + 1;
    uint64_t limit = UINT64_MAX / span * span;
    uint64_t v;
    do {
        v = rlo_next_u64(r);
    } while (v >= limit);
    return lo + (int64_t)(v % span);
}

void rlo_raw_u64(uint64_t seed, uint64_t sid, uint64_t count, uint64_t* out) {
    rlo_rng r;
    rlo_rng_init(&r, seed, sid);
    for (uint64_t i = 0; i < count; ++i)
        out[i] = rlo_next_u64(&r);
}

/* random_gen.cpp:72-80 */
int rlo_gaussian_matrix(uint64_t m, uint64_t n, double mu, double sigma, uint64_t seed,
                        uint64_t sid, double* out) {
    if (!(sigma > 0.0))
        return 2;
    rlo_rng r;
    rlo_rng_init(&r, seed, sid);
    for (uint64_t i = 0; i < m * n; ++i)
        out[i] = mu + sigma * rlo_gaussian(&r);
    return 0;
}

/* random_gen.cpp:82-88 */
void rlo_uniform_matrix(uint64_t m, uint64_t n, uint64_t seed, uint64_t sid, double* out) {
    rlo_rng r;
    rlo_rng_init(&r, seed, sid);
    for (uint64_t i = 0; i < m * n; ++i)
        out[i] = rlo_uniform_pm1(&r);
}

/* random_gen.cpp:112-119 (CirculantSign first column) */
void rlo_sign_vector(uint64_t n, uint64_t seed, uint64_t sid, double* out) {
    rlo_rng r;
    rlo_rng_init(&r, seed, sid);
    for (uint64_t i = 0; i < n; ++i)
        out[i] = rlo_sign(&r);
}

/* NEW multiplier (no reference): u1 then u2, n signs each, from
 * one Rng on the stream — the same draw order as householder_sign's u, v
 * (random_gen.cpp:128-132), without its resampling (u^T u = n never vanishes). */
void rlo_householder_pair_signs(uint64_t n, uint64_t seed, uint64_t sid, double* u1, double* u2) {
    rlo_rng r;
    rlo_rng_init(&r, seed, sid);
    for (uint64_t i = 0; i < n; ++i)
        u1[i] = rlo_sign(&r);
    for (uint64_t i = 0; i < n; ++i)
        u2[i] = rlo_sign(&r);
}

/* NEW multiplier (no reference): for each column j, nnz distinct
 * rows by uniform_int(0, n-1) with duplicate rejection, then nnz signs. */
int rlo_sparse_pm1(uint64_t n, int nnz, uint64_t seed, uint64_t sid, int32_t* rows, double* signs) {
    if (nnz < 1 || (uint64_t)nnz > n)
        return 2;
    rlo_rng r;
    rlo_rng_init(&r, seed, sid);
    for (uint64_t j = 0; j < n; ++j) {
        int32_t* rj = rows + j * (uint64_t)nnz;
        for (int t = 0; t < nnz; ++t) {
            for (;;) {
                int32_t v = (int32_t)rlo_uniform_int(&r, 0, (int64_t)n - 1);
                int dup = 0;
                for (int s = 0; s < t; ++s)
                    dup |= (rj[s] == v);
                if (!dup) {
                    rj[t] = v;
                    break;
                }
            }
        }
        for (int t = 0; t < nnz; ++t)
            signs[j * (uint64_t)nnz + t] = rlo_sign(&r);
    }
    return 0;
}

/* ------------------------------------------------------------- dense ---- */

/* matrix.cpp:86-102: i-k-j, ascending k, skip zero a(i,k). */
void rlo_matmul(uint64_t m, uint64_t k, uint64_t n, const double* a, const double* b, double* c) {
    memset(c, 0, m * n * sizeof(double));
    if (g_threads > 1 && m >= 64) { /* rows are independent: bit-identical when threaded */
        par_rows(m, matmul_rows, &(struct mm_args){k, n, a, b, c});
        return;
    }
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t kk = 0; kk < k; ++kk) {
            double av = a[i * k + kk];
            if (av == 0.0)
                continue;
            const double* rr = b + kk * n;
            double* orow = c + i * n;
            for (uint64_t j = 0; j < n; ++j)
                orow[j] += av * rr[j];
        }
}

/* matrix.cpp:104-116 */
void rlo_matvec(uint64_t m, uint64_t n, const double* a, const double* x, double* y) {
    for (uint64_t i = 0; i < m; ++i) {
        double s = 0.0;
        const double* r = a + i * n;
        for (uint64_t j = 0; j < n; ++j)
            s += r[j] * x[j];
        y[i] = s;
    }
}

void rlo_transpose(uint64_t m, uint64_t n, const double* a, double* t) {
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < n; ++j)
            t[j * m + i] = a[i * n + j];
}

/* genp.cpp:11-41, packed: the multiplier l(i,k) is stored in w(i,k). */
int rlo_genp_factor(uint64_t n, double* w, double pivot_floor, double* pivots) {
    if (g_threads > 1 && n >= 512) {
        struct ge_shared s;
        memset(&s, 0, sizeof(s));
        s.n = n;
        s.w = w;
        s.floor = pivot_floor;
        s.pivots = pivots;
        s.t = g_threads;
        pthread_barrier_init(&s.bar, NULL, (unsigned)g_threads);
        pthread_t th[256];
        struct ge_job jobs[256];
        for (int i = 0; i < g_threads; ++i) {
            jobs[i].s = &s;
            jobs[i].tid = i;
            pthread_create(&th[i], NULL, ge_worker, &jobs[i]);
        }
        for (int i = 0; i < g_threads; ++i)
            pthread_join(th[i], NULL);
        pthread_barrier_destroy(&s.bar);
        return s.stop ? -s.stop : 0;
    }
    for (uint64_t k = 0; k < n; ++k) {
        double p = w[k * n + k];
        if (pivots)
            pivots[k] = fabs(p);
        if (fabs(p) < pivot_floor)
            return -(int)(k + 1);
        for (uint64_t i = k + 1; i < n; ++i) {
            double mlt = (p == 0.0) ? 0.0 : w[i * n + k] / p;
            w[i * n + k] = mlt;
            if (mlt != 0.0)
                for (uint64_t j = k + 1; j < n; ++j)
                    w[i * n + j] -= mlt * w[k * n + j];
        }
    }
    return 0;
}

/* genp.cpp:106-124 */
void rlo_genp_solve(uint64_t n, const double* lu, const double* b, double* y) {
    if (y != b)
        memcpy(y, b, n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) {
        double s = y[i];
        for (uint64_t j = 0; j < i; ++j)
            s -= lu[i * n + j] * y[j];
        y[i] = s;
    }
    for (uint64_t ii = n; ii-- > 0;) {
        double s = y[ii];
        for (uint64_t j = ii + 1; j < n; ++j)
            s -= lu[ii * n + j] * y[j];
        y[ii] = s / lu[ii * n + ii];
    }
}

/* genp.cpp:146-155 */
double rlo_relative_residual(uint64_t n, const double* a, const double* y, const double* b) {
    double num = 0.0, den = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (uint64_t j = 0; j < n; ++j)
            s += a[i * n + j] * y[j];
        double d = s - b[i];
        num += d * d;
        den += b[i] * b[i];
    }
    return sqrt(num) / sqrt(den);
}

/* -------------------------------------------------------- structured ---- */

static int is_pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }

/* structured.cpp:96-130: iterative radix-2, twiddles by repeated w *= wlen. */
int rlo_fft(uint64_t n, double* re, double* im, int inverse) {
    if (!is_pow2(n))
        return 6;
    for (uint64_t i = 1, j = 0; i < n; ++i) {
        uint64_t bit = n >> 1;
        for (; j & bit; bit >>= 1)
            j ^= bit;
        j ^= bit;
        if (i < j) {
            double t = re[i]; re[i] = re[j]; re[j] = t;
            t = im[i]; im[i] = im[j]; im[j] = t;
        }
    }
    const double sgn = inverse ? 1.0 : -1.0;
    for (uint64_t len = 2; len <= n; len <<= 1) {
        double ang = sgn * 2.0 * kPi / (double)len;
        double wlr = cos(ang), wli = sin(ang);
        for (uint64_t i = 0; i < n; i += len) {
            double wr = 1.0, wi = 0.0;
            for (uint64_t k = 0; k < len / 2; ++k) {
                double ur = re[i + k], ui = im[i + k];
                double xr = re[i + k + len / 2], xi = im[i + k + len / 2];
                double vr = xr * wr - xi * wi, vi = xr * wi + xi * wr;
                re[i + k] = ur + vr;
                im[i + k] = ui + vi;
                re[i + k + len / 2] = ur - vr;
                im[i + k + len / 2] = ui - vi;
                double nr = wr * wlr - wi * wli, ni = wr * wli + wi * wlr;
                wr = nr;
                wi = ni;
            }
        }
    }
    if (inverse)
        for (uint64_t i = 0; i < n; ++i) {
            re[i] /= (double)n;
            im[i] /= (double)n;
        }
    return 0;
}

static double vnorm2(uint64_t n, const double* v) {
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i)
        s += v[i] * v[i];
    return sqrt(s);
}

/* structured.cpp:132-154 (+ fft_convolve :23-35, take_real :39-50) */
int rlo_circ_mul(uint64_t n, const double* c, const double* x, double* y) {
    double scale = vnorm2(n, c) * vnorm2(n, x);
    uint64_t len = n;
    if (!is_pow2(n)) {
        len = 1;
        while (len < 2 * n - 1)
            len <<= 1;
    }
    double* buf = (double*)calloc(4 * len, sizeof(double));
    double *ar = buf, *ai = buf + len, *br = buf + 2 * len, *bi = buf + 3 * len;
    for (uint64_t i = 0; i < n; ++i) {
        ar[i] = c[i];
        br[i] = x[i];
    }
    rlo_fft(len, ar, ai, 0);
    rlo_fft(len, br, bi, 0);
    for (uint64_t i = 0; i < len; ++i) {
        double r = ar[i] * br[i] - ai[i] * bi[i];
        double im = ar[i] * bi[i] + ai[i] * br[i];
        ar[i] = r;
        ai[i] = im;
    }
    rlo_fft(len, ar, ai, 1);
    if (len != n)
        for (uint64_t i = 0; i < n; ++i)
            if (i + n < 2 * n - 1) {
                ar[i] += ar[i + n];
                ai[i] += ai[i + n];
            }
    double max_imag = 0.0;
    for (uint64_t i = 0; i < n; ++i)
        max_imag = fmax(max_imag, fabs(ai[i]));
    int st = 0;
    if (max_imag >= 1e-10 * fmax(scale, 1e-300))
        st = 11;
    for (uint64_t i = 0; i < n; ++i)
        y[i] = ar[i];
    free(buf);
    return st;
}

/* structured.cpp:178-189: spec * A, column by column. */
int rlo_circ_apply_left(uint64_t n, const double* c, uint64_t cols, const double* a, double* out) {
    double* col = (double*)malloc(2 * n * sizeof(double));
    int st = 0;
    for (uint64_t j = 0; j < cols && !st; ++j) {
        for (uint64_t i = 0; i < n; ++i)
            col[i] = a[i * cols + j];
        st = rlo_circ_mul(n, c, col, col + n);
        for (uint64_t i = 0; i < n; ++i)
            out[i * cols + j] = col[n + i];
    }
    free(col);
    return st;
}

/* genp.cpp:175-180: A*C = (C^T A^T)^T with transpose_spec (structured.cpp:85-94):
 * row i of the result = circ_mul(c^T, row i of A). */
int rlo_circ_apply_right(uint64_t n, const double* c, const double* a, double* out) {
    double* ct = (double*)malloc(n * sizeof(double));
    for (uint64_t k = 0; k < n; ++k)
        ct[k] = c[(n - k) % n];
    int st = 0;
    for (uint64_t i = 0; i < n && !st; ++i)
        st = rlo_circ_mul(n, ct, a + i * n, out + i * n);
    free(ct);
    return st;
}

/* structured.cpp:156-176: T x for the m x n Toeplitz (first column col, first row row), via
 * the circulant of power-of-two order len >= m + n - 1 whose first column is col followed by the
 * reversed strict first row in the wrap-around positions; y = the first m entries. */
int rlo_toeplitz_mul(uint64_t m, uint64_t n, const double* col, const double* row, const double* x, double* y) {
    uint64_t len = 1;
    while (len < m + n - 1)
        len <<= 1;
    double* buf = (double*)calloc(3 * len, sizeof(double));
    double *ce = buf, *xp = buf + len, *full = buf + 2 * len;
    for (uint64_t i = 0; i < m; ++i)
        ce[i] = col[i];
    for (uint64_t j = 1; j < n; ++j)
        ce[len - j] = row[j];
    for (uint64_t i = 0; i < n; ++i)
        xp[i] = x[i];
    int st = rlo_circ_mul(len, ce, xp, full);
    for (uint64_t i = 0; i < m; ++i)
        y[i] = full[i];
    free(buf);
    return st;
}

/* NEW: A*H1*H2, H_i = I - (2/n) u_i u_i^T, u_i in {+-1}^n:
 *   w1 = A u1, t1 = (2/n) w1, w2 = A u2 - t1 (u1^T u2), t2 = (2/n) w2,
 *   out(i,j) = (A(i,j) - t1(i) u1(j)) - t2(i) u2(j). */
void rlo_hh2_apply_right(uint64_t n, const double* u1, const double* u2, const double* a, double* out) {
    double s12 = 0.0;
    for (uint64_t j = 0; j < n; ++j)
        s12 += u1[j] * u2[j];
    const double c = 2.0 / (double)n;
    for (uint64_t i = 0; i < n; ++i) {
        const double* r = a + i * n;
        double w1 = 0.0, w2 = 0.0;
        for (uint64_t j = 0; j < n; ++j) {
            w1 += r[j] * u1[j];
            w2 += r[j] * u2[j];
        }
        double t1 = c * w1;
        double t2 = c * (w2 - t1 * s12);
        for (uint64_t j = 0; j < n; ++j)
            out[i * n + j] = (r[j] - t1 * u1[j]) - t2 * u2[j];
    }
}

/* NEW: x = H1 (H2 y). */
void rlo_hh2_apply_vec(uint64_t n, const double* u1, const double* u2, const double* y, double* x) {
    const double c = 2.0 / (double)n;
    double d2 = 0.0;
    for (uint64_t i = 0; i < n; ++i)
        d2 += u2[i] * y[i];
    double* v = (double*)malloc(n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i)
        v[i] = y[i] - (c * d2) * u2[i];
    double d1 = 0.0;
    for (uint64_t i = 0; i < n; ++i)
        d1 += u1[i] * v[i];
    for (uint64_t i = 0; i < n; ++i)
        x[i] = v[i] - (c * d1) * u1[i];
    free(v);
}

/* Pairwise sum of v[0..m): sum(v[0:h]) + sum(v[h:m]), h = ceil(m / 2) — the defined order
 * of the sparse product (for nnz = 4: (v0 + v1) + (v2 + v3)). */
static double rlo_pairwise(const double* v, int m) {
    if (m == 1)
        return v[0];
    int h = (m + 1) / 2;
    return rlo_pairwise(v, h) + rlo_pairwise(v + h, m - h);
}

/* NEW: (A S)(i,j) = sum_t s_jt A(i, r_jt), summed pairwise over t (rlo_pairwise). */
void rlo_sparse_apply_right(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                            const double* a, double* out) {
    double v[64];
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < n; ++j) {
            for (int t = 0; t < nnz; ++t)
                v[t] = signs[j * nnz + t] * a[i * n + (uint64_t)rows[j * nnz + t]];
            out[i * n + j] = rlo_pairwise(v, nnz);
        }
}

/* NEW: x = S y, accumulated in ascending (j, t) order per row. */
void rlo_sparse_apply_vec(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                          const double* y, double* x) {
    memset(x, 0, n * sizeof(double));
    for (uint64_t j = 0; j < n; ++j)
        for (int t = 0; t < nnz; ++t)
            x[rows[j * nnz + t]] += signs[j * nnz + t] * y[j];
}

/* ------------------------------------------------- randomized_genp ---- */

enum { TAG_GAUSSIAN = 0, TAG_UNIFORM = 1, TAG_TOEPLITZ = 2, TAG_CIRC_GAUSS = 3, TAG_CIRC_SIGN = 4,
       TAG_HH_SIGN = 5, TAG_HH_PAIR = 6, TAG_SPARSE = 7 };
enum { SIDE_LEFT = 0, SIDE_RIGHT = 1, SIDE_BOTH = 2 };

typedef struct {
    int tag;
    uint64_t n;
    double* dense; /* n x n for dense kinds */
    double* v1;    /* circulant first col / u1 / sparse signs */
    double* v2;    /* u2 */
    int32_t* rows; /* sparse */
} mult_t;

static int draw(mult_t* m, int tag, double mu, double sigma, uint64_t n, uint64_t seed, uint64_t sid) {
    memset(m, 0, sizeof(*m));
    m->tag = tag;
    m->n = n;
    switch (tag) {
    case TAG_GAUSSIAN:
        m->dense = (double*)malloc(n * n * sizeof(double));
        return rlo_gaussian_matrix(n, n, mu, sigma, seed, sid, m->dense);
    case TAG_UNIFORM:
        m->dense = (double*)malloc(n * n * sizeof(double));
        rlo_uniform_matrix(n, n, seed, sid, m->dense);
        return 0;
    case TAG_CIRC_SIGN:
        m->v1 = (double*)malloc(n * sizeof(double));
        rlo_sign_vector(n, seed, sid, m->v1);
        return 0;
    case TAG_CIRC_GAUSS: {
        m->v1 = (double*)malloc(n * sizeof(double));
        rlo_rng r;
        rlo_rng_init(&r, seed, sid);
        for (uint64_t i = 0; i < n; ++i)
            m->v1[i] = mu + sigma * rlo_gaussian(&r);
        return 0;
    }
    case TAG_TOEPLITZ: { /* random_gen.cpp:94-103: col[0], col[1..n-1], row[1..n-1]; row[0] = col[0] */
        m->v1 = (double*)malloc(n * sizeof(double));
        m->v2 = (double*)malloc(n * sizeof(double));
        rlo_rng r;
        rlo_rng_init(&r, seed, sid);
        m->v1[0] = mu + sigma * rlo_gaussian(&r);
        m->v2[0] = m->v1[0];
        for (uint64_t i = 1; i < n; ++i)
            m->v1[i] = mu + sigma * rlo_gaussian(&r);
        for (uint64_t j = 1; j < n; ++j)
            m->v2[j] = mu + sigma * rlo_gaussian(&r);
        return 0;
    }
    case TAG_HH_SIGN: { /* random_gen.cpp:125-143: I - u v^T / (u^T v), resampled while u^T v == 0 */
        double* u = (double*)malloc(2 * n * sizeof(double));
        double* v = u + n;
        rlo_rng r;
        rlo_rng_init(&r, seed, sid);
        for (int attempt = 0; attempt < 64; ++attempt) {
            for (uint64_t i = 0; i < n; ++i)
                u[i] = rlo_sign(&r);
            for (uint64_t i = 0; i < n; ++i)
                v[i] = rlo_sign(&r);
            double uv = 0.0;
            for (uint64_t i = 0; i < n; ++i)
                uv += u[i] * v[i];
            if (uv == 0.0)
                continue;
            m->dense = (double*)malloc(n * n * sizeof(double));
            for (uint64_t i = 0; i < n; ++i)
                for (uint64_t j = 0; j < n; ++j)
                    m->dense[i * n + j] = (i == j ? 1.0 : 0.0) - u[i] * v[j] / uv;
            free(u);
            return 0;
        }
        free(u);
        return 9; /* Degenerate */
    }
    case TAG_HH_PAIR:
        m->v1 = (double*)malloc(n * sizeof(double));
        m->v2 = (double*)malloc(n * sizeof(double));
        rlo_householder_pair_signs(n, seed, sid, m->v1, m->v2);
        return 0;
    case TAG_SPARSE:
        m->v1 = (double*)malloc(4 * n * sizeof(double));
        m->rows = (int32_t*)malloc(4 * n * sizeof(int32_t));
        return rlo_sparse_pm1(n, 4, seed, sid, m->rows, m->v1);
    default:
        return 2;
    }
}

static void mult_free(mult_t* m) {
    free(m->dense);
    free(m->v1);
    free(m->v2);
    free(m->rows);
}

/* Multiplier::apply(Matrix) (genp.cpp:164-166): M * A */
static int apply_left_mat(const mult_t* m, const double* a, double* out) {
    uint64_t n = m->n;
    switch (m->tag) {
    case TAG_GAUSSIAN:
    case TAG_UNIFORM:
    case TAG_HH_SIGN:
        rlo_matmul(n, n, n, m->dense, a, out);
        return 0;
    case TAG_CIRC_SIGN:
    case TAG_CIRC_GAUSS:
        return rlo_circ_apply_left(n, m->v1, n, a, out);
    case TAG_TOEPLITZ: { /* structured.cpp:178-189: column by column */
        double* col = (double*)malloc(2 * n * sizeof(double));
        int st = 0;
        for (uint64_t j = 0; j < n && !st; ++j) {
            for (uint64_t i = 0; i < n; ++i)
                col[i] = a[i * n + j];
            st = rlo_toeplitz_mul(n, n, m->v1, m->v2, col, col + n);
            for (uint64_t i = 0; i < n; ++i)
                out[i * n + j] = col[n + i];
        }
        free(col);
        return st;
    }
    default:
        return 2; /* new kinds: Right side only */
    }
}

/* Multiplier::apply_right (genp.cpp:175-180): A * M */
static int apply_right_mat(const mult_t* m, const double* a, double* out) {
    uint64_t n = m->n;
    switch (m->tag) {
    case TAG_GAUSSIAN:
    case TAG_UNIFORM:
    case TAG_HH_SIGN:
        rlo_matmul(n, n, n, a, m->dense, out);
        return 0;
    case TAG_CIRC_SIGN:
    case TAG_CIRC_GAUSS:
        return rlo_circ_apply_right(n, m->v1, a, out);
    case TAG_TOEPLITZ: { /* genp.cpp:175-180: row i of A T = toeplitz_mul(T^T, row i), T^T = toeplitz(row, col) */
        int st = 0;
        for (uint64_t i = 0; i < n && !st; ++i)
            st = rlo_toeplitz_mul(n, n, m->v2, m->v1, a + i * n, out + i * n);
        return st;
    }
    case TAG_HH_PAIR:
        rlo_hh2_apply_right(n, m->v1, m->v2, a, out);
        return 0;
    case TAG_SPARSE:
        rlo_sparse_apply_right(n, 4, m->rows, m->v1, a, out);
        return 0;
    default:
        return 2;
    }
}

/* Multiplier::apply(span) (genp.cpp:167-172): M * v */
static int apply_vec(const mult_t* m, const double* v, double* out) {
    uint64_t n = m->n;
    switch (m->tag) {
    case TAG_GAUSSIAN:
    case TAG_UNIFORM:
    case TAG_HH_SIGN:
        rlo_matvec(n, n, m->dense, v, out);
        return 0;
    case TAG_CIRC_SIGN:
    case TAG_CIRC_GAUSS:
        return rlo_circ_mul(n, m->v1, v, out);
    case TAG_TOEPLITZ:
        return rlo_toeplitz_mul(n, n, m->v1, m->v2, v, out);
    case TAG_HH_PAIR:
        rlo_hh2_apply_vec(n, m->v1, m->v2, v, out);
        return 0;
    case TAG_SPARSE:
        rlo_sparse_apply_vec(n, 4, m->rows, m->v1, v, out);
        return 0;
    default:
        return 2;
    }
}

static int all_finite(uint64_t n, const double* v) {
    for (uint64_t i = 0; i < n; ++i)
        if (!isfinite(v[i]))
            return 0;
    return 1;
}

/* genp.cpp:34-39: std::min / std::max fold starting from pivots[0] */
static void minmax(uint64_t n, const double* p, double* mn, double* mx) {
    double a = n ? p[0] : 0.0, b = a;
    for (uint64_t i = 0; i < n; ++i) {
        a = (p[i] < a) ? p[i] : a;
        b = (b < p[i]) ? p[i] : b;
    }
    *mn = a;
    *mx = b;
}

/* genp.cpp:207-291 */
int rlo_randomized_genp(uint64_t n, const double* a, const double* b, int tag, double mu,
                        double sigma, int side, int refine, uint64_t seed, uint64_t sid, double* y,
                        double* report, int* extra) {
    if (refine < 0 || refine > 2)
        return 2;
    if ((tag == TAG_HH_PAIR || tag == TAG_SPARSE) && side != SIDE_RIGHT)
        return 2;
    const uint64_t nn = n * n;
    double* w = (double*)malloc(nn * sizeof(double));
    double* sys = (double*)malloc(nn * sizeof(double));
    double* piv = (double*)malloc(n * sizeof(double));
    double* v = (double*)malloc(6 * n * sizeof(double));
    double *z = v, *rhs = v + n, *yy = v + 2 * n, *r = v + 3 * n, *t = v + 4 * n, *best_y = v + 5 * n;
    double rep[6] = {0, 0, 0, 0, 0, 0}, best_rep[6];
    int have_best = 0, status = 0, accepted = -1, drawn = 0, best_attempt = -1;

    /* raw-GENP contrast arm (genp.cpp:222-234); floor 0 never breaks down */
    memcpy(w, a, nn * sizeof(double));
    rlo_genp_factor(n, w, 0.0, piv);
    rlo_genp_solve(n, w, b, z);
    rep[1] = all_finite(n, z) ? rlo_relative_residual(n, a, z, b) : INFINITY;
    minmax(n, piv, &rep[4], &rep[5]);
    memcpy(best_rep, rep, sizeof(rep));

    for (int attempt = 0; attempt < 8; ++attempt) {
        uint64_t ds = sid + 7919ULL * (uint64_t)attempt;
        mult_t left, right;
        int use_left = (side == SIDE_LEFT || side == SIDE_BOTH);
        int use_right = (side == SIDE_RIGHT || side == SIDE_BOTH);
        ++drawn;
        /* Only the multipliers the side uses are materialised: the unused one is an
         * independent Rng with no side effect on the returned values. */
        int st = 0;
        memset(&left, 0, sizeof(left));
        memset(&right, 0, sizeof(right));
        if (use_left)
            st = draw(&left, tag, mu, sigma, n, seed, ds);
        if (!st && use_right)
            st = draw(&right, tag, mu, sigma, n, seed, ds ^ 0x5000000000000000ULL);
        if (st) {
            mult_free(&left);
            mult_free(&right);
            status = st;
            break;
        }
        memcpy(sys, a, nn * sizeof(double));
        if (use_left) {
            st = apply_left_mat(&left, sys, w);
            memcpy(sys, w, nn * sizeof(double));
        }
        if (!st && use_right) {
            st = apply_right_mat(&right, sys, w);
            memcpy(sys, w, nn * sizeof(double));
        }
        if (!st) {
            if (use_left)
                st = apply_vec(&left, b, rhs);
            else
                memcpy(rhs, b, n * sizeof(double));
        }
        if (st) { /* structured::Error (imaginary residue) propagates (not caught upstream) */
            mult_free(&left);
            mult_free(&right);
            status = st;
            break;
        }
        int fst = rlo_genp_factor(n, sys, 1e-300, piv);
        if (fst != 0) { /* PivotBreakdown (genp.cpp:285-288) */
            mult_free(&left);
            mult_free(&right);
            if (attempt + 1 >= 8 && !have_best) {
                status = 3;
                break;
            }
            continue;
        }
        rlo_genp_solve(n, sys, rhs, z);
        if (side == SIDE_LEFT)
            memcpy(yy, z, n * sizeof(double));
        else
            st = apply_vec(&right, z, yy);
        for (int s = 0; s < refine && !st; ++s) {
            rlo_matvec(n, n, a, yy, t);
            for (uint64_t i = 0; i < n; ++i)
                r[i] = b[i] - t[i];
            if (use_left) {
                st = apply_vec(&left, r, t);
                memcpy(r, t, n * sizeof(double));
            }
            rlo_genp_solve(n, sys, r, z);
            if (side == SIDE_LEFT)
                memcpy(t, z, n * sizeof(double));
            else
                st = st ? st : apply_vec(&right, z, t);
            for (uint64_t i = 0; i < n; ++i)
                yy[i] += t[i];
        }
        mult_free(&left);
        mult_free(&right);
        if (st) {
            status = st;
            break;
        }
        rep[0] = rlo_relative_residual(n, a, yy, b);
        minmax(n, piv, &rep[2], &rep[3]);
        if (rep[0] <= 1e-7) {
            memcpy(y, yy, n * sizeof(double));
            memcpy(report, rep, sizeof(rep));
            accepted = attempt;
            goto done;
        }
        if (!have_best || rep[0] < best_rep[0]) {
            memcpy(best_y, yy, n * sizeof(double));
            memcpy(best_rep, rep, sizeof(rep));
            have_best = 1;
            best_attempt = attempt;
        }
    }
    if (!status) {
        memcpy(y, best_y, n * sizeof(double));
        memcpy(report, best_rep, sizeof(rep));
        accepted = best_attempt;
    }
done:
    if (extra) {
        extra[0] = accepted;
        extra[1] = drawn;
    }
    free(w);
    free(sys);
    free(piv);
    free(v);
    return status;
}

/* One right-hand side of an attempt (genp.cpp:256-274) on the factored system: rhs (already
 * multiplied by the left multiplier when used), solve, y = right z, `refine` refinement steps.
 * v holds 4 scratch vectors of n. */
static int solve_column(uint64_t n, const double* a, const double* b, const double* sys, const mult_t* left,
                        const mult_t* right, int side, int refine, const double* rhs, double* yy, double* v) {
    const int use_left = (side == SIDE_LEFT || side == SIDE_BOTH);
    double *z = v, *r = v + n, *t = v + 2 * n;
    int st = 0;
    rlo_genp_solve(n, sys, rhs, z);
    if (side == SIDE_LEFT)
        memcpy(yy, z, n * sizeof(double));
    else
        st = apply_vec(right, z, yy);
    for (int s = 0; s < refine && !st; ++s) {
        rlo_matvec(n, n, a, yy, t);
        for (uint64_t i = 0; i < n; ++i)
            r[i] = b[i] - t[i];
        if (use_left) {
            st = apply_vec(left, r, t);
            memcpy(r, t, n * sizeof(double));
        }
        rlo_genp_solve(n, sys, r, z);
        if (side == SIDE_LEFT)
            memcpy(t, z, n * sizeof(double));
        else
            st = st ? st : apply_vec(right, z, t);
        for (uint64_t i = 0; i < n; ++i)
            yy[i] += t[i];
    }
    return st;
}

/* randomized_genp (genp.cpp:207-291) for nrhs right-hand sides at once: column j behaves as an
 * independent reference call randomized_genp(a, B[:, j], ...) on the same stream — the draws of
 * attempt a do not depend on b, so attempt a's multipliers and factorization are shared, and each
 * column keeps the first attempt whose residual is <= 1e-7 (else its best). Per column the
 * operations are exactly those of the single-RHS call (solve_column), so the bits agree with it.
 * B, Y row-major n x nrhs; reports: nrhs x 6 (rep[] of the single call); extras: nrhs x 2
 * (accepted attempt, attempts drawn). skip_raw: leave the contrast-arm fields at 0. */
int rlo_randomized_genp_multi(uint64_t n, uint64_t nrhs, const double* a, const double* B, int tag, double mu,
                              double sigma, int side, int refine, uint64_t seed, uint64_t sid, int skip_raw,
                              double* Y, double* reports, int* extras) {
    if (refine < 0 || refine > 2)
        return 2;
    if ((tag == TAG_HH_PAIR || tag == TAG_SPARSE) && side != SIDE_RIGHT)
        return 2;
    const uint64_t nn = n * n;
    double* w = (double*)malloc(nn * sizeof(double));
    double* sys = (double*)malloc(nn * sizeof(double));
    double* piv = (double*)malloc(n * sizeof(double));
    double* v = (double*)malloc((6 + 2 * nrhs) * n * sizeof(double));
    double *bj = v, *rhs = v + n, *yy = v + 2 * n, *scr = v + 3 * n; /* scr: 3 vectors */
    double* best_y = v + 6 * n;                                      /* nrhs x n */
    double* col_b = best_y + nrhs * n;                               /* nrhs x n */
    int* done = (int*)calloc(nrhs, sizeof(int));
    int* have = (int*)calloc(nrhs, sizeof(int));
    double raw[6] = {0, 0, 0, 0, 0, 0};
    int status = 0, drawn = 0;
    for (uint64_t j = 0; j < nrhs; ++j)
        for (uint64_t i = 0; i < n; ++i)
            col_b[j * n + i] = B[i * nrhs + j];
    if (!skip_raw) {
        memcpy(w, a, nn * sizeof(double));
        rlo_genp_factor(n, w, 0.0, piv);
        minmax(n, piv, &raw[4], &raw[5]);
    }
    for (uint64_t j = 0; j < nrhs; ++j) {
        double* rep = reports + 6 * j;
        memset(rep, 0, 6 * sizeof(double));
        if (!skip_raw) {
            rlo_genp_solve(n, w, col_b + j * n, yy);
            rep[1] = all_finite(n, yy) ? rlo_relative_residual(n, a, yy, col_b + j * n) : INFINITY;
            rep[4] = raw[4];
            rep[5] = raw[5];
        }
        extras[2 * j] = -1;
    }
    for (int attempt = 0; attempt < 8; ++attempt) {
        uint64_t ds = sid + 7919ULL * (uint64_t)attempt;
        mult_t left, right;
        int use_left = (side == SIDE_LEFT || side == SIDE_BOTH);
        int use_right = (side == SIDE_RIGHT || side == SIDE_BOTH);
        int pending = 0;
        for (uint64_t j = 0; j < nrhs; ++j)
            pending += !done[j];
        if (!pending)
            break;
        ++drawn;
        int st = 0;
        memset(&left, 0, sizeof(left));
        memset(&right, 0, sizeof(right));
        if (use_left)
            st = draw(&left, tag, mu, sigma, n, seed, ds);
        if (!st && use_right)
            st = draw(&right, tag, mu, sigma, n, seed, ds ^ 0x5000000000000000ULL);
        memcpy(sys, a, nn * sizeof(double));
        if (!st && use_left) {
            st = apply_left_mat(&left, sys, w);
            memcpy(sys, w, nn * sizeof(double));
        }
        if (!st && use_right) {
            st = apply_right_mat(&right, sys, w);
            memcpy(sys, w, nn * sizeof(double));
        }
        if (st) {
            mult_free(&left);
            mult_free(&right);
            status = st;
            break;
        }
        if (rlo_genp_factor(n, sys, 1e-300, piv) != 0) {
            mult_free(&left);
            mult_free(&right);
            continue;
        }
        double pmn, pmx;
        minmax(n, piv, &pmn, &pmx);
        for (uint64_t j = 0; j < nrhs && !st; ++j) {
            if (done[j])
                continue;
            memcpy(bj, col_b + j * n, n * sizeof(double));
            if (use_left)
                st = apply_vec(&left, bj, rhs);
            else
                memcpy(rhs, bj, n * sizeof(double));
            if (!st)
                st = solve_column(n, a, bj, sys, &left, &right, side, refine, rhs, yy, scr);
            if (st)
                break;
            double res = rlo_relative_residual(n, a, yy, bj);
            double* rep = reports + 6 * j;
            if (res <= 1e-7 || !have[j] || res < rep[0]) {
                memcpy(best_y + j * n, yy, n * sizeof(double));
                rep[0] = res;
                rep[2] = pmn;
                rep[3] = pmx;
                have[j] = 1;
                extras[2 * j] = attempt;
            }
            done[j] = res <= 1e-7;
        }
        mult_free(&left);
        mult_free(&right);
        if (st) {
            status = st;
            break;
        }
    }
    for (uint64_t j = 0; j < nrhs; ++j) {
        extras[2 * j + 1] = done[j] ? extras[2 * j] + 1 : drawn; /* the single call stops at acceptance */
        if (!have[j] && !status)
            status = 3;
        for (uint64_t i = 0; i < n; ++i)
            Y[i * nrhs + j] = best_y[j * n + i];
    }
    free(w);
    free(sys);
    free(piv);
    free(v);
    free(done);
    free(have);
    return status;
}

/* ------------------------------------------------------ range finder ---- */

/* dense_core.cpp:86-115 semantics: Householder QR, rank check
 * min|R_ii| > 1e-13 sigma_1(R), then positive diagonal. */
int rlo_qr_positive(uint64_t m, uint64_t n, const double* a, double* q, double* r) {
    if (m < n)
        return 2;
    double* w = (double*)malloc(m * n * sizeof(double));
    double* tau = (double*)calloc(n, sizeof(double));
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < n; ++j)
            w[j * m + i] = a[i * n + j];
    for (uint64_t k = 0; k < n; ++k) {
        double* x = w + k * m;
        double sn = 0.0;
        for (uint64_t i = k + 1; i < m; ++i)
            sn += x[i] * x[i];
        double alpha = x[k];
        if (sn == 0.0)
            continue;
        double beta = -copysign(sqrt(alpha * alpha + sn), alpha);
        tau[k] = (beta - alpha) / beta;
        double sc = 1.0 / (alpha - beta);
        for (uint64_t i = k + 1; i < m; ++i)
            x[i] *= sc;
        x[k] = beta;
        for (uint64_t j = k + 1; j < n; ++j) {
            double* yv = w + j * m;
            double s = yv[k];
            for (uint64_t i = k + 1; i < m; ++i)
                s += x[i] * yv[i];
            s *= tau[k];
            yv[k] -= s;
            for (uint64_t i = k + 1; i < m; ++i)
                yv[i] -= s * x[i];
        }
    }
    memset(r, 0, n * n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = i; j < n; ++j)
            r[i * n + j] = w[j * m + i];
    double* qc = (double*)calloc(m * n, sizeof(double));
    for (uint64_t j = 0; j < n; ++j)
        qc[j * m + j] = 1.0;
    for (uint64_t kk = n; kk-- > 0;) {
        const double* x = w + kk * m;
        for (uint64_t j = 0; j < n; ++j) {
            double* yv = qc + j * m;
            double s = yv[kk];
            for (uint64_t i = kk + 1; i < m; ++i)
                s += x[i] * yv[i];
            s *= tau[kk];
            yv[kk] -= s;
            for (uint64_t i = kk + 1; i < m; ++i)
                yv[i] -= s * x[i];
        }
    }
    double min_diag = INFINITY;
    for (uint64_t i = 0; i < n; ++i)
        min_diag = fmin(min_diag, fabs(r[i * n + i]));
    double* sg = (double*)malloc(n * sizeof(double));
    rlo_singular_values(n, n, r, sg);
    int st = (min_diag > 1e-13 * sg[0]) ? 0 : 4;
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < n; ++j)
            q[i * n + j] = qc[j * m + i];
    for (uint64_t i = 0; i < n; ++i)
        if (r[i * n + i] < 0.0) {
            for (uint64_t j = 0; j < n; ++j)
                r[i * n + j] = -r[i * n + j];
            for (uint64_t k = 0; k < m; ++k)
                q[k * n + i] = -q[k * n + i];
        }
    free(sg);
    free(qc);
    free(w);
    free(tau);
    return st;
}

static int cmp_desc(const void* x, const void* y) {
    double a = *(const double*)x, b = *(const double*)y;
    return (a < b) - (a > b);
}

/* Singular values by one-sided Jacobi (dense_core.cpp:117-136 computes them with
 * Eigen JacobiSVD/BDCSVD; Eigen's rounding is unpinned upstream). */
void rlo_singular_values(uint64_t m, uint64_t n, const double* a, double* sigma) {
    int tr = m < n;
    uint64_t mm = tr ? n : m, nn = tr ? m : n;
    double* w = (double*)malloc(mm * nn * sizeof(double));
    /* column-major working copy: column j contiguous */
    for (uint64_t i = 0; i < mm; ++i)
        for (uint64_t j = 0; j < nn; ++j)
            w[j * mm + i] = tr ? a[j * n + i] : a[i * n + j];
    for (int sweep = 0; sweep < 80; ++sweep) {
        double off = 0.0;
        for (uint64_t p = 0; p + 1 < nn; ++p)
            for (uint64_t q = p + 1; q < nn; ++q) {
                double* wp = w + p * mm;
                double* wq = w + q * mm;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (uint64_t i = 0; i < mm; ++i) {
                    al += wp[i] * wp[i];
                    be += wq[i] * wq[i];
                    ga += wp[i] * wq[i];
                }
                if (ga == 0.0)
                    continue;
                double rel = fabs(ga) / sqrt(al * be);
                if (!(rel > 1e-15))
                    continue;
                if (rel > off)
                    off = rel;
                double zeta = (be - al) / (2.0 * ga);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (uint64_t i = 0; i < mm; ++i) {
                    double x = wp[i], yv = wq[i];
                    wp[i] = c * x - s * yv;
                    wq[i] = s * x + c * yv;
                }
            }
        if (off <= 1e-15)
            break;
    }
    for (uint64_t j = 0; j < nn; ++j)
        sigma[j] = vnorm2(mm, w + j * mm);
    qsort(sigma, nn, sizeof(double), cmp_desc);
    free(w);
}

/* Thin SVD of the m x n (m >= n) matrix a by the one-sided Jacobi above: sigma (descending) and
 * the left singular vectors u (m x n row-major, column j for sigma_j; columns of zero singular
 * values are left zero).  dense::svd (dense_core.cpp:117-136) is Eigen's; its rounding and the
 * signs of the vectors are unpinned upstream, so the restatement fixes its own (the Jacobi
 * result). */
void rlo_svd_left(uint64_t m, uint64_t n, const double* a, double* sigma, double* u) {
    double* w = (double*)malloc(m * n * sizeof(double));
    for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < n; ++j)
            w[j * m + i] = a[i * n + j];
    for (int sweep = 0; sweep < 80; ++sweep) {
        double off = 0.0;
        for (uint64_t p = 0; p + 1 < n; ++p)
            for (uint64_t q = p + 1; q < n; ++q) {
                double *wp = w + p * m, *wq = w + q * m;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (uint64_t i = 0; i < m; ++i) {
                    al += wp[i] * wp[i];
                    be += wq[i] * wq[i];
                    ga += wp[i] * wq[i];
                }
                if (ga == 0.0)
                    continue;
                double rel = fabs(ga) / sqrt(al * be);
                if (!(rel > 1e-15))
                    continue;
                if (rel > off)
                    off = rel;
                double zeta = (be - al) / (2.0 * ga);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
                for (uint64_t i = 0; i < m; ++i) {
                    double x = wp[i], yv = wq[i];
                    wp[i] = c * x - sn * yv;
                    wq[i] = sn * x + c * yv;
                }
            }
        if (off <= 1e-15)
            break;
    }
    /* order by descending norm (stable: ties keep column order) */
    uint64_t* ord = (uint64_t*)malloc(n * sizeof(uint64_t));
    double* nr = (double*)malloc(n * sizeof(double));
    for (uint64_t j = 0; j < n; ++j) {
        ord[j] = j;
        nr[j] = vnorm2(m, w + j * m);
    }
    for (uint64_t i = 1; i < n; ++i)
        for (uint64_t k = i; k > 0 && nr[ord[k]] > nr[ord[k - 1]]; --k) {
            uint64_t tmp = ord[k];
            ord[k] = ord[k - 1];
            ord[k - 1] = tmp;
        }
    for (uint64_t j = 0; j < n; ++j) {
        const double sg = nr[ord[j]];
        sigma[j] = sg;
        for (uint64_t i = 0; i < m; ++i)
            u[i * n + j] = sg > 0.0 ? w[ord[j] * m + i] / sg : 0.0;
    }
    free(ord);
    free(nr);
    free(w);
}

/* lowrank::proto_lowrank (lowrank.cpp:108-177) for the Gaussian kind, RightSpace sketches
 * (approx_basis, lowrank.cpp:67-106: sketch = A^T G, G = gaussian_matrix(m, rho_plus)), with
 * the restated SVD above.  Outputs rho, basis (n x rho, ld rho_plus), approx (m x n), residual,
 * ok.  Returns 2 on a bad argument. */
int rlo_proto_lowrank(uint64_t m, uint64_t n, const double* a, uint64_t rho_plus, double tau, double tau_prime,
                      int tag, double mu, double sig_g, uint64_t seed, uint64_t sid, uint64_t* rho_out,
                      double* basis, double* approx, double* residual, int* ok) {
    /* lowrank.cpp:110-125: the tau checks, then ||A||; the zero matrix is accepted before
     * approx_basis validates rho_plus or the kind */
    if (!(tau_prime > 0.0 && tau_prime < 1.0) || (tau > 0.0 && !(tau < 1.0)))
        return 2;
    int all_zero = 1;
    for (uint64_t i = 0; i < m * n && all_zero; ++i)
        all_zero = a[i] == 0.0;
    if (all_zero) {
        *rho_out = 0;
        *residual = 0.0;
        *ok = 1;
        memset(approx, 0, m * n * sizeof(double));
        return 0;
    }
    if (tag != TAG_GAUSSIAN && tag != TAG_TOEPLITZ)
        return 2;
    if (rho_plus < 1 || rho_plus > (m < n ? m : n))
        return 2;
    const uint64_t k = m < n ? m : n;
    double* sg = (double*)malloc((k + rho_plus) * sizeof(double));
    double* ua = (double*)malloc(m * n * sizeof(double));
    /* ||A||_2 = sigma_1(A) */
    if (m >= n)
        rlo_svd_left(m, n, a, sg, ua);
    else {
        double* at = (double*)malloc(m * n * sizeof(double));
        rlo_transpose(m, n, a, at);
        rlo_svd_left(n, m, at, sg, ua);
        free(at);
    }
    const double norm_a = sg[0];
    *rho_out = 0;
    *residual = 0.0;
    *ok = 0;
    memset(approx, 0, m * n * sizeof(double));
    if (norm_a == 0.0) {
        *ok = 1;
        free(sg);
        free(ua);
        return 0;
    }
    double* g = (double*)malloc(m * rho_plus * sizeof(double));
    double* sk = (double*)malloc(n * rho_plus * sizeof(double));
    double* us = (double*)malloc(n * rho_plus * sizeof(double));
    double* ss = sg + k;
    double* at = (double*)malloc(m * n * sizeof(double));
    double* ab = (double*)malloc(m * rho_plus * sizeof(double));
    double* diff = (double*)malloc(m * n * sizeof(double));
    rlo_transpose(m, n, a, at);
    for (int attempt = 0; attempt <= 3; ++attempt) {
        const uint64_t ds = sid + 104729ULL * (uint64_t)attempt;
        if (tag == TAG_TOEPLITZ) { /* random_structured(kind, m, rho_plus): col[0..m-1], row[1..rho_plus-1] */
            rlo_rng r;
            rlo_rng_init(&r, seed, ds);
            double* gv = (double*)malloc((m + rho_plus) * sizeof(double));
            for (uint64_t i = 0; i < m + rho_plus - 1; ++i)
                gv[i] = mu + sig_g * rlo_gaussian(&r);
            for (uint64_t i = 0; i < m; ++i)
                for (uint64_t j = 0; j < rho_plus; ++j)
                    g[i * rho_plus + j] = i >= j ? gv[i - j] : gv[m - 1 + (j - i)];
            free(gv);
        } else {
            rlo_gaussian_matrix(m, rho_plus, mu, sig_g, seed, ds, g);
        }
        rlo_matmul(n, m, rho_plus, at, g, sk); /* A^T G */
        rlo_svd_left(n, rho_plus, sk, ss, us);
        double tau_eff = tau;
        if (tau_eff <= 0.0) { /* lowrank.cpp:132-147 */
            tau_eff = 1e-6;
            double best_gap = 1.0;
            for (uint64_t j = 1; j < rho_plus; ++j) {
                if (ss[j] >= 1e-3 * ss[0])
                    continue;
                double gap = ss[j] / fmax(ss[j - 1], 1e-300);
                if (gap < best_gap) {
                    best_gap = gap;
                    tau_eff = sqrt(fmax(ss[j] * ss[j - 1], 1e-300)) / norm_a;
                }
            }
        }
        uint64_t s = rho_plus;
        while (s > 0 && ss[s - 1] <= tau_eff * norm_a)
            --s;
        if (s == 0) { /* only the zero matrix passes (handled above) */
            *rho_out = 0;
            memset(approx, 0, m * n * sizeof(double));
            *residual = 1.0;
            *ok = 0;
            continue;
        }
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t j = 0; j < rho_plus; ++j)
                basis[i * rho_plus + j] = j < s ? us[i * rho_plus + j] : 0.0;
        /* project_onto_basis (lowrank.cpp:45-65), Right, orthonormal: (A T) T^T */
        for (uint64_t i = 0; i < m; ++i)
            for (uint64_t j = 0; j < s; ++j) {
                double acc = 0.0;
                for (uint64_t l = 0; l < n; ++l)
                    acc += a[i * n + l] * basis[l * rho_plus + j];
                ab[i * rho_plus + j] = acc;
            }
        for (uint64_t i = 0; i < m; ++i)
            for (uint64_t l = 0; l < n; ++l) {
                double acc = 0.0;
                for (uint64_t j = 0; j < s; ++j)
                    acc += ab[i * rho_plus + j] * basis[l * rho_plus + j];
                approx[i * n + l] = acc;
                diff[i * n + l] = a[i * n + l] - acc;
            }
        if (m >= n)
            rlo_svd_left(m, n, diff, sg, ua);
        else {
            rlo_transpose(m, n, diff, at);
            rlo_svd_left(n, m, at, sg, ua);
            rlo_transpose(m, n, a, at);
        }
        *rho_out = s;
        *residual = sg[0] / norm_a;
        *ok = *residual <= tau_prime;
        if (*ok)
            break;
    }
    free(g);
    free(sk);
    free(us);
    free(at);
    free(ab);
    free(diff);
    free(sg);
    free(ua);
    return 0;
}

/* dense_core.cpp:161-169 */
uint64_t rlo_numerical_rank(uint64_t l, const double* sigma, double tol) {
    if (l == 0 || sigma[0] == 0.0)
        return 0;
    uint64_t r = 0;
    for (uint64_t j = 0; j < l; ++j)
        if (sigma[j] >= tol * sigma[0])
            r = j + 1;
    return r;
}

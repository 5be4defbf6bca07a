// Host orchestration of genp::randomized_genp on device data
// (proj/src/genp.cpp:207-291): raw-GENP contrast arm, up to 8 multiplier draws on
// stream id + 7919*attempt (left multiplier from that stream, right from
// stream ^ 0x5000000000000000), system M A / A N / M A N, blocked GENP with pivot
// floor 1e-300, solves, y = N z, refinement, residual-gated acceptance at 1e-7,
// best-attempt fallback, PivotBreakdown rethrown only when the last attempt breaks
// down with no best.  Every FLOP runs on the GPU; the host only reads back the
// scalars the protocol branches on (breakdown flag, residuals, pivots).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <vector>

#include "rl_internal.cuh"

namespace rl {

// genp.cu
void genp_factor_blocked(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                         unsigned long long* d_breakdown, double* aux);
void genp_solve_blocked(uint64_t n, uint64_t nrhs, const double* lu, uint64_t lda, const double* aux,
                        double* b, uint64_t ldb);
void copy2d_dev(uint64_t rows, uint64_t cols, const double* src, uint64_t lds, double* dst, uint64_t ldd);
void axpy_dev(uint64_t count, double alpha, const double* x, double* y);
// structured.cu
void circulant_dense_dev(uint64_t n, const double* c, double* out);
void rank1_dense_dev(uint64_t n, const double* u, const double* v, double inv_uv, double* out);
void toeplitz_dense_dev(uint64_t n, const double* g, double* out);
void hh2_apply_right_dev(uint64_t n, const double* a, uint64_t lda, const double* u1, const double* u2,
                         double s12, double* out, uint64_t ldo, const double* s12p = nullptr);
void dot_pm1_dev(uint64_t n, const double* u1, const double* u2, double* d_out);
void hh2_apply_vec_dev(uint64_t n, uint64_t nrhs, const double* u1, const double* u2, const double* y,
                       double* x);
void sparse_apply_right_dev(uint64_t n, int nnz, const int32_t* rows, const double* signs,
                            const double* a, uint64_t lda, double* out, uint64_t ldo);
bool circ_fft_supported(uint64_t n);
void circ_apply_right_fft_dev(uint64_t m, uint64_t n, const double* c, const double* a, uint64_t lda, double* out,
                              uint64_t ldo);
uint64_t toeplitz_fft_len(uint64_t n);
void toeplitz_apply_right_fft_dev(uint64_t m, uint64_t n, const double* g, const double* a, uint64_t lda,
                                  double* out, uint64_t ldo);
void toeplitz_apply_vec_dev(uint64_t n, uint64_t nrhs, const double* g, const double* z, double* y);
void spec_transpose_dev(uint64_t n, bool toeplitz, const double* g, double* out);
void transpose_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda, double* t, uint64_t ldt);
struct SparseT {
    int32_t* row_ptr;
    int32_t* col_j;
    double* col_s;
};
SparseT sparse_transpose_dev(uint64_t n, int nnz, const int32_t* rows, const double* signs);
void sparse_apply_vec_dev(uint64_t n, uint64_t nrhs, const SparseT& s, const double* y, double* x);
void circ_apply_vec_dev(uint64_t n, uint64_t nrhs, const double* c, const double* z, double* y);
// genp_batched.cu
rl_status batched_circ64(uint64_t batch, const double* dA, const double* dB, int refine, int left, uint64_t seed,
                         const uint64_t* d_sids, double* dX, rl_precond_report* d_rep);

namespace {

constexpr int NB = 128;

} // namespace

void wait_upload(const double* dev) {
    PendingUpload& up = ctx().upload;
    if (up.dev != dev || up.npanels == 0)
        return;
    for (int p = 0; p < up.npanels; ++p) {
        RL_CUDA(cudaStreamWaitEvent(stream(), up.done[p], 0));
    }
    up = PendingUpload{};
}

namespace {

struct Mult {
    int tag = 0;
    uint64_t n = 0;
    double* dense = nullptr; // n x n (dense kinds; circulant densified for the left product)
    double* c = nullptr;     // circulant first column; Toeplitz col[0..n-1], row[1..n-1]
    double* u1 = nullptr;
    double* u2 = nullptr;
    double s12 = 0.0;
    int32_t* rows = nullptr;
    double* signs = nullptr;
    SparseT st{};
};

std::vector<double> to_host(const double* d, uint64_t count) {
    std::vector<double> h(count);
    RL_CUDA(cudaMemcpyAsync(h.data(), d, count * sizeof(double), cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
    return h;
}

// draw_multiplier (genp.cpp:183-203) on the GPU; `slot_dense` / `slot_vec` are scratch slots.
void draw(Mult& m, int tag, double mu, double sigma, uint64_t n, uint64_t seed, uint64_t sid,
          int slot_dense, int slot_vec, bool want_dense) {
    m.tag = tag;
    m.n = n;
    switch (tag) {
    case RL_GAUSSIAN:
        if (!(sigma > 0.0))
            fail(RL_INVALID_ARGUMENT, "gaussian_matrix: sigma must be positive");
        m.dense = ws<double>(slot_dense, n * n);
        rng_generate(seed, sid, Draw::Gaussian, n * n, mu, sigma, m.dense);
        break;
    case RL_UNIFORM_PM1:
        m.dense = ws<double>(slot_dense, n * n);
        rng_generate(seed, sid, Draw::UniformPm1, n * n, 0.0, 1.0, m.dense);
        break;
    case RL_CIRCULANT_SIGN:
    case RL_CIRCULANT_GAUSSIAN:
        m.c = ws<double>(slot_vec, n);
        if (tag == RL_CIRCULANT_SIGN)
            rng_generate(seed, sid, Draw::Sign, n, 0.0, 1.0, m.c);
        else
            rng_generate(seed, sid, Draw::Gaussian, n, mu, sigma, m.c);
        if (want_dense) {
            m.dense = ws<double>(slot_dense, n * n);
            circulant_dense_dev(n, m.c, m.dense);
        }
        break;
    case RL_TOEPLITZ_GAUSSIAN: {
        // random_structured (random_gen.cpp:94-103): n x n, col[0], col[1..n-1], row[1..n-1]
        // on one stream (row[0] = col[0]); on the Right through the FFT of its circulant
        // embedding when next_pow2(2n - 1) <= 8192 (as toeplitz_mul, structured.cpp:156-176),
        // densified otherwise
        double* g = ws<double>(slot_vec, 2 * n);
        rng_generate(seed, sid, Draw::Gaussian, 2 * n - 1, mu, sigma, g);
        m.c = g;
        if (want_dense) {
            m.dense = ws<double>(slot_dense, n * n);
            toeplitz_dense_dev(n, g, m.dense);
        }
        break;
    }
    case RL_HOUSEHOLDER_SIGN: {
        // random_gen.cpp:125-143: u, v signs; resample while u^T v == 0 (<= 64)
        double* uv = ws<double>(slot_vec, 2 * n * 64);
        rng_generate(seed, sid, Draw::Sign, 2 * n * 64, 0.0, 1.0, uv);
        std::vector<double> h = to_host(uv, 2 * n * 64);
        int found = -1;
        double dotv = 0.0;
        for (int r = 0; r < 64 && found < 0; ++r) {
            double s = 0.0;
            for (uint64_t i = 0; i < n; ++i)
                s += h[2 * n * r + i] * h[2 * n * r + n + i];
            if (s != 0.0) {
                found = r;
                dotv = s;
            }
        }
        if (found < 0)
            fail(RL_DEGENERATE, "householder_sign: u^T v == 0 after 64 resamples");
        m.dense = ws<double>(slot_dense, n * n);
        rank1_dense_dev(n, uv + 2 * n * found, uv + 2 * n * found + n, 1.0 / dotv, m.dense);
        break;
    }
    case RL_HOUSEHOLDER_PAIR: {
        double* u = ws<double>(slot_vec, 2 * n);
        rng_generate(seed, sid, Draw::Sign, 2 * n, 0.0, 1.0, u);
        m.u1 = u;
        m.u2 = u + n;
        std::vector<double> h = to_host(u, 2 * n);
        double s = 0.0;
        for (uint64_t i = 0; i < n; ++i)
            s += h[i] * h[n + i];
        m.s12 = s;
        break;
    }
    case RL_SPARSE_SIGN: {
        const int nnz = 4;
        if (n < 4)
            fail(RL_INVALID_ARGUMENT, "sparse multiplier needs n >= 4");
        char* base = ws<char>(slot_vec, n * nnz * 12 + 64);
        m.signs = reinterpret_cast<double*>(base);
        m.rows = reinterpret_cast<int32_t*>(base + n * nnz * 8);
        rng_sparse_sign(seed, sid, n, nnz, m.rows, m.signs);
        m.st = sparse_transpose_dev(n, nnz, m.rows, m.signs);
        break;
    }
    default:
        fail(RL_INVALID_ARGUMENT, "randomized_genp: unsupported multiplier kind");
    }
}

// out = sys * M  (out != sys)
void apply_right(const Mult& m, const double* sys, double* out) {
    const uint64_t n = m.n;
    PendingUpload& up = ctx().upload;
    if (up.dev == sys && up.npanels > 0 && m.dense && m.tag != RL_HOUSEHOLDER_PAIR && m.tag != RL_SPARSE_SIGN) {
        // sys is still arriving from the host: one GEMM per row panel, each after its copy
        uint64_t r0 = 0;
        for (int p = 0; p < up.npanels; ++p) {
            RL_CUDA(cudaStreamWaitEvent(stream(), up.done[p], 0));
            const uint64_t r1 = up.row_end[p];
            gemm(false, false, r1 - r0, n, n, 1.0, sys + r0 * n, n, m.dense, n, 0.0, out + r0 * n, n);
            r0 = r1;
        }
        up = PendingUpload{};
        return;
    }
    wait_upload(sys);
    switch (m.tag) {
    case RL_HOUSEHOLDER_PAIR:
        hh2_apply_right_dev(n, sys, n, m.u1, m.u2, m.s12, out, n);
        return;
    case RL_SPARSE_SIGN:
        sparse_apply_right_dev(n, 4, m.rows, m.signs, sys, n, out, n);
        return;
    case RL_CIRCULANT_SIGN:
    case RL_CIRCULANT_GAUSSIAN:
        if (!m.dense) {
            circ_apply_right_fft_dev(n, n, m.c, sys, n, out, n);
            return;
        }
        [[fallthrough]];
    case RL_TOEPLITZ_GAUSSIAN:
        if (!m.dense) {
            toeplitz_apply_right_fft_dev(n, n, m.c, sys, n, out, n);
            return;
        }
        [[fallthrough]];
    default:
        gemm(false, false, n, n, n, 1.0, sys, n, m.dense, n, 0.0, out, n);
    }
}

// out = M * sys (out != sys)
void apply_left(const Mult& m, const double* sys, uint64_t cols, double* out) {
    const uint64_t n = m.n;
    wait_upload(sys);
    if (!m.dense && (m.tag == RL_CIRCULANT_SIGN || m.tag == RL_CIRCULANT_GAUSSIAN || m.tag == RL_TOEPLITZ_GAUSSIAN)) {
        // M A = (A^T M^T)^T with M^T = transpose_spec(M) (structured.cpp:85-94): the Right-side
        // FFT product between two transposes
        const bool tp = m.tag == RL_TOEPLITZ_GAUSSIAN;
        double* t1 = ws<double>(WS_T1, n * cols);
        double* t2 = ws<double>(WS_T2, n * cols + 2 * n);
        double* spec = t2 + n * cols;
        transpose_dev(n, cols, sys, cols, t1, n);
        spec_transpose_dev(n, tp, m.c, spec);
        if (tp)
            toeplitz_apply_right_fft_dev(cols, n, spec, t1, n, t2, n);
        else
            circ_apply_right_fft_dev(cols, n, spec, t1, n, t2, n);
        transpose_dev(cols, n, t2, n, out, cols);
        return;
    }
    gemm(false, false, n, cols, n, 1.0, m.dense, n, sys, cols, 0.0, out, cols);
}

// out = M * v  (v n x nrhs)
void apply_vec(const Mult& m, const double* v, uint64_t nrhs, double* out) {
    const uint64_t n = m.n;
    switch (m.tag) {
    case RL_CIRCULANT_SIGN:
    case RL_CIRCULANT_GAUSSIAN:
        circ_apply_vec_dev(n, nrhs, m.c, v, out);
        return;
    case RL_TOEPLITZ_GAUSSIAN:
        if (!m.dense) {
            toeplitz_apply_vec_dev(n, nrhs, m.c, v, out);
            return;
        }
        gemm(false, false, n, nrhs, n, 1.0, m.dense, n, v, nrhs, 0.0, out, nrhs);
        return;
    case RL_HOUSEHOLDER_PAIR:
        hh2_apply_vec_dev(n, nrhs, m.u1, m.u2, v, out);
        return;
    case RL_SPARSE_SIGN:
        sparse_apply_vec_dev(n, nrhs, m.st, v, out);
        return;
    default:
        gemm(false, false, n, nrhs, n, 1.0, m.dense, n, v, nrhs, 0.0, out, nrhs);
    }
}

void minmax_fold(const std::vector<double>& p, double* mn, double* mx) {
    double a = p.empty() ? 0.0 : p[0], b = a;
    for (double v : p) {
        a = (v < a) ? v : a;
        b = (b < v) ? v : b;
    }
    *mn = a;
    *mx = b;
}

// max over columns of per-column relative residuals (nrhs = 1: the reference metric);
// non-finite columns count as +inf when check_finite.
double residual_max(uint64_t n, uint64_t nrhs, const double* a, const double* x, const double* b,
                    bool check_finite) {
    double* tmp = ws<double>(WS_RESID, n * nrhs + nrhs);
    double* out = tmp + n * nrhs;
    residuals_dev(n, nrhs, a, x, b, tmp, out);
    std::vector<double> r = to_host(out, nrhs);
    double worst = 0.0;
    std::vector<double> xs;
    if (check_finite)
        xs = to_host(x, n * nrhs);
    for (uint64_t j = 0; j < nrhs; ++j) {
        double v = r[j];
        if (check_finite)
            for (uint64_t i = 0; i < n; ++i)
                if (!std::isfinite(xs[i * nrhs + j])) {
                    v = std::numeric_limits<double>::infinity();
                    break;
                }
        if (j == 0 || v > worst || std::isnan(v))
            worst = v;
    }
    return worst;
}

} // namespace

void init_device(int device);

namespace {
// One persistent helper thread per calling thread: randomized_genp's raw-GENP contrast arm runs
// on it (its own stream, workspaces and LU streams) while the calling thread draws, applies
// and factors the attempts — the two factorizations are independent and both latency-bound at
// small n.
class AsyncWorker {
  public:
    AsyncWorker() : th_([this] { loop(); }) {}
    ~AsyncWorker() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    void submit(std::function<void()> f) {
        std::lock_guard<std::mutex> lk(m_);
        job_ = std::move(f);
        has_ = true;
        done_ = false;
        cv_.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return done_; });
    }

  private:
    void loop() {
        std::unique_lock<std::mutex> lk(m_);
        for (;;) {
            cv_.wait(lk, [&] { return stop_ || has_; });
            if (stop_ && !has_)
                return;
            std::function<void()> job = std::move(job_);
            has_ = false;
            lk.unlock();
            job();
            lk.lock();
            done_ = true;
            cv_.notify_all();
        }
    }
    std::mutex m_;
    std::condition_variable cv_;
    std::function<void()> job_;
    bool has_ = false, done_ = true, stop_ = false;
    std::thread th_;
};
AsyncWorker& contrast_worker() {
    static thread_local AsyncWorker w;
    return w;
}
// joins the helper on every exit path (the job references the caller's locals)
struct JoinGuard {
    AsyncWorker* w = nullptr;
    ~JoinGuard() {
        if (w)
            w->wait();
    }
};
} // namespace

// Per-column outcome of this thread's last randomized_genp_dev call (rl_last_column_reports).
thread_local std::vector<rl_column_report> g_last_cols;

rl_status randomized_genp_dev(uint64_t n, uint64_t nrhs, const double* A, const double* B, int tag,
                              double mu, double sigma, int side, int refine, uint64_t seed, uint64_t sid,
                              double* X, rl_precond_report* report, uint32_t flags) {
    g_last_cols.clear();
    if (refine < 0 || refine > 2)
        fail(RL_INVALID_ARGUMENT, "randomized_genp: refine must be in {0, 1, 2}");
    if (side < 0 || side > 2)
        fail(RL_INVALID_ARGUMENT, "randomized_genp: bad side");
    if ((tag == RL_HOUSEHOLDER_PAIR || tag == RL_SPARSE_SIGN) && side != RL_RIGHT)
        fail(RL_INVALID_ARGUMENT, "randomized_genp: the new multiplier kinds are applied on the right");
    const bool use_left = side == RL_LEFT || side == RL_BOTH;
    const bool use_right = side == RL_RIGHT || side == RL_BOTH;
    const uint64_t nblk = (n + NB - 1) / NB;
    double* sys = ws<double>(WS_SYS, n * n);
    double* tmp = ws<double>(WS_OUT, n * n);
    double* aux = ws<double>(WS_LU_AUX, nblk * 2 * NB * NB);
    double* vecs = ws<double>(WS_RHS, 4 * n * nrhs);
    double* Z = vecs;
    double* Y = Z + n * nrhs;
    double* R = Y + n * nrhs;
    double* D = R + n * nrhs;
    // One host read per attempt: pack = [per-column residuals | |pivots| | breakdown step]
    double* pack = ws<double>(WS_PACK, nrhs + n + 1);
    double* piv = pack + nrhs;
    unsigned long long* brk = reinterpret_cast<unsigned long long*>(piv + n);
    cudaStream_t st = stream();

    bool have_best = false;
    rl_status status = RL_OK;
    static const bool debug = std::getenv("RL_DEBUG") != nullptr;
    std::vector<char> col_accepted(nrhs, 0), col_have(nrhs, 0);
    std::vector<double> col_best(nrhs, 0.0), col_pmin(nrhs, 0.0), col_pmax(nrhs, 0.0);
    std::vector<int> col_attempt(nrhs, -1);
    // Speculative multipliers: for a dense right-only multiplier, attempt a+1's G is generated
    // on a side stream while attempt a solves (the wavefront solve leaves most SMs idle), and
    // attempt 0's G beside the contrast arm; a speculative draw is used if its attempt
    // happens, else discarded.  Attempts alternate between two multiplier slots so the
    // speculation never overwrites the live one.
    const bool speculate = use_right && !use_left && (tag == RL_GAUSSIAN || tag == RL_UNIFORM_PM1);
    struct Spec {
        cudaStream_t s = nullptr;
        cudaEvent_t start = nullptr, done = nullptr;
        int device = -1;
    };
    static thread_local Spec sp;
    if (speculate && sp.device != ctx().device) {
        RL_CUDA(cudaStreamCreateWithFlags(&sp.s, cudaStreamNonBlocking));
        RL_CUDA(cudaEventCreateWithFlags(&sp.start, cudaEventDisableTiming));
        RL_CUDA(cudaEventCreateWithFlags(&sp.done, cudaEventDisableTiming));
        sp.device = ctx().device;
    }
    int spec_attempt = -1; // attempt whose right multiplier the side stream has generated
    const int mult_slot[2] = {WS_MULT, WS_MULT2};
    auto spec_draw = [&](int a) { // attempt a's right multiplier on the side stream
        const uint64_t dn = (sid + 7919ULL * static_cast<uint64_t>(a)) ^ 0x5000000000000000ULL;
        double* next = ws<double>(mult_slot[a & 1], n * n);
        RL_CUDA(cudaEventRecord(sp.start, st));
        RL_CUDA(cudaStreamWaitEvent(sp.s, sp.start, 0));
        ctx().stream = sp.s;
        rng_generate(seed, dn, tag == RL_GAUSSIAN ? Draw::Gaussian : Draw::UniformPm1, n * n,
                     tag == RL_GAUSSIAN ? mu : 0.0, tag == RL_GAUSSIAN ? sigma : 1.0, next);
        ctx().stream = st;
        RL_CUDA(cudaEventRecord(sp.done, sp.s));
        spec_attempt = a;
    };

    rl_precond_report rep{};
    rep.attempt = -1;
    if (speculate && !(flags & 1u))
        spec_draw(0); // beside the contrast arm
    // raw-GENP contrast arm (genp.cpp:222-234) on the helper thread, concurrently with the attempts
    struct RawArm {
        double res = 0.0, pmin = 0.0, pmax = 0.0;
        std::exception_ptr err;
    } raw;
    JoinGuard join;
    static const bool raw_serial = std::getenv("RL_RAW_SERIAL") != nullptr; // dev comparison
    if (!(flags & 1u) && raw_serial) {
        wait_upload(A);
        copy2d_dev(n, n, A, n, sys, n);
        RL_CUDA(cudaMemsetAsync(brk, 0xff, 8, st));
        genp_factor_blocked(n, sys, n, 0.0, piv, brk, aux);
        copy2d_dev(n, nrhs, B, nrhs, Z, nrhs);
        genp_solve_blocked(n, nrhs, sys, n, aux, Z, nrhs);
        raw.res = residual_max(n, nrhs, A, Z, B, true);
        minmax_fold(to_host(piv, n), &raw.pmin, &raw.pmax);
    }
    if (!(flags & 1u) && !raw_serial) {
        wait_upload(A); // A and B are resident on this stream before the helper reads them
        static thread_local cudaEvent_t ev_in = nullptr;
        if (!ev_in)
            RL_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        RL_CUDA(cudaEventRecord(ev_in, st));
        const int dev = ctx().device;
        const cudaEvent_t e_in = ev_in;
        contrast_worker().submit([&raw, dev, e_in, n, nrhs, A, B, nblk] {
            try {
                init_device(dev);
                RL_CUDA(cudaStreamWaitEvent(stream(), e_in, 0));
                double* rs = ws<double>(WS_SYS, n * n);
                double* raux = ws<double>(WS_LU_AUX, nblk * 2 * NB * NB);
                double* rz = ws<double>(WS_RHS, n * nrhs);
                double* rpiv = ws<double>(WS_PACK, n + 1);
                unsigned long long* rbrk = reinterpret_cast<unsigned long long*>(rpiv + n);
                copy2d_dev(n, n, A, n, rs, n);
                RL_CUDA(cudaMemsetAsync(rbrk, 0xff, 8, stream()));
                genp_factor_blocked(n, rs, n, 0.0, rpiv, rbrk, raux);
                copy2d_dev(n, nrhs, B, nrhs, rz, nrhs);
                genp_solve_blocked(n, nrhs, rs, n, raux, rz, nrhs);
                raw.res = residual_max(n, nrhs, A, rz, B, true);
                minmax_fold(to_host(rpiv, n), &raw.pmin, &raw.pmax);
            } catch (...) {
                raw.err = std::current_exception();
            }
        });
        join.w = &contrast_worker();
    }
    rl_precond_report best = rep;
    for (int attempt = 0; attempt < 8; ++attempt) {
        const uint64_t ds = sid + 7919ULL * static_cast<uint64_t>(attempt);
        rep.attempts_drawn = attempt + 1;
        Mult left, right;
        if (use_left) // circulant / Toeplitz multipliers stay matrix-free when the FFT path takes them
            draw(left, tag, mu, sigma, n, seed, ds, WS_MULT, WS_LVEC,
                 !(((tag == RL_CIRCULANT_SIGN || tag == RL_CIRCULANT_GAUSSIAN) && circ_fft_supported(n)) ||
                   (tag == RL_TOEPLITZ_GAUSSIAN && toeplitz_fft_len(n) != 0)));
        if (use_right) {
            if (spec_attempt == attempt) {
                right.tag = tag;
                right.n = n;
                right.dense = ws<double>(mult_slot[attempt & 1], n * n);
                RL_CUDA(cudaStreamWaitEvent(st, sp.done, 0));
                spec_attempt = -1;
            } else {
                // circulant multipliers of power-of-two n <= 8192 are applied on the right through
                // the FFT (matrix-free); everything else is densified
                const bool fft = ((tag == RL_CIRCULANT_SIGN || tag == RL_CIRCULANT_GAUSSIAN) && circ_fft_supported(n)) ||
                                 (tag == RL_TOEPLITZ_GAUSSIAN && toeplitz_fft_len(n) != 0);
                draw(right, tag, mu, sigma, n, seed, ds ^ 0x5000000000000000ULL,
                     use_left ? WS_RF1 : (speculate ? mult_slot[attempt & 1] : WS_MULT), WS_RF2, !fft);
            }
        }
        const double* src = A;
        if (use_left) {
            apply_left(left, src, n, tmp);
            std::swap(sys, tmp);
            src = sys;
        }
        if (use_right) {
            apply_right(right, src, tmp);
            std::swap(sys, tmp);
        }
        if (!use_left && !use_right) {
            wait_upload(A);
            copy2d_dev(n, n, A, n, sys, n);
        }
        wait_upload(A); // (no-op once the first product consumed the upload)
        if (use_left)
            apply_vec(left, B, nrhs, Z);
        else
            copy2d_dev(n, nrhs, B, nrhs, Z, nrhs);
        RL_CUDA(cudaMemsetAsync(brk, 0xff, 8, st));
        genp_factor_blocked(n, sys, n, 1e-300, piv, brk, aux);
        // The breakdown flag is read with the residuals (one host synchronisation per attempt):
        // the solves run on a broken factorization too and their results are then discarded.
        if (speculate && attempt + 1 < 8) // next attempt's G beside this attempt's solves
            spec_draw(attempt + 1);
        genp_solve_blocked(n, nrhs, sys, n, aux, Z, nrhs);
        if (use_right)
            apply_vec(right, Z, nrhs, Y);
        else
            copy2d_dev(n, nrhs, Z, nrhs, Y, nrhs);
        for (int s = 0; s < refine; ++s) {
            copy2d_dev(n, nrhs, B, nrhs, R, nrhs);
            gemm(false, false, n, nrhs, n, -1.0, A, n, Y, nrhs, 1.0, R, nrhs); // r = b - A y
            if (use_left) {
                apply_vec(left, R, nrhs, D);
                copy2d_dev(n, nrhs, D, nrhs, R, nrhs);
            }
            genp_solve_blocked(n, nrhs, sys, n, aux, R, nrhs);
            if (use_right)
                apply_vec(right, R, nrhs, D);
            else
                copy2d_dev(n, nrhs, R, nrhs, D, nrhs);
            axpy_dev(n * nrhs, 1.0, D, Y); // y += d
        }
        // Acceptance per right-hand side (genp.cpp:275-282): nrhs columns behave as nrhs
        // independent reference calls sharing the stream — a column keeps the first attempt
        // whose residual is <= 1e-7, else its best attempt.
        {
            double* tmpr = ws<double>(WS_RESID, n * nrhs);
            residuals_dev(n, nrhs, A, Y, B, tmpr, pack);
        }
        const std::vector<double> hp = to_host(pack, nrhs + n + 1);
        long long hb = -1;
        std::memcpy(&hb, &hp[nrhs + n], 8);
        if (hb >= 0) { // PivotBreakdown (genp.cpp:285-288)
            if (attempt + 1 >= 8 && !have_best) {
                status = RL_PIVOT_BREAKDOWN;
                set_error("genp_factor: pivot below floor at step " + std::to_string(hb));
            }
            continue;
        }
        const std::vector<double> res(hp.begin(), hp.begin() + nrhs);
        double pmn = 0.0, pmx = 0.0;
        minmax_fold(std::vector<double>(hp.begin() + nrhs, hp.begin() + nrhs + n), &pmn, &pmx);
        if (debug)
            for (uint64_t j = 0; j < nrhs; ++j)
                std::fprintf(stderr, "[rl] attempt %d column %llu residual %.3e\n", attempt,
                             static_cast<unsigned long long>(j), res[j]);
        bool all_done = true;
        for (uint64_t j = 0; j < nrhs; ++j) {
            if (col_accepted[j])
                continue;
            const bool acc = res[j] <= 1e-7;
            if (acc || !col_have[j] || res[j] < col_best[j]) {
                copy2d_dev(n, 1, Y + j, nrhs, X + j, nrhs);
                col_best[j] = res[j];
                col_have[j] = true;
                col_attempt[j] = attempt;
                col_pmin[j] = pmn;
                col_pmax[j] = pmx;
            }
            col_accepted[j] = acc;
            all_done = all_done && acc;
        }
        have_best = true;
        if (all_done)
            break;
    }
    if (spec_attempt >= 0) // an unused speculative draw still owns its slot and the RNG workspace
        RL_CUDA(cudaStreamWaitEvent(st, sp.done, 0));
    if (have_best) {
        g_last_cols.resize(nrhs);
        for (uint64_t j = 0; j < nrhs; ++j)
            g_last_cols[j] = rl_column_report{col_best[j], col_pmin[j], col_pmax[j], col_attempt[j],
                                              col_accepted[j] ? col_attempt[j] + 1 : rep.attempts_drawn};
        // report: worst column; its attempt and pivots (nrhs = 1: exactly the reference's report)
        uint64_t w = 0;
        for (uint64_t j = 1; j < nrhs; ++j)
            if (col_best[j] > col_best[w] || std::isnan(col_best[j]))
                w = j;
        rep.residual = col_best[w];
        rep.attempt = col_attempt[w];
        rep.pivot_min = col_pmin[w];
        rep.pivot_max = col_pmax[w];
        best = rep;
        status = RL_OK;
    }
    if (join.w) {
        join.w->wait();
        join.w = nullptr;
        if (raw.err)
            std::rethrow_exception(raw.err);
    }
    if (!(flags & 1u)) { // the contrast arm's report fields
        best.raw_residual = raw.res;
        best.raw_pivot_min = raw.pmin;
        best.raw_pivot_max = raw.pmax;
    }
    if (status == RL_OK && report) {
        best.attempts_drawn = rep.attempts_drawn;
        *report = best;
    }
    RL_CUDA(cudaStreamSynchronize(st));
    return status;
}

const std::vector<rl_column_report>& last_column_reports() { return g_last_cols; }

const char* last_error();

namespace {
// Host worker pool for the general batched path.  The reference runs table1_genp's trials on
// parallel_trials worker threads (bench.cpp:63-93); here each worker keeps its own per-thread
// context (stream, workspaces, the LU's lookahead streams), so the systems' latency-bound
// launches overlap on the GPU.  Persistent (the per-thread workspaces are allocated once);
// one batched call at a time uses it.
class SystemPool {
  public:
    static SystemPool& get() {
        static SystemPool p;
        return p;
    }
    int size() const { return static_cast<int>(threads_.size()); }
    // job(worker) on every worker; returns when all are done
    void run(int device, const std::function<void(int)>& job) {
        std::lock_guard<std::mutex> one(run_m_);
        std::unique_lock<std::mutex> lk(m_);
        job_ = &job;
        device_ = device;
        pending_ = size();
        ++gen_;
        cv_.notify_all();
        done_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    ~SystemPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_)
            t.join();
    }

  private:
    SystemPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        int n = static_cast<int>(std::max(1u, std::min(8u, hw ? hw : 1u)));
        if (const char* e = std::getenv("RL_BATCH_THREADS")) // RL_BATCH_THREADS=1: the serial order
            n = std::max(1, std::min(64, std::atoi(e)));
        for (int i = 0; i < n; ++i)
            threads_.emplace_back([this, i] { loop(i); });
    }
    void loop(int id) {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(m_);
        for (;;) {
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_)
                return;
            seen = gen_;
            const std::function<void(int)>* job = job_;
            const int dev = device_;
            lk.unlock();
            try {
                init_device(dev);
                (*job)(id);
            } catch (...) {
            }
            lk.lock();
            if (--pending_ == 0)
                done_.notify_all();
        }
    }
    std::vector<std::thread> threads_;
    std::mutex m_, run_m_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    int device_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};
} // namespace

rl_status randomized_genp_batched_dev(uint64_t batch, uint64_t n, const double* dA, const double* dB,
                                      int tag, double mu, double sigma, int side, int refine,
                                      uint64_t seed, const uint64_t* d_sids, double* dX,
                                      rl_precond_report* d_rep) {
    if (refine < 0 || refine > 2)
        fail(RL_INVALID_ARGUMENT, "randomized_genp: refine must be in {0, 1, 2}");
    if (tag == RL_CIRCULANT_SIGN && (side == RL_RIGHT || side == RL_LEFT) && n == 64)
        return batched_circ64(batch, dA, dB, refine, side == RL_LEFT ? 1 : 0, seed, d_sids, dX, d_rep);
    // general kinds / sizes: the blocked single-system path, systems spread over the host worker
    // pool (each worker's own stream and workspaces; the result of a system does not depend on
    // which worker ran it)
    std::vector<uint64_t> sids(batch);
    RL_CUDA(cudaMemcpyAsync(sids.data(), d_sids, batch * 8, cudaMemcpyDeviceToHost, stream()));
    RL_CUDA(cudaStreamSynchronize(stream())); // also: the inputs are resident before the workers read them
    std::vector<rl_precond_report> reps(batch);
    std::vector<rl_status> st(batch, RL_OK);
    std::vector<std::string> msg(batch);
    std::atomic<uint64_t> next{0};
    SystemPool::get().run(ctx().device, [&](int) {
        for (uint64_t t = next++; t < batch; t = next++) {
            try {
                st[t] = randomized_genp_dev(n, 1, dA + t * n * n, dB + t * n, tag, mu, sigma, side, refine, seed,
                                            sids[t], dX + t * n, &reps[t], 0);
                if (st[t] != RL_OK)
                    msg[t] = last_error();
            } catch (const Failure& f) {
                st[t] = f.code;
                msg[t] = f.msg;
            }
        }
    });
    for (uint64_t t = 0; t < batch; ++t) // the first failing system, as the serial loop reported
        if (st[t] != RL_OK) {
            set_error(msg[t]);
            return st[t];
        }
    RL_CUDA(cudaMemcpyAsync(d_rep, reps.data(), batch * sizeof(rl_precond_report), cudaMemcpyHostToDevice,
                            stream()));
    RL_CUDA(cudaStreamSynchronize(stream()));
    return RL_OK;
}

} // namespace rl

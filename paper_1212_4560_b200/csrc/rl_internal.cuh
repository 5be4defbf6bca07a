// Internal runtime of librl_b200: per-thread stream/workspace, error plumbing,
// launch accounting.  Not part of the C-ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "rl_b200.h"

namespace rl {

// Thrown internally and converted to rl_status at the C-ABI boundary.
struct Failure {
    rl_status code;
    std::string msg;
};

[[noreturn]] void fail(rl_status code, const std::string& msg);
void set_error(const std::string& msg);

#define RL_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t err__ = (call);                                                        \
        if (err__ != cudaSuccess)                                                          \
            ::rl::fail(RL_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(err__)); \
    } while (0)

#define RL_LAUNCHED()                                                                      \
    do {                                                                                   \
        ::rl::count_launch();                                                              \
        cudaError_t err__ = cudaGetLastError();                                            \
        if (err__ != cudaSuccess)                                                          \
            ::rl::fail(RL_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(err__)); \
    } while (0)

void count_launch();

// Grow-only device scratch buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    void* get(size_t need);
    ~DevBuf();
};

// A host -> device upload of a row-major matrix still in flight, in row panels (the
// host-pointer entry points overlap the upload of A with the first A * G product).
struct PendingUpload {
    const double* dev = nullptr; // device copy being filled
    int npanels = 0;
    uint64_t row_end[8] = {};    // panel p covers rows [row_end[p-1], row_end[p])
    cudaEvent_t done[8] = {};    // recorded on the copy stream after panel p
};

struct Ctx {
    int device = -1;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr; // what rl_dev_* calls launch on
    DevBuf ws[64];                 // named scratch slots (see WS_* below)
    uint64_t launches = 0;
    int sms = 148;
    PendingUpload upload;          // set only inside a host-pointer call
};

// Make the current stream wait for every panel of a pending upload of `dev` (no-op when
// none is pending); the upload is then complete as far as this stream is concerned.
void wait_upload(const double* dev);

enum WsSlot {
    WS_IN_A = 0, WS_IN_B, WS_OUT, WS_MULT, WS_SYS, WS_RHS, WS_TMP1, WS_TMP2, WS_RNG,
    WS_RNG2, WS_SMALL, WS_LU_AUX, WS_BATCH, WS_RF1, WS_RF2, WS_RF3, WS_LVEC, WS_RESID, WS_RF4,
    WS_RF5, WS_RF6, WS_H0, WS_H1, WS_H2, WS_H3, WS_WAVE, WS_MULT2, WS_RNG3, WS_RNG4, WS_SPLAN, WS_T1, WS_T2,
    WS_FFT_GEN, WS_FFT_C, WS_FFT_X, WS_FFT_TMP, WS_FFT_OUT, WS_FFT_FLAG, WS_FLAGS, WS_RF3B, WS_RF5B,
    WS_ES0, WS_ES1, WS_ES2, WS_ES3, WS_ES4, WS_ES5, WS_PACK, WS_RF7, WS_RF8
};

Ctx& ctx();          // thread-local context (initialises the device on first use)
void ensure_device(); // throws RL_NO_DEVICE when no GPU is present
inline cudaStream_t stream() { return ctx().stream; }

template <typename T>
T* ws(int slot, size_t count) {
    return static_cast<T*>(ctx().ws[slot].get(count * sizeof(T)));
}

inline unsigned cdiv(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// ------------------------------------------------------------------ RNG ----
// mt19937_64 stream generation (rng_mt64.cu).
enum class Draw : int { RawU64 = 0, Uniform01 = 1, UniformPm1 = 2, Gaussian = 3, Sign = 4 };
// Generate `count` transformed draws of stream (seed, sid) into d_out (double, or
// uint64 for RawU64).  Gaussian uses mu + sigma * g with the reference's Box-Muller
// pairing; `count` Gaussians consume `count` (rounded up to even) engine outputs.
void rng_generate(uint64_t seed, uint64_t sid, Draw kind, uint64_t count, double mu, double sigma,
                  void* d_out);
// Same for outputs [offset, offset + count) (offset even for Gaussians).
void rng_generate_at(uint64_t seed, uint64_t sid, Draw kind, uint64_t offset, uint64_t count, double mu,
                     double sigma, void* d_out);
// Box-Muller of consecutive raw pairs (random_gen.cpp:46-52).
void box_muller_pairs_dev(const uint64_t* d_raw, uint64_t npairs, double* d_out);
void box_muller_hash_dev(uint64_t seed, uint64_t npairs, uint64_t chunk, unsigned long long* d_hashes);
// One stream per element of d_sids (seed shared, stream id ^ xor_mask + add): n sign
// draws each into d_out[t*n ...]  (batched circulant first columns).
void rng_sign_vectors_batched(uint64_t seed, const uint64_t* d_sids, uint64_t add, uint64_t xor_mask,
                              uint64_t batch, uint64_t n, double* d_out);
// Sparse +-1 multiplier (serial consumption of a parallel raw pool).
void rng_sparse_sign(uint64_t seed, uint64_t sid, uint64_t n, int nnz, int32_t* d_rows,
                     double* d_signs);

// ----------------------------------------------------------------- GEMM ----
// Row-major C = alpha op(A) op(B) + beta C on the current stream.
void gemm(bool ta, bool tb, uint64_t m, uint64_t n, uint64_t k, double alpha, const double* a,
          uint64_t lda, const double* b, uint64_t ldb, double beta, double* c, uint64_t ldc);

// ----------------------------------------------------------------- GENP ----
struct GenpAux {
    double* pivots;      // n |pivots|
    int64_t* breakdown;  // device int64: first step with |p| < floor, or -1
};
// Blocked in-place GENP on device (packed LU), pivots into aux.
void genp_factor_dev(uint64_t n, double* a, uint64_t lda, double pivot_floor, double* d_pivots,
                     int64_t* d_breakdown);
// Multi-RHS solve with the packed LU: B (n x nrhs, ld = ldb) overwritten by X.
// rows x cols row-major f64 (ld doubles) as a TMA tensor map: box box_rows x 16 doubles, 128-byte
// swizzle, zero fill past the edges (dgemm_dmma.cu); false when the driver entry is missing or
// the layout is not TMA-addressable (base / ld not 16-byte aligned)
bool make_tmap(CUtensorMap* tm, const double* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows);

void genp_solve_dev(uint64_t n, uint64_t nrhs, const double* lu, uint64_t lda, double* b,
                    uint64_t ldb);

// ------------------------------------------------------------ misc kernels --
void transpose_dev(uint64_t m, uint64_t n, const double* a, uint64_t lda, double* t, uint64_t ldt);
// residual norms per column: r_j = ||A x_j - b_j|| / ||b_j|| (genp.cpp:146-155) into d_out[nrhs]
void residuals_dev(uint64_t n, uint64_t nrhs, const double* a, const double* x, const double* b,
                   double* d_tmp, double* d_out);

} // namespace rl

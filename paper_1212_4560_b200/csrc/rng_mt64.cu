// K1: the reference's random streams on the GPU, bit-exact.
//
// Reference: rnd::Rng (proj/src/random_gen.cpp:13-70) = splitmix64-mixed seed ->
// std::mt19937_64 -> discard(8), one SEQUENTIAL stream per generated matrix
// (gaussian_matrix random_gen.cpp:72-80 fills row-major entries in draw order).
//
// B200 design: a stream of N outputs is cut into chunks of J = 2^15 engine steps,
// one warp per chunk.  The engine state at the start of chunk c is
//     s_{8 + cJ} = p(T) s_0,   p = x^(8 + cJ) mod phi
// (phi = characteristic polynomial of the mt19937_64 transition, table built at
// build time by mt64_jumpgen.cpp).  Applying p is a GF(2) correlation of the
// polynomial's set bits with the word sequence (k_jump).  Two levels keep the
// table small: level-1 windows every 2^21 steps from s_0, level-2 windows every
// 2^15 steps from each level-1 window.  The warp then twists its 312-word window
// in shared memory and tempers / transforms 312 outputs per twist.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "glibc_math.cuh"
#include <algorithm>

#include "rl_internal.cuh"

namespace rl {

namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL,
                   kMatA = 0xB5026F5AA96619E9ULL;
constexpr int kLog2J = 15;
constexpr uint64_t kJ = 1ULL << kLog2J;
constexpr int kSeqWords = 19937 + kN - 1; // words x_t .. x_{t+20247} feed a jump
constexpr uint64_t kSmallMax = 1ULL << 12; // streams this short run on one warp (beyond ~3K draws the
                                            // chunked path's ~0.1 ms fixed cost wins)

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// random_gen.cpp:22-29: the engine seed of stream (seed, sid)
__host__ __device__ __forceinline__ uint64_t engine_seed(uint64_t seed, uint64_t sid) {
    uint64_t s = seed;
    uint64_t a = splitmix64(s);
    s ^= sid * 0xda942042e4dd58b5ULL + 0x2545f4914f6cdd1dULL;
    uint64_t b = splitmix64(s);
    return a ^ (b << 1);
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

__device__ __forceinline__ uint64_t twist_word(uint64_t xi, uint64_t xi1, uint64_t xim) {
    uint64_t y = (xi & kUpper) | (xi1 & kLower);
    return xim ^ (y >> 1) ^ ((y & 1ULL) ? kMatA : 0ULL);
}

// mt19937_64::seed(v) by lane 0 (sequential recurrence), window = x_0..x_311
__device__ void warp_seed_window(uint64_t* w, uint64_t v, int lane) {
    if (lane == 0) {
        w[0] = v;
        for (int i = 1; i < kN; ++i) {
            v = 6364136223846793005ULL * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
            w[i] = v;
        }
    }
    __syncwarp();
}

// In-place twist of a 312-word window held in shared memory by one warp.
// Same recurrence as libstdc++'s mersenne_twister_engine::_M_gen_rand: new[i] =
// x[i+156] ^ tw(x[i], x[i+1]) for i < 156 (old values only), then for i >= 156 from the
// new first half.  Each phase loads all its operands before any store (5 words per lane)
// so the phase costs one shared-memory round trip.
__device__ void warp_twist(uint64_t* w, int lane) {
    uint64_t v[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) { // branch-free loads (clamped index) so all 15 overlap
        const int i = min(lane + 32 * q, kN - kM - 1);
        v[q] = twist_word(w[i], w[i + 1], w[i + kM]);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int i = lane + 32 * q;
        if (i < kN - kM)
            w[i] = v[q];
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int i = min(kN - kM + lane + 32 * q, kN - 1);
        v[q] = twist_word(w[i], w[i + 1 < kN ? i + 1 : 0], w[i - kM]);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int i = kN - kM + lane + 32 * q;
        if (i < kN)
            w[i] = v[q];
    }
    __syncwarp();
}

struct GenParams {
    int kind;        // Draw
    double mu, sigma;
    uint64_t count;  // number of transformed values (Gaussian: entries)
    void* out;
    int64_t base;    // output index of out[0] (stream offset of a partial block)
};

// Box-Muller pair of random_gen.cpp:46-52 from two raw draws; returns (cos, sin) entries.
// log and sincos are glibc 2.39's FMA builds step for step (glibc_math.cuh), so every entry
// carries the reference's exact bits; the rest are single IEEE operations in source order.
__device__ __forceinline__ void box_muller(uint64_t r1, uint64_t r2, double mu, double sigma,
                                           double* g0, double* g1) {
    const double u1 = __dsub_rn(1.0, __dmul_rn(static_cast<double>(r1 >> 11), 0x1.0p-53));
    const double u2 = __dmul_rn(static_cast<double>(r2 >> 11), 0x1.0p-53);
    const double r = __dsqrt_rn(__dmul_rn(-2.0, glm::log_fma(u1)));
    double s, c;
    glm::sincos_fma(__dmul_rn(2.0 * 3.14159265358979323846, u2), &s, &c);
    *g0 = __dadd_rn(mu, __dmul_rn(sigma, __dmul_rn(r, c)));
    *g1 = __dadd_rn(mu, __dmul_rn(sigma, __dmul_rn(r, s)));
}

// Emit the outputs carried by one freshly twisted window whose word 0 is stream
// output index o0 (may be negative during the constructor's discard), limited to
// outputs [lo, hi).
__device__ __forceinline__ void emit_block(const uint64_t* w, int64_t o0, int64_t lo, int64_t hi,
                                           const GenParams& p, int lane) {
    if (p.kind == static_cast<int>(Draw::Gaussian)) {
        // pairs (o, o+1) with o even: entries o (cos) and o+1 (sin)
        // two independent Box-Muller pairs per iteration (q, q + 32): branch-free bodies so
        // the two double-double chains interleave (ILP for the latency-bound FP64 pipe)
        double* out = static_cast<double*>(p.out) - p.base;
        auto store = [&](int q, double g0, double g1) {
            const int64_t o = o0 + 2 * q;
            if (o < lo || o >= hi)
                return;
            if (static_cast<uint64_t>(o) + 1 < p.count)
                *reinterpret_cast<double2*>(out + o) = make_double2(g0, g1);
            else
                out[o] = g0;
        };
        for (int q0 = lane; q0 < kN / 2; q0 += 64) {
            const int q1 = q0 + 32;
            const bool v1 = q1 < kN / 2;
            const int qq = v1 ? q1 : q0;
            double g00, g01, g10, g11;
            box_muller(temper(w[2 * q0]), temper(w[2 * q0 + 1]), p.mu, p.sigma, &g00, &g01);
            box_muller(temper(w[2 * qq]), temper(w[2 * qq + 1]), p.mu, p.sigma, &g10, &g11);
            store(q0, g00, g01);
            if (v1)
                store(q1, g10, g11);
        }
        return;
    }
    for (int i = lane; i < kN; i += 32) {
        int64_t o = o0 + i;
        if (o < lo || o >= hi)
            continue;
        uint64_t z = temper(w[i]);
        const int64_t oi = o - p.base;
        switch (p.kind) {
        case static_cast<int>(Draw::RawU64):
            static_cast<uint64_t*>(p.out)[oi] = z;
            break;
        case static_cast<int>(Draw::Uniform01):
            static_cast<double*>(p.out)[oi] = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
            break;
        case static_cast<int>(Draw::UniformPm1):
            static_cast<double*>(p.out)[oi] =
                __dsub_rn(__dmul_rn(2.0, __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53)), 1.0);
            break;
        default: // Sign
            static_cast<double*>(p.out)[oi] = (z & 1ULL) ? 1.0 : -1.0;
            break;
        }
    }
}

// Short streams: one warp from the seed; outputs [p.base, nout).
__global__ void k_gen_small(uint64_t eseed, uint64_t nout, GenParams p) {
    __shared__ uint64_t w[kN];
    int lane = threadIdx.x;
    warp_seed_window(w, eseed, lane);
    // window at time 0; after each twist word 0 is stream position 312k -> output 312k - 8
    for (int64_t pos = 0; pos < static_cast<int64_t>(nout) + 8; pos += kN) {
        warp_twist(w, lane);
        if (pos + kN - 8 > p.base)
            emit_block(w, pos - 8, p.base, static_cast<int64_t>(nout), p, lane);
    }
}

// Word sequences x_0 .. x_{kSeqWords-1} that feed the jumps: from a seeded engine
// (k_base_sequence, the base for level-1 jumps) or continuing each jumped window
// (k_window_sequence).  One 320-thread CTA per sequence, every thread twisting
// (cta_twist_oop): 65 twist blocks in a row, where one warp per sequence was latency-bound.
constexpr int kSeqThreads = 320;
__device__ __forceinline__ void cta_twist_oop(const uint64_t* src, uint64_t* dst, int t);
__device__ __forceinline__ void cta_sequence(uint64_t (*wb)[kN], uint64_t* seq, int t, int words = kSeqWords) {
    int cur = 0;
    for (int base = 0; base < words; base += kN) {
        if (t < kN && base + t < words)
            seq[base + t] = wb[cur][t];
        if (base + kN < words)
            cta_twist_oop(wb[cur], wb[cur ^ 1], t);
        cur ^= 1;
    }
}
__global__ void __launch_bounds__(kSeqThreads) k_base_sequence(uint64_t eseed, uint64_t* seq) {
    __shared__ uint64_t wb[2][kN];
    const int t = threadIdx.x;
    if (t < 32)
        warp_seed_window(wb[0], eseed, t);
    __syncthreads();
    cta_sequence(wb, seq, t, kSeqWords + 8); // + 8: from x_8 it is also level-1 window 0's sequence
}
__global__ void __launch_bounds__(kSeqThreads) k_window_sequence(const uint64_t* windows, uint64_t* seqs) {
    __shared__ uint64_t wb[2][kN];
    const int t = threadIdx.x;
    const uint64_t* src = windows + static_cast<size_t>(blockIdx.x) * kN;
    if (t < kN)
        wb[0][t] = src[t];
    __syncthreads();
    cta_sequence(wb, seqs + static_cast<size_t>(blockIdx.x) * kSeqWords, t);
}

// Jump: out window t = XOR_{i : poly[i]} seq[i + j], j = 0..311.
// Target b of block uses poly polys[(first_poly + b) % poly_mod] and base sequence
// seqs[(b / seq_div)].  The XOR is shared-memory-bandwidth bound (~10^4 terms per word);
// with parts > 1 the terms of one target are split over `parts` CTAs (each loads only the
// sequence slice its terms touch) and k_jump_xor folds the partial windows: a draw of a
// few chunks then uses the whole GPU instead of one SM per chunk.
constexpr int kJumpThreads = 320;
__global__ void __launch_bounds__(kJumpThreads) k_jump(const uint64_t* polys, uint64_t poly_mod,
                                                       const uint64_t* seqs, bool seq_single,
                                                       uint64_t c_first, int stride, uint64_t a_first,
                                                       int ntargets, int parts, uint64_t* out,
                                                       uint64_t* partial) {
    extern __shared__ __align__(16) uint64_t sm[];
    uint64_t* x = sm;                                              // kSeqWords
    uint16_t* list = reinterpret_cast<uint16_t*>(sm + kSeqWords);  // up to 19937 offsets
    __shared__ int wcount[kN];
    __shared__ int total;
    const int tgt = blockIdx.x / parts, part = blockIdx.x - tgt * parts;
    if (tgt >= ntargets)
        return;
    // target chunk c = c_first + stride * tgt: poly c mod poly_mod applied to base sequence
    // c / poly_mod (relative to a_first), result in out slot c - c_first
    const uint64_t c = c_first + static_cast<uint64_t>(stride) * tgt;
    const uint64_t* poly = polys + static_cast<size_t>(c % poly_mod) * kN;
    const uint64_t* seq = seqs + (seq_single ? 0 : static_cast<size_t>(c / poly_mod - a_first) * kSeqWords);
    const int t = threadIdx.x;
    uint64_t pw = 0;
    if (t < kN) {
        pw = poly[t];
        wcount[t] = __popcll(pw);
    }
    __syncthreads();
    if (t == 0) { // exclusive scan of 312 counts (tiny)
        int acc = 0;
        for (int i = 0; i < kN; ++i) {
            int c2 = wcount[i];
            wcount[i] = acc;
            acc += c2;
        }
        total = acc;
    }
    __syncthreads();
    if (t < kN) {
        int pos = wcount[t];
        while (pw) {
            int b = __ffsll(static_cast<long long>(pw)) - 1;
            pw &= pw - 1;
            list[pos++] = static_cast<uint16_t>(64 * t + b);
        }
    }
    __syncthreads();
    const int n = total;
    const int k_lo = static_cast<int>(static_cast<int64_t>(n) * part / parts);
    const int k_hi = static_cast<int>(static_cast<int64_t>(n) * (part + 1) / parts);
    // offsets ascend: this part reads seq[list[k_lo] .. list[k_hi - 1] + 311]
    const int x_lo = k_hi > k_lo ? list[k_lo] : 0;
    const int x_hi = k_hi > k_lo ? min(static_cast<int>(list[k_hi - 1]) + kN, kSeqWords) : 0;
    for (int i = x_lo + t; i < x_hi; i += kJumpThreads)
        x[i] = seq[i];
    __syncthreads();
    if (t < kN) {
        uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        const uint64_t* xj = x + t;
        int k = k_lo;
        for (; k < k_hi && (k & 3); ++k) // to a 4-aligned list index for the 8-byte reads
            a0 ^= xj[list[k]];
        for (; k + 4 <= k_hi; k += 4) {
            uint2 ids = *reinterpret_cast<const uint2*>(list + k); // 4 x u16, 8B aligned
            a0 ^= xj[ids.x & 0xffffu];
            a1 ^= xj[ids.x >> 16];
            a2 ^= xj[ids.y & 0xffffu];
            a3 ^= xj[ids.y >> 16];
        }
        for (; k < k_hi; ++k)
            a0 ^= xj[list[k]];
        const uint64_t r = a0 ^ a1 ^ a2 ^ a3;
        if (parts == 1)
            out[static_cast<size_t>(c - c_first) * kN + t] = r;
        else
            partial[static_cast<size_t>(blockIdx.x) * kN + t] = r;
    }
}

// out slot of target b = XOR of its `parts` partial windows
__global__ void k_jump_xor(const uint64_t* partial, int parts, int stride, uint64_t* out) {
    const int tgt = blockIdx.x, t = threadIdx.x;
    if (t >= kN)
        return;
    uint64_t r = 0;
    for (int p = 0; p < parts; ++p)
        r ^= partial[(static_cast<size_t>(tgt) * parts + p) * kN + t];
    out[static_cast<size_t>(tgt) * stride * kN + t] = r;
}

// CTA-parallel twist of one 312-word block (threads 0..311 each own one word): two phases
// (words 0..155 from the old block, 156..311 from the new first half), two barriers.
__device__ __forceinline__ void cta_twist_oop(const uint64_t* src, uint64_t* dst, int t) {
    if (t < kN - kM)
        dst[t] = twist_word(src[t], src[t + 1], src[t + kM]);
    __syncthreads();
    if (t >= kN - kM && t < kN)
        dst[t] = twist_word(src[t], t + 1 < kN ? src[t + 1] : dst[0], dst[t - kM]);
    __syncthreads();
}

// Tempered words of chunks (raw output of k_gen_chunks for Draw::RawU64), one 320-thread CTA
// per chunk twisting with every thread: for draws of a few chunks, whose single-warp twist
// chain would set the time.
__global__ void __launch_bounds__(kJumpThreads) k_raw_chunks(const uint64_t* windows, uint64_t c_first,
                                                             uint64_t nchunks, uint64_t nout, int64_t base,
                                                             uint64_t* raw) {
    __shared__ uint64_t wb[2][kN];
    const int t = threadIdx.x;
    const uint64_t ci = blockIdx.x;
    if (ci >= nchunks)
        return;
    const uint64_t c = c_first + ci;
    if (t < kN)
        wb[1][t] = windows[ci * kN + t];
    __syncthreads();
    cta_twist_oop(wb[1], wb[0], t);
    const int64_t clo = static_cast<int64_t>(c * kJ);
    const int64_t lo = max(clo, base);
    const int64_t hi = static_cast<int64_t>(min(nout, (c + 1) * kJ));
    int cur = 0;
    for (int64_t o0 = clo; o0 < hi; o0 += kN) {
        if (t < kN) {
            const int64_t o = o0 + t;
            if (o >= lo && o < hi)
                raw[o - base] = temper(wb[cur][t]);
        }
        if (o0 + kN < hi)
            cta_twist_oop(wb[cur], wb[cur ^ 1], t);
        cur ^= 1;
    }
}

// Chunk windows between jumped ones by twisting forward: warp k starts from the jumped
// window of chunk kS and emits the windows of chunks kS + s (s = 1..S-1), which start
// s J words later (J = 105 * 312 + 8, so a window straddles two twist blocks).  About
// 105 twists per window instead of a 19937-term jump.
__global__ void k_window_forward(uint64_t* cw, uint64_t nchunks, int stride) {
    __shared__ uint64_t cur[kN], prev[kN];
    const int lane = threadIdx.x;
    const uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * stride;
    for (int i = lane; i < kN; i += 32)
        cur[i] = cw[k0 * kN + i];
    __syncwarp();
    uint64_t m = 0; // cur holds block m (words [312 m, 312 m + 312) after the jumped window)
    for (int sidx = 1; sidx < stride && k0 + sidx < nchunks; ++sidx) {
        const uint64_t P = static_cast<uint64_t>(sidx) * kJ, mb = P / kN;
        const int off = static_cast<int>(P % kN);
        while (m < mb) {
            warp_twist(cur, lane);
            ++m;
        }
        uint64_t* dst = cw + (k0 + sidx) * kN;
        if (off == 0) {
            for (int i = lane; i < kN; i += 32)
                dst[i] = cur[i];
            continue;
        }
        for (int i = lane; i < kN; i += 32)
            prev[i] = cur[i];
        __syncwarp();
        warp_twist(cur, lane);
        ++m;
        for (int i = lane; i < kN; i += 32)
            dst[i] = (i < kN - off) ? prev[off + i] : cur[i - (kN - off)];
        __syncwarp();
    }
}

// Out-of-place twist dst = twist(src) by one warp (same recurrence as warp_twist).
__device__ void warp_twist_oop(const uint64_t* src, uint64_t* dst, int lane) {
    uint64_t v[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int i = min(lane + 32 * q, kN - kM - 1);
        v[q] = twist_word(src[i], src[i + 1], src[i + kM]);
    }
#pragma unroll
    for (int q = 0; q < 5; ++q)
        if (lane + 32 * q < kN - kM)
            dst[lane + 32 * q] = v[q];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int i = min(kN - kM + lane + 32 * q, kN - 1);
        v[q] = twist_word(src[i], i + 1 < kN ? src[i + 1] : dst[0], dst[i - kM]);
    }
#pragma unroll
    for (int q = 0; q < 5; ++q)
        if (kN - kM + lane + 32 * q < kN)
            dst[kN - kM + lane + 32 * q] = v[q];
}

// One CTA of 160 threads per chunk: window at stream position 8 + cJ -> outputs
// [cJ, cJ + J).  Per 312-word block warp 0 twists the next block into the other buffer
// while every thread transforms its share of the current one (one Box-Muller pair per
// thread for Gaussians), one barrier per block: five warps per chunk keep the FP64 pipe
// fed where one warp per chunk left it latency-bound.
constexpr int kGenThreads = 160;

__device__ __forceinline__ void store_pair(const GenParams& p, int64_t o, double g0, double g1) {
    double* out = static_cast<double*>(p.out) - p.base;
    if (static_cast<uint64_t>(o) + 1 < p.count)
        *reinterpret_cast<double2*>(out + o) = make_double2(g0, g1);
    else
        out[o] = g0;
}
__global__ void __launch_bounds__(kGenThreads) k_gen_chunks(const uint64_t* windows, uint64_t c_first,
                                                            uint64_t nchunks, uint64_t nout, GenParams p) {
    __shared__ uint64_t wb[2][kN];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t ci = blockIdx.x;
    if (ci >= nchunks)
        return;
    const uint64_t c = c_first + ci;
    for (int i = tid; i < kN; i += kGenThreads)
        wb[1][i] = windows[ci * kN + i];
    __syncthreads();
    if (warp == 0)
        warp_twist_oop(wb[1], wb[0], lane);
    __syncthreads();
    const int64_t clo = static_cast<int64_t>(c * kJ);
    const int64_t lo = max(clo, p.base);
    const int64_t hi = static_cast<int64_t>(min(nout, (c + 1) * kJ));
    int cur = 0;
    for (int64_t o0 = clo; o0 < hi; o0 += kN) {
        const uint64_t* w = wb[cur];
        if (warp == 0 && o0 + kN < hi)
            warp_twist_oop(w, wb[cur ^ 1], lane);
        if (o0 + kN > lo) {
            if (p.kind == static_cast<int>(Draw::Gaussian)) {
                const int q = tid; // pair (o, o + 1), o = o0 + 2q: entries o (cos) and o + 1 (sin)
                if (q < kN / 2) {
                    const int64_t o = o0 + 2 * q;
                    if (o >= lo && o < hi) {
                        const uint64_t w0 = temper(w[2 * q]), w1 = temper(w[2 * q + 1]);
                        double g0, g1;
                        box_muller(w0, w1, p.mu, p.sigma, &g0, &g1);
                        store_pair(p, o, g0, g1);
                    }
                }
            } else {
                for (int i = tid; i < kN; i += kGenThreads) {
                    const int64_t o = o0 + i;
                    if (o < lo || o >= hi)
                        continue;
                    const uint64_t z = temper(w[i]);
                    const int64_t oi = o - p.base;
                    switch (p.kind) {
                    case static_cast<int>(Draw::RawU64):
                        static_cast<uint64_t*>(p.out)[oi] = z;
                        break;
                    case static_cast<int>(Draw::Uniform01):
                        static_cast<double*>(p.out)[oi] = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
                        break;
                    case static_cast<int>(Draw::UniformPm1):
                        static_cast<double*>(p.out)[oi] =
                            __dsub_rn(__dmul_rn(2.0, __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53)), 1.0);
                        break;
                    default: // Sign
                        static_cast<double*>(p.out)[oi] = (z & 1ULL) ? 1.0 : -1.0;
                        break;
                    }
                }
            }
        }
        __syncthreads();
        cur ^= 1;
    }
}

// Gaussian pairs from tempered words: pair q = entries base + 2q (cos), base + 2q + 1 (sin).
__global__ void k_gaussian_pairs(const uint64_t* raw, uint64_t npairs, GenParams p) {
    const uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (q >= npairs)
        return;
    const ulonglong2 w = reinterpret_cast<const ulonglong2*>(raw)[q];
    double g0, g1;
    box_muller(w.x, w.y, p.mu, p.sigma, &g0, &g1);
    store_pair(p, p.base + static_cast<int64_t>(2 * q), g0, g1);
}

// Per-thread streams, n <= 148 sign draws each (only the first twist's phase 1 is
// needed: new[i] = x[i+156] ^ tw(x[i], x[i+1]) for i < 8 + n <= 156).
__global__ void k_sign_batched(uint64_t seed, const uint64_t* sids, uint64_t add, uint64_t xor_mask,
                               uint64_t batch, int n, double* out) {
    uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= batch)
        return;
    uint64_t v = engine_seed(seed, (sids[t] + add) ^ xor_mask);
    const int need = 8 + n; // new words 0 .. need-1
    uint64_t lo[157], hi[157];
    lo[0] = v;
    for (int i = 1; i < kN; ++i) {
        v = 6364136223846793005ULL * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
        if (i <= need)
            lo[i] = v;
        if (i >= kM && i < kM + need)
            hi[i - kM] = v;
        if (i >= kM + need)
            break;
    }
    for (int i = 8; i < need; ++i) {
        uint64_t z = temper(twist_word(lo[i], lo[i + 1], hi[i]));
        out[t * n + (i - 8)] = (z & 1ULL) ? 1.0 : -1.0;
    }
}

// ---------------------------------------------------------------- tables --
struct JumpTable {
    uint64_t* d_l1 = nullptr;
    uint64_t* d_l2 = nullptr;
    int n_l1 = 0, n_l2 = 0;
};

std::mutex g_jt_mu;
JumpTable g_jt[16];

std::string lib_dir() {
    Dl_info info;
    if (dladdr(reinterpret_cast<void*>(&lib_dir), &info) && info.dli_fname) {
        std::string p(info.dli_fname);
        auto s = p.rfind('/');
        return s == std::string::npos ? std::string(".") : p.substr(0, s);
    }
    return ".";
}

const JumpTable& jump_table() {
    int dev = ctx().device;
    std::lock_guard<std::mutex> lk(g_jt_mu);
    JumpTable& jt = g_jt[dev & 15];
    if (jt.d_l1)
        return jt;
    std::string path = lib_dir() + "/mt64_jump.bin";
    FILE* fh = std::fopen(path.c_str(), "rb");
    if (!fh)
        fail(RL_ERROR, "mt19937_64 jump table missing: " + path + " (run __graft_entry__.build())");
    uint64_t magic = 0;
    uint32_t hdr[4] = {0, 0, 0, 0};
    bool ok = std::fread(&magic, 8, 1, fh) == 1 && std::fread(hdr, 4, 4, fh) == 4 &&
              magic == 0x314A3436544D4C52ULL && hdr[0] == kN && hdr[1] == kLog2J;
    std::vector<uint64_t> buf;
    if (ok) {
        buf.resize(static_cast<size_t>(hdr[2] + hdr[3]) * kN);
        ok = std::fread(buf.data(), 8, buf.size(), fh) == buf.size();
    }
    std::fclose(fh);
    if (!ok)
        fail(RL_ERROR, "mt19937_64 jump table corrupt: " + path);
    uint64_t* d = nullptr;
    RL_CUDA(cudaMalloc(&d, buf.size() * 8));
    RL_CUDA(cudaMemcpy(d, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice));
    jt.d_l1 = d;
    jt.d_l2 = d + static_cast<size_t>(hdr[2]) * kN;
    jt.n_l1 = static_cast<int>(hdr[2]);
    jt.n_l2 = static_cast<int>(hdr[3]);
    return jt;
}

constexpr size_t kJumpSmem = kSeqWords * 8 + 19968 * 2 + 16;
constexpr int kFwdStride = 8; // chunks per level-2 jump (the rest twist forward)

} // namespace

// Outputs [offset, offset + count) of stream (seed, sid) (offset must be even for Gaussians).
void rng_generate_at(uint64_t seed, uint64_t sid, Draw kind, uint64_t offset, uint64_t count, double mu,
                     double sigma, void* d_out) {
    if (count == 0)
        return;
    if (kind == Draw::Gaussian && (offset & 1ULL))
        fail(RL_INVALID_ARGUMENT, "rng: Gaussian blocks start at an even stream offset");
    const uint64_t end = offset + count;
    GenParams p{static_cast<int>(kind), mu, sigma, end, d_out, static_cast<int64_t>(offset)};
    uint64_t nend = (kind == Draw::Gaussian) ? ((end + 1) & ~1ULL) : end;
    uint64_t eseed = engine_seed(seed, sid);
    cudaStream_t st = stream();
    if (nend <= kSmallMax) {
        k_gen_small<<<1, 32, 0, st>>>(eseed, end, p);
        RL_LAUNCHED();
        return;
    }
    const JumpTable& jt = jump_table();
    const uint64_t c_first = offset / kJ, c_last = (nend - 1) / kJ;
    const uint64_t nchunks = c_last - c_first + 1;
    const uint64_t a_first = c_first / jt.n_l2, a_last = c_last / jt.n_l2;
    const uint64_t nl1 = a_last - a_first + 1;
    if (a_last >= static_cast<uint64_t>(jt.n_l1))
        fail(RL_TOO_LARGE, "rng: stream longer than 2^30 draws");
    static bool attr_set[16] = {};
    if (!attr_set[ctx().device & 15]) {
        RL_CUDA(cudaFuncSetAttribute(k_jump, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kJumpSmem)));
        attr_set[ctx().device & 15] = true;
    }
    uint64_t* base = ws<uint64_t>(WS_RNG, kSeqWords + 8 + nl1 * kN + nl1 * kSeqWords);
    uint64_t* l1w = base + kSeqWords + 8;
    uint64_t* l1s = l1w + nl1 * kN;
    uint64_t* cw = ws<uint64_t>(WS_RNG2, nchunks * kN);
    k_base_sequence<<<1, kSeqThreads, 0, st>>>(eseed, base);
    RL_LAUNCHED();
    if (a_first == 0 && nl1 == 1) {
        // level-1 window 0 is the state at stream position 8, x_8 .. x_319: its word sequence
        // is the base sequence from x_8 (no level-1 jump, no second sequence)
        l1s = base + 8;
    } else {
        k_jump<<<static_cast<unsigned>(nl1), kJumpThreads, kJumpSmem, st>>>(jt.d_l1, 1ULL << 40, base, true, a_first,
                                                                            1, a_first, static_cast<int>(nl1), 1, l1w,
                                                                            nullptr);
        RL_LAUNCHED();
        k_window_sequence<<<static_cast<unsigned>(nl1), kSeqThreads, 0, st>>>(l1w, l1s);
        RL_LAUNCHED();
    }
    // level-2 jumps for every stride-th chunk, the others by twisting forward.  A draw of at
    // most one wave of chunks jumps to every chunk (the jumps run side by side; forward
    // twisting would add a serial 7-chunk walk).
    const uint64_t sms = static_cast<uint64_t>(ctx().sms);
    const int stride = nchunks <= sms ? 1 : kFwdStride;
    const uint64_t njump = (nchunks + stride - 1) / stride;
    // fewer jumps than SMs: split each jump's XOR terms over several CTAs
    const int parts = njump * 2 <= sms ? static_cast<int>(std::min<uint64_t>(16, sms / njump)) : 1;
    uint64_t* partial = parts > 1 ? ws<uint64_t>(WS_RNG4, njump * parts * kN) : nullptr;
    k_jump<<<static_cast<unsigned>(njump * parts), kJumpThreads, kJumpSmem, st>>>(
        jt.d_l2, static_cast<uint64_t>(jt.n_l2), l1s, false, c_first, stride, a_first, static_cast<int>(njump),
        parts, cw, partial);
    RL_LAUNCHED();
    if (parts > 1) {
        k_jump_xor<<<static_cast<unsigned>(njump), kJumpThreads, 0, st>>>(partial, parts, stride, cw);
        RL_LAUNCHED();
    }
    if (stride > 1 && nchunks > 1) {
        k_window_forward<<<static_cast<unsigned>(njump), 32, 0, st>>>(cw, nchunks, stride);
        RL_LAUNCHED();
    }
    if (kind == Draw::Gaussian && nchunks * 2 <= sms) {
        // few chunks: one CTA per chunk would run the Box-Muller chain latency-bound on a
        // handful of SMs; emit the tempered words, then transform all pairs grid-wide
        uint64_t* raw = ws<uint64_t>(WS_RNG3, nend - offset);
        k_raw_chunks<<<static_cast<unsigned>(nchunks), kJumpThreads, 0, st>>>(cw, c_first, nchunks, nend,
                                                                               static_cast<int64_t>(offset), raw);
        RL_LAUNCHED();
        const uint64_t npairs = (nend - offset) / 2;
        k_gaussian_pairs<<<cdiv(npairs, 128), 128, 0, st>>>(raw, npairs, p);
        RL_LAUNCHED();
        return;
    }
    k_gen_chunks<<<static_cast<unsigned>(nchunks), kGenThreads, 0, st>>>(cw, c_first, nchunks, end, p);
    RL_LAUNCHED();
}

void rng_generate(uint64_t seed, uint64_t sid, Draw kind, uint64_t count, double mu, double sigma,
                  void* d_out) {
    rng_generate_at(seed, sid, kind, 0, count, mu, sigma, d_out);
}

namespace {
__global__ void k_box_muller_pairs(const uint64_t* raw, uint64_t npairs, double* out) {
    uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (q >= npairs)
        return;
    double g0, g1;
    box_muller(raw[2 * q], raw[2 * q + 1], 0.0, 1.0, &g0, &g1);
    out[2 * q] = g0;
    out[2 * q + 1] = g1;
}
} // namespace

// Box-Muller (random_gen.cpp:46-52) of consecutive raw pairs: out[2q] = r cos a, out[2q+1] = r sin a.
void box_muller_pairs_dev(const uint64_t* d_raw, uint64_t npairs, double* d_out) {
    if (npairs == 0)
        return;
    k_box_muller_pairs<<<cdiv(npairs, 128), 128, 0, stream()>>>(d_raw, npairs, d_out);
    RL_LAUNCHED();
}

void rng_sign_vectors_batched(uint64_t seed, const uint64_t* d_sids, uint64_t add, uint64_t xor_mask,
                              uint64_t batch, uint64_t n, double* d_out) {
    if (batch == 0)
        return;
    if (n > 148)
        fail(RL_INVALID_ARGUMENT, "batched sign vectors: n > 148");
    k_sign_batched<<<cdiv(batch, 128), 128, 0, stream()>>>(seed, d_sids, add, xor_mask, batch,
                                                           static_cast<int>(n), d_out);
    RL_LAUNCHED();
}

// ------------------------------------------------------ sparse +-1 (NEW) --
namespace {
// Consumption of a raw pool (random_gen.cpp:59-70 uniform_int rejection, then signs): per
// column nnz distinct rows by uniform_int(0, n-1) then nnz signs, columns in order on ONE
// stream.  A column normally takes 2 nnz draws; a rejected or duplicate row costs one more,
// which shifts every later column.  One CTA resolves the offsets by fixed-point iteration:
// every column is consumed in parallel from its current offset guess, the guesses are
// replaced by the exclusive prefix sum of the draw counts, and this repeats until no count
// changes (the first column whose count changed is exact after each round, and extra draws
// are rare: a few rounds).  The result equals the serial consumption bit for bit.
constexpr int kSpThreads = 1024;
__device__ __forceinline__ int sparse_column(const uint64_t* pool, uint64_t pool_len, uint64_t s, uint64_t span,
                                             uint64_t limit, int nnz, int32_t* rj, double* sj, bool write,
                                             bool& exhausted) {
    uint64_t k = s;
    int32_t rows[8];
    for (int t = 0; t < nnz; ++t) {
        for (;;) {
            if (k >= pool_len) {
                exhausted = true;
                return static_cast<int>(k - s);
            }
            const uint64_t v = pool[k++];
            if (v >= limit)
                continue;
            const int32_t r = static_cast<int32_t>(v % span);
            bool dup = false;
            for (int u = 0; u < t; ++u)
                dup |= (rows[u] == r);
            if (!dup) {
                rows[t] = r;
                break;
            }
        }
    }
    for (int t = 0; t < nnz; ++t) {
        if (k >= pool_len) {
            exhausted = true;
            return static_cast<int>(k - s);
        }
        const double sg = (pool[k++] & 1ULL) ? 1.0 : -1.0;
        if (write) {
            rj[t] = rows[t];
            sj[t] = sg;
        }
    }
    return static_cast<int>(k - s);
}

__global__ void __launch_bounds__(kSpThreads) k_sparse_consume(const uint64_t* pool, uint64_t pool_len, uint64_t n,
                                                               int nnz, int32_t* rows, double* signs,
                                                               uint64_t* offs, int* status) {
    __shared__ unsigned long long part[kSpThreads];
    __shared__ int changed, exhausted_any;
    const int tid = threadIdx.x;
    const uint64_t span = n, limit = (~0ULL) / span * span;
    const uint64_t per = (n + kSpThreads - 1) / kSpThreads; // columns per thread (contiguous)
    const uint64_t j0 = tid * per, j1 = j0 + per < n ? j0 + per : n;
    for (uint64_t j = j0; j < j1; ++j)
        offs[j] = static_cast<uint64_t>(2 * nnz) * j;
    __syncthreads();
    for (int round = 0; round < 64; ++round) {
        if (tid == 0) {
            changed = 0;
            exhausted_any = 0;
        }
        __syncthreads();
        // draw counts from the current offsets, prefix sums within the thread's columns
        unsigned long long local = 0;
        bool ex = false;
        for (uint64_t j = j0; j < j1; ++j)
            local += sparse_column(pool, pool_len, offs[j], span, limit, nnz, nullptr, nullptr, false, ex);
        part[tid] = local;
        if (ex)
            exhausted_any = 1;
        __syncthreads();
        // exclusive scan of the per-thread totals (Hillis-Steele over 1024 entries)
        for (int d = 1; d < kSpThreads; d <<= 1) {
            const unsigned long long v = tid >= d ? part[tid - d] : 0ULL;
            __syncthreads();
            part[tid] += v;
            __syncthreads();
        }
        uint64_t s = tid ? part[tid - 1] : 0ULL;
        for (uint64_t j = j0; j < j1; ++j) {
            if (offs[j] != s) {
                offs[j] = s;
                changed = 1;
            }
            bool ex2 = false;
            s += sparse_column(pool, pool_len, s, span, limit, nnz, nullptr, nullptr, false, ex2);
        }
        __syncthreads();
        if (!changed)
            break;
        __syncthreads();
    }
    bool ex = false;
    if (!changed) {
        for (uint64_t j = j0; j < j1; ++j)
            sparse_column(pool, pool_len, offs[j], span, limit, nnz, rows + j * nnz, signs + j * nnz, true, ex);
    } else if (tid == 0) { // no fixed point within the round cap: the serial consumption
        uint64_t k = 0;
        for (uint64_t j = 0; j < n && !ex; ++j)
            k += sparse_column(pool, pool_len, k, span, limit, nnz, rows + j * nnz, signs + j * nnz, true, ex);
    }
    if (ex)
        exhausted_any = 1;
    __syncthreads();
    if (tid == 0)
        *status = exhausted_any ? 1 : 0;
}
} // namespace

void rng_sparse_sign(uint64_t seed, uint64_t sid, uint64_t n, int nnz, int32_t* d_rows,
                     double* d_signs) {
    // 2 nnz draws per column + slack for (rare) rejections; retried with a larger pool.
    uint64_t slack = 1024 + n / 8;
    for (int tries = 0; tries < 4; ++tries, slack *= 8) {
        uint64_t len = 2ULL * nnz * n + slack;
        uint64_t* pool = ws<uint64_t>(WS_TMP2, len + n + 1);
        uint64_t* offs = pool + len;
        int* d_status = reinterpret_cast<int*>(offs + n);
        rng_generate(seed, sid, Draw::RawU64, len, 0.0, 1.0, pool);
        k_sparse_consume<<<1, kSpThreads, 0, stream()>>>(pool, len, n, nnz, d_rows, d_signs, offs, d_status);
        RL_LAUNCHED();
        int h = 0;
        RL_CUDA(cudaMemcpyAsync(&h, d_status, sizeof(int), cudaMemcpyDeviceToHost, stream()));
        RL_CUDA(cudaStreamSynchronize(stream()));
        if (h == 0)
            return;
    }
    fail(RL_ERROR, "sparse_sign: draw pool exhausted");
}


namespace {
// Per-chunk checksums of Box-Muller outputs for the pairs (splitmix64(seed + 2q),
// splitmix64(seed + 2q + 1)), q < npairs: hashes[q / chunk] += mix(q, bits(r cos a),
// bits(r sin a)) (wrapping integer sums: independent of the summation order). The host side
// (tests/cpp/bm_libm_check.cpp) forms the same sums with the installed libm.
__global__ void k_bm_hash(uint64_t seed, uint64_t npairs, uint64_t chunk, unsigned long long* hashes) {
    for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < npairs;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t st = seed + 2 * q;
        const uint64_t w0 = splitmix64(st);
        const uint64_t w1 = splitmix64(st);
        double g0, g1;
        box_muller(w0, w1, 0.0, 1.0, &g0, &g1);
        const uint64_t h = glm::pair_hash(q, static_cast<uint64_t>(__double_as_longlong(g0)),
                                        static_cast<uint64_t>(__double_as_longlong(g1)));
        atomicAdd(&hashes[q / chunk], static_cast<unsigned long long>(h));
    }
}
} // namespace

void box_muller_hash_dev(uint64_t seed, uint64_t npairs, uint64_t chunk, unsigned long long* d_hashes) {
    cudaStream_t st = stream();
    const uint64_t nchunks = (npairs + chunk - 1) / chunk;
    RL_CUDA(cudaMemsetAsync(d_hashes, 0, nchunks * sizeof(unsigned long long), st));
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((npairs + 255) / 256, 148ULL * 16));
    k_bm_hash<<<blocks, 256, 0, st>>>(seed, npairs, chunk, d_hashes);
    RL_LAUNCHED();
}
} // namespace rl

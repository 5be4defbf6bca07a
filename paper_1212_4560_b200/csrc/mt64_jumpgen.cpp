// Build-time generator of the mt19937_64 jump-ahead table (lib/mt64_jump.bin).
//
// The reference draws every multiplier from ONE sequential mt19937_64 stream per
// (seed, stream_id) (random_gen.cpp:22-31, 72-80).  To generate an n x n
// Gaussian on 148 SMs the GPU splits the stream into chunks of J = 2^15 engine
// steps and starts each chunk from the engine state T^t s_0 (t = 8 + c*J; the 8
// is the constructor's discard(8)).  T^t = p_t(T) with p_t = x^t mod phi, phi the
// degree-19937 characteristic polynomial of the mt19937_64 transition, so the
// state at time t is the GF(2) combination  XOR_{i: p_t[i]=1} (window at time i).
//
// phi is found by Berlekamp-Massey on the low bit of the untempered word
// sequence, and every table polynomial is verified against the defining
// relation in tests (tests/test_rng.py).  Table layout (little endian):
//   u64 magic 'RLMT64J1', u32 words (312), u32 log2J (15), u32 n_l1, u32 n_l2,
//   then n_l1 polys  x^(8 + a*2^21) mod phi   (a = 0..n_l1-1, level-1 windows)
//   then n_l2 polys  x^(b*2^15) mod phi       (b = 0..n_l2-1, level-2 offsets)
// each poly = 312 u64 words, bit i of word w = coefficient of x^(64w+i).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

constexpr int kDeg = 19937;
constexpr int kWords = 312; // 312*64 = 19968 >= 19937
constexpr int kLog2J = 15;
constexpr int kL1 = 512; // 512 * 2^21 = 2^30 outputs per stream
constexpr int kL2 = 64;  // 64 * 2^15 = 2^21

using Poly = std::vector<uint64_t>;

// untempered mt19937_64 word sequence x_0, x_1, ... from an arbitrary seed
std::vector<uint64_t> word_sequence(uint64_t seed, std::size_t count) {
    std::vector<uint64_t> x(count + 312);
    x[0] = seed;
    for (int i = 1; i < 312; ++i)
        x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + static_cast<uint64_t>(i);
    for (std::size_t k = 0; k + 312 < x.size(); ++k) {
        uint64_t y = (x[k] & 0xFFFFFFFF80000000ULL) | (x[k + 1] & 0x7FFFFFFFULL);
        x[k + 312] = x[k + 156] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    return x;
}

inline int getbit(const Poly& p, int i) { return static_cast<int>((p[i >> 6] >> (i & 63)) & 1ULL); }

// Berlekamp-Massey over GF(2); returns phi as a bit polynomial (bit i = coeff x^i).
Poly berlekamp_massey(const std::vector<uint8_t>& s) {
    const int N = static_cast<int>(s.size());
    const int W = (N + 63) / 64 + 2;
    Poly C(W, 0), B(W, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    // reversed sequence bit array so that sum_{i=1..L} C_i s_{n-i} is a window AND
    std::vector<uint64_t> rev(W + 2, 0);
    for (int k = 0; k < N; ++k)
        if (s[N - 1 - k])
            rev[k >> 6] |= 1ULL << (k & 63);
    auto rev_window = [&](int off) -> uint64_t { // bits rev[off .. off+63]
        int w = off >> 6, b = off & 63;
        uint64_t lo = rev[w] >> b;
        uint64_t hi = b ? (rev[w + 1] << (64 - b)) : 0ULL;
        return lo | hi;
    };
    for (int n = 0; n < N; ++n) {
        // d = s_n + sum_{i=1..L} C_i s_{n-i};  s_{n-i} = rev[N-1-n+i]
        uint64_t acc = 0;
        const int base = N - 1 - n; // rev index of s_n (i = 0)
        const int words = (L + 64) / 64;
        for (int w = 0; w < words; ++w)
            acc ^= C[w] & rev_window(base + 64 * w);
        // bits of C beyond L are zero, C_0 = 1 contributes s_n itself
        int d = __builtin_parityll(acc);
        if (!d) {
            ++m;
            continue;
        }
        T = C;
        // C -= x^m B
        const int ws = m >> 6, bs = m & 63;
        for (int w = W - 1; w >= 0; --w) {
            uint64_t v = 0;
            if (w - ws >= 0)
                v = B[w - ws] << bs;
            if (bs && w - ws - 1 >= 0)
                v |= B[w - ws - 1] >> (64 - bs);
            C[w] ^= v;
        }
        if (2 * L <= n) {
            L = n + 1 - L;
            B = T;
            m = 1;
        } else {
            ++m;
        }
    }
    if (L != kDeg) {
        std::fprintf(stderr, "mt64_jumpgen: BM found degree %d, expected %d\n", L, kDeg);
        std::exit(1);
    }
    // phi(x) = x^L C(1/x): coefficient of x^(L-i) is C_i
    Poly phi(kWords + 1, 0);
    for (int i = 0; i <= L; ++i)
        if (getbit(C, i))
            phi[(L - i) >> 6] |= 1ULL << ((L - i) & 63);
    return phi;
}

struct Field {
    Poly phi;                              // degree kDeg, kWords+1 words
    std::vector<Poly> phi_sh;              // phi << s, s = 0..63
    explicit Field(Poly p) : phi(std::move(p)) {
        phi_sh.resize(64);
        for (int s = 0; s < 64; ++s) {
            Poly q(kWords + 2, 0);
            for (int w = 0; w <= kWords; ++w) {
                q[w] ^= phi[w] << s;
                if (s)
                    q[w + 1] ^= phi[w] >> (64 - s);
            }
            phi_sh[s] = q;
        }
    }
    // reduce r (2*kWords+2 words) mod phi in place; result in the first kWords words
    void reduce(Poly& r) const {
        for (int i = 64 * static_cast<int>(r.size()) - 1; i >= kDeg; --i) {
            if (!((r[i >> 6] >> (i & 63)) & 1ULL))
                continue;
            int sh = i - kDeg; // xor phi << sh
            int ws = sh >> 6, bs = sh & 63;
            const Poly& q = phi_sh[bs];
            for (int w = 0; w < kWords + 2 && w + ws < static_cast<int>(r.size()); ++w)
                r[w + ws] ^= q[w];
        }
        r.resize(kWords);
    }
    Poly mulmod(const Poly& a, const Poly& b) const {
        std::vector<Poly> bsh(64, Poly(kWords + 1, 0));
        for (int s = 0; s < 64; ++s)
            for (int w = 0; w < kWords; ++w) {
                bsh[s][w] ^= b[w] << s;
                if (s)
                    bsh[s][w + 1] ^= b[w] >> (64 - s);
            }
        Poly r(2 * kWords + 2, 0);
        for (int w = 0; w < kWords; ++w) {
            uint64_t aw = a[w];
            while (aw) {
                int s = __builtin_ctzll(aw);
                aw &= aw - 1;
                const Poly& q = bsh[s];
                for (int k = 0; k <= kWords; ++k)
                    r[w + k] ^= q[k];
            }
        }
        reduce(r);
        return r;
    }
    Poly x_pow2k(int k) const { // x^(2^k) mod phi
        Poly p(kWords, 0);
        p[0] = 2; // x
        for (int i = 0; i < k; ++i)
            p = mulmod(p, p);
        return p;
    }
};

} // namespace

int main(int argc, char** argv) {
    if (argc != 2) {
        std::fprintf(stderr, "usage: mt64_jumpgen OUT.bin\n");
        return 2;
    }
    const int N = 2 * kDeg + 64;
    auto x = word_sequence(5489ULL, static_cast<std::size_t>(N));
    std::vector<uint8_t> bits(N);
    for (int i = 0; i < N; ++i)
        bits[i] = static_cast<uint8_t>(x[i + 1] & 1ULL); // x_1.. (x_0's low bits are not state)
    Field f(berlekamp_massey(bits));

    std::vector<Poly> l1, l2;
    Poly one(kWords, 0);
    one[0] = 1;
    Poly q = f.x_pow2k(kLog2J); // x^(2^15)
    Poly cur = one;
    for (int b = 0; b < kL2; ++b) {
        l2.push_back(cur);
        cur = f.mulmod(cur, q);
    }
    Poly r = f.x_pow2k(kLog2J + 6); // x^(2^21)
    Poly x8(kWords, 0);
    x8[0] = 1ULL << 8;
    cur = x8;
    for (int a = 0; a < kL1; ++a) {
        l1.push_back(cur);
        cur = f.mulmod(cur, r);
    }
    FILE* fh = std::fopen(argv[1], "wb");
    if (!fh) {
        std::perror("mt64_jumpgen");
        return 1;
    }
    uint64_t magic = 0x314A3436544D4C52ULL; // "RLMT64J1"
    uint32_t hdr[4] = {kWords, kLog2J, kL1, kL2};
    std::fwrite(&magic, 8, 1, fh);
    std::fwrite(hdr, 4, 4, fh);
    for (auto& p : l1)
        std::fwrite(p.data(), 8, kWords, fh);
    for (auto& p : l2)
        std::fwrite(p.data(), 8, kWords, fh);
    std::fclose(fh);
    return 0;
}

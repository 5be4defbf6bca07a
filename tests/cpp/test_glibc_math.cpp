// Host check of csrc/glibc_math.cuh against the installed libm, bit for bit.
// Build: g++ -O2 -std=c++17 -mfma -ffp-contract=off -pthread -I<csrc> test_glibc_math.cpp
// Run:   test_glibc_math [log2 samples per family] [threads]
// Families: the Box-Muller domain of the reference's Rng::gaussian (random_gen.cpp:46-52) —
// log(1 - k·2^-53) and sincos(2π·k·2^-53) for random 53-bit k — plus random doubles over
// (0, 1] by exponent, [0, 2π), the ±1e-3 neighbourhoods of the branch points, and edges.
// Prints one line per family and exits 1 on any mismatch.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>
#include <thread>
#include <vector>

#include "glibc_math.cuh"

static inline uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t b64(double x) { return glm::bits(x); }

struct Counts {
    std::atomic<uint64_t> n{0}, bad{0};
};

static bool check_log(double x, Counts& c) {
    const double want = log(x), got = glm::log_fma(x);
    c.n++;
    if (b64(want) != b64(got)) {
        if (c.bad++ < 5)
            printf("  log mismatch x=%a libm=%a port=%a\n", x, want, got);
        return false;
    }
    return true;
}
static bool check_sincos(double x, Counts& c) {
    double s0, c0, s1, c1;
    sincos(x, &s0, &c0);
    if (!glm::sincos_fma(x, &s1, &c1))
        return true;  // outside the restated range
    c.n++;
    if (b64(s0) != b64(s1) || b64(c0) != b64(c1)) {
        if (c.bad++ < 5)
            printf("  sincos mismatch x=%a libm=(%a,%a) port=(%a,%a)\n", x, s0, c0, s1, c1);
        return false;
    }
    return true;
}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 24;
    const int nt = argc > 2 ? atoi(argv[2]) : (int)std::thread::hardware_concurrency();
    const uint64_t N = 1ULL << lg;
    const double two_pi = 2.0 * 3.14159265358979323846;
    struct Fam {
        const char* name;
        int kind;
    } fams[] = {{"box_muller_log", 0}, {"box_muller_sincos", 1}, {"log_unit_by_exponent", 2},
                {"sincos_0_2pi", 3},   {"sincos_branch_points", 4}, {"log_near_one", 5},
                {"sincos_signed", 6}};
    int fail = 0;
    for (const Fam& f : fams) {
        Counts c;
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                uint64_t s = 0x1234567ULL + 0x9e37ULL * (uint64_t)t + 1000003ULL * (uint64_t)f.kind;
                for (uint64_t i = t; i < N; i += nt) {
                    const uint64_t r = splitmix(s);
                    switch (f.kind) {
                    case 0:
                        check_log(1.0 - (double)(r >> 11) * 0x1.0p-53, c);
                        break;
                    case 1:
                        check_sincos(two_pi * ((double)(r >> 11) * 0x1.0p-53), c);
                        break;
                    case 2: {  // random mantissa, exponent in [-1074, 0]
                        const int e = (int)(r % 1075);
                        const double m = 1.0 + (double)(splitmix(s) >> 12) * 0x1.0p-52;
                        double x = ldexp(m, -e);
                        if (x > 1.0) x = 1.0;
                        if (x > 0.0) check_log(x, c);
                        break;
                    }
                    case 3:
                        check_sincos(7.0 * ((double)(r >> 11) * 0x1.0p-53), c);
                        break;
                    case 4: {
                        static const double pts[] = {0.126, 0.855469, 0.85546875, 2.426265,
                                                     0x1.921fb54442d18p+0, 0x1.921fb54442d18p+1,
                                                     0x1.2d97c7f3321d2p+1, 0x1.921fb54442d18p+2,
                                                     0x1p-27, 0x1p-26};
                        const double p = pts[r % 10];
                        const double d = ((double)(splitmix(s) >> 11) * 0x1.0p-53 - 0.5) * 2e-3 * p;
                        check_sincos(p + d, c);
                        break;
                    }
                    case 5: {
                        const double x = 0.93 + 0.14 * ((double)(r >> 11) * 0x1.0p-53);
                        check_log(x, c);
                        break;
                    }
                    case 6: // negative and positive arguments (the FFT's forward twiddles are < 0)
                        check_sincos(14.0 * ((double)(r >> 11) * 0x1.0p-53) - 7.0, c);
                        break;
                    }
                }
            });
        for (auto& x : th) x.join();
        printf("%-24s %12llu checked %8llu mismatches\n", f.name, (unsigned long long)c.n.load(),
               (unsigned long long)c.bad.load());
        fail |= c.bad.load() != 0;
    }
    // Edges: every value Box-Muller's u1 can take at its ends, and x = 0, tiny, ulp steps.
    Counts e;
    for (int k = 0; k < 4096; ++k) {
        check_log(1.0 - (double)k * 0x1.0p-53, e);
        check_log((double)(k + 1) * 0x1.0p-53, e);
        check_sincos(two_pi * ((double)k * 0x1.0p-53), e);
        check_sincos(two_pi * (1.0 - (double)(k + 1) * 0x1.0p-53), e);
    }
    for (int k = 1; k < 40; ++k) { // structured::fft's wlen angles: +-(2 pi) / 2^k
        check_sincos(2.0 * 3.14159265358979323846 / ldexp(1.0, k), e);
        check_sincos(-2.0 * 3.14159265358979323846 / ldexp(1.0, k), e);
    }
    check_log(0x1p-1074, e);
    check_log(0x1.fffffffffffffp-1023, e);
    printf("%-24s %12llu checked %8llu mismatches\n", "edges", (unsigned long long)e.n.load(),
           (unsigned long long)e.bad.load());
    fail |= e.bad.load() != 0;
    return fail;
}

// GPU Box-Muller (rl_box_muller_hash) against this host's libm log/sincos, bit for bit.
// The reference's Rng::gaussian (/root/reference/proj/src/random_gen.cpp:46-52) computed on the
// host is the oracle here: same raw pairs (splitmix64, see rl_b200.h), same per-chunk order-free
// checksums; any chunk whose sums differ is re-run through rl_box_muller and its mismatching
// pairs are printed.
// Usage: bm_libm_check [log2 pairs (default 26)] [seed]
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <thread>
#include <vector>

#include "glibc_math.cuh"  // pair_hash only
#include "rl_b200.h"

static uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Rng::gaussian with the host libm: -2.0 * log(u1), sqrt, 2*pi*u2, sincos (what GCC emits
// for the reference's std::sin / std::cos pair).
static void host_pair(uint64_t w0, uint64_t w1, double* g0, double* g1) {
    volatile double u1 = 1.0 - (double)(w0 >> 11) * 0x1.0p-53;
    volatile double u2 = (double)(w1 >> 11) * 0x1.0p-53;
    double r = sqrt(-2.0 * log(u1));
    double a = 2.0 * 3.14159265358979323846 * u2;
    double s, c;
    sincos(a, &s, &c);
    *g0 = r * c;
    *g1 = r * s;
}
static uint64_t b64(double x) {
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 26;
    const uint64_t seed = argc > 2 ? strtoull(argv[2], nullptr, 0) : 0x5eed1234ULL;
    const uint64_t npairs = 1ULL << lg, chunk = 1ULL << 20;
    const uint64_t nchunks = (npairs + chunk - 1) / chunk;
    std::vector<uint64_t> gpu(nchunks), host(nchunks, 0);
    if (rl_box_muller_hash(seed, npairs, chunk, gpu.data()) != RL_OK) {
        fprintf(stderr, "rl_box_muller_hash: %s\n", rl_last_error());
        return 2;
    }
    const int nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (uint64_t c = t; c < nchunks; c += nt) {
                uint64_t h = 0;
                for (uint64_t q = c * chunk; q < std::min(npairs, (c + 1) * chunk); ++q) {
                    uint64_t st = seed + 2 * q;
                    const uint64_t w0 = splitmix64(st), w1 = splitmix64(st);
                    double g0, g1;
                    host_pair(w0, w1, &g0, &g1);
                    h += glm::pair_hash(q, b64(g0), b64(g1));
                }
                host[c] = h;
            }
        });
    for (auto& x : th) x.join();
    uint64_t bad_chunks = 0;
    for (uint64_t c = 0; c < nchunks; ++c) {
        if (gpu[c] == host[c])
            continue;
        if (bad_chunks++ >= 4)
            continue;
        // drill down: the chunk's raw pairs through rl_box_muller
        const uint64_t q0 = c * chunk, m = std::min(npairs, (c + 1) * chunk) - q0;
        std::vector<uint64_t> raw(2 * m);
        std::vector<double> out(2 * m);
        for (uint64_t i = 0; i < m; ++i) {
            uint64_t st = seed + 2 * (q0 + i);
            raw[2 * i] = splitmix64(st);
            raw[2 * i + 1] = splitmix64(st);
        }
        rl_box_muller(m, raw.data(), out.data());
        int shown = 0;
        for (uint64_t i = 0; i < m && shown < 5; ++i) {
            double g0, g1;
            host_pair(raw[2 * i], raw[2 * i + 1], &g0, &g1);
            if (b64(g0) != b64(out[2 * i]) || b64(g1) != b64(out[2 * i + 1])) {
                printf("pair %llu: u1=%a u2=%a host=(%a,%a) gpu=(%a,%a)\n",
                       (unsigned long long)(q0 + i), 1.0 - (double)(raw[2 * i] >> 11) * 0x1.0p-53,
                       (double)(raw[2 * i + 1] >> 11) * 0x1.0p-53, g0, g1, out[2 * i], out[2 * i + 1]);
                ++shown;
            }
        }
    }
    printf("{\"pairs\": %llu, \"chunks\": %llu, \"mismatched_chunks\": %llu, \"host_threads\": %d}\n",
           (unsigned long long)npairs, (unsigned long long)nchunks, (unsigned long long)bad_chunks, nt);
    return bad_chunks ? 1 : 0;
}

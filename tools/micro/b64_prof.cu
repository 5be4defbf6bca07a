// Phase timer for one config-2 system (dev aid): the batched kernel compiled with RL_B64_PROF,
// launched for 1 and for 888 systems; prints clock64 cycles per phase of system 0.
// Build: see tools/micro/b64_prof.sh
#define RL_B64_PROF 1
#include "../../paper_1212_4560_b200/csrc/genp_batched.cu"
#include <cstdio>
#include <random>
#include <vector>

int main() {
    rl_init(0);
    const uint64_t B = 4096;
    std::vector<double> hA(B * 4096), hb(B * 64);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (auto& v : hA) v = nd(g);
    for (auto& v : hb) v = nd(g);
    std::vector<uint64_t> hs(B);
    for (uint64_t i = 0; i < B; ++i) hs[i] = i;
    double *dA, *db, *dx;
    uint64_t* ds;
    rl_precond_report* dr;
    cudaMalloc(&dA, hA.size() * 8);
    cudaMalloc(&db, hb.size() * 8);
    cudaMalloc(&dx, hb.size() * 8);
    cudaMalloc(&ds, B * 8);
    cudaMalloc(&dr, B * sizeof(rl_precond_report));
    cudaMemcpy(dA, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, hs.data(), B * 8, cudaMemcpyHostToDevice);
    const char* names[] = {"-", "setup/top/mask", "spectrum", "stage A", "FFT", "wb/cyclic load", "LU",
                           "store+fold", "brk/lft", "solve", "y=Cz", "refine", "residual", "tail"};
    for (uint64_t nb : {1ULL, 888ULL, 4096ULL}) {
        for (int rep = 0; rep < 2; ++rep) {
            long long z[32] = {};
            cudaMemcpyToSymbol(rl::g_b64_prof, z, sizeof(z));
            rl::batched_circ64(nb, dA, db, 0, 0, 5, ds, dx, dr);
            cudaDeviceSynchronize();
            cudaMemcpyFromSymbol(z, rl::g_b64_prof, sizeof(z));
            if (rep == 1) {
                long long tot = 0;
                for (int i = 1; i < 14; ++i) tot += z[i];
                printf("batch %llu: system 0 total %lld cycles\n", (unsigned long long)nb, tot);
                for (int i = 1; i < 14; ++i) printf("  %-16s %8lld\n", names[i], z[i]);
            }
        }
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (uint64_t nb : {148ULL, 888ULL, 4096ULL}) {
        rl::batched_circ64(nb, dA, db, 0, 0, 5, ds, dx, dr);
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i)
            rl::batched_circ64(nb, dA, db, 0, 0, 5, ds, dx, dr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("batch %5llu: %.1f us per call (incl. sign draw + status read)\n", (unsigned long long)nb, ms * 100.0);
    }
    rl_precond_report r;
    cudaMemcpy(&r, dr, sizeof(r), cudaMemcpyDeviceToHost);
    printf("system 0 attempt %d residual %.3e raw %.3e\n", r.attempt, r.residual, r.raw_residual);
    return 0;
}

// Host replay microbench: replay_host_impl with and without the folded drain-verification checksums
// (ReplayChecksums), best of 5. Build: see scripts/gpu_r02_hostsums.sh.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include "internal.h"
int main(int argc, char **argv) {
    uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 24);
    uint32_t K = argc > 2 ? atoi(argv[2]) : 8;
    int threads = argc > 3 ? atoi(argv[3]) : 0;
    std::vector<float> p(n, 0.5f), m(n, 1e-3f), v(n, 1e-6f);
    uint64_t lo[64], hi[64];
    for (uint32_t i = 0; i < K; ++i) { lo[i] = n * i / K; hi[i] = n * (i + 1) / K; }
    std::vector<std::vector<uint16_t>> gl(K);
    const uint16_t *g[64];
    for (uint32_t i = 0; i < K; ++i) { gl[i].assign(hi[i], 0x3c00); g[i] = gl[i].data(); }
    gck_step_record r[64];
    for (uint32_t i = 0; i < K; ++i) { std::memset(&r[i], 0, sizeof(r[i])); r[i].b1=0.9f; r[i].c1=0.1f; r[i].b2=0.999f; r[i].c2=0.001f; r[i].bc1=0.5f; r[i].bc2=0.1f; r[i].lr=1e-3f; r[i].eps=1e-8f; r[i].wd=0.01f; r[i].gs=1.0f; }
    for (int mode = 0; mode < 2; ++mode) {
        double best = 1e30;
        for (int rep = 0; rep < 5; ++rep) {
            gck::ReplayChecksums sums; std::memset(&sums, 0, sizeof(sums));
            int used = 0;
            auto t = std::chrono::steady_clock::now();
            gck::replay_host_impl(r, K, lo, hi, p.data(), m.data(), v.data(), g, threads, &used, nullptr, mode ? &sums : nullptr);
            double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
            if (ms < best) best = ms;
        }
        printf("n=%llu K=%u T=%d sums=%d best %.2f ms\n", (unsigned long long)n, K, threads, mode, best);
    }
}

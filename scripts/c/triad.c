/* Host DRAM roofline for the host replay: STREAM-style triad a = b + s*c over 3 x 2^28 floats
 * with T OpenMP threads; prints GB/s (3 x 4 B per element moved: 2 reads + 1 write). */
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>

int main(int argc, char **argv) {
    const long n = 1L << 28;
    const int T = argc > 1 ? atoi(argv[1]) : omp_get_max_threads();
    float *a = aligned_alloc(64, n * 4), *b = aligned_alloc(64, n * 4), *c = aligned_alloc(64, n * 4);
#pragma omp parallel for num_threads(T)
    for (long i = 0; i < n; ++i) { a[i] = 0; b[i] = 1; c[i] = 2; }
    double best = 1e30;
    for (int r = 0; r < 5; ++r) {
        double t0 = omp_get_wtime();
#pragma omp parallel for num_threads(T)
        for (long i = 0; i < n; ++i) a[i] = b[i] + 3.0f * c[i];
        double t = omp_get_wtime() - t0;
        if (t < best) best = t;
    }
    printf("{\"threads\": %d, \"triad_gbs\": %.1f, \"check\": %.1f}\n", T, 3.0 * 4 * n / best / 1e9, a[n / 2]);
    return 0;
}

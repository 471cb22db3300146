/* A plain-C user of libgockpt (no Python, no torch): one GoCkpt session through the C ABI.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_demo.c \
 *       -L paper_2511_07035_b200 -lgockpt -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o demo
 *   ./demo [n] [K]
 *
 * Generates a synthetic optimizer shard with the harness generator, runs a K-part session of
 * fused AdamW steps, takes the synchronous snapshot S(T) before the last step, finalizes and
 * checks the consistent checkpoint equals the snapshot bit for bit. Exit code 0 on success.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gockpt.h"

#define CK(call)                                                                     \
    do {                                                                             \
        gck_status st_ = (call);                                                     \
        if (st_ != GCK_OK) {                                                         \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, (int)st_, gck_last_error(ctx)); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(int argc, char **argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], NULL, 10) : (1u << 20) + 7;
    const uint32_t K = argc > 2 ? (uint32_t)atoi(argv[2]) : 4;
    gck_ctx *ctx = NULL;
    if (gck_device_count() < 1) {
        fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    float *p, *m, *v;
    uint16_t *g, *w;
    if (cudaMalloc((void **)&p, n * 4) || cudaMalloc((void **)&m, n * 4) || cudaMalloc((void **)&v, n * 4) ||
        cudaMalloc((void **)&g, n * 2) || cudaMalloc((void **)&w, n * 2))
        return 3;
    CK(gck_h_generate(1, 0, 42, 0, 0, n, 0, p, NULL));
    CK(gck_h_generate(2, 0, 42, 0, 0, n, 0, m, NULL));
    CK(gck_h_generate(3, 0, 42, 0, 0, n, 0, v, NULL));

    gck_config cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.abi_version = GCK_ABI_VERSION;
    cfg.n = n;
    cfg.k_min = K;
    cfg.k_max = K;
    cfg.timing = 1;
    cfg.eager_replay = 1;
    const gck_hparams hp = {0.9, 0.999, 1e-8, 0.01};
    const gck_tensors t = {p, m, v, w};
    CK(gck_create(&cfg, &hp, &t, &ctx));

    const uint64_t t0 = 10;
    float *snap_p = malloc(n * 4), *snap_m = malloc(n * 4), *snap_v = malloc(n * 4);
    CK(gck_begin_checkpoint(ctx, t0, K));
    for (uint32_t i = 1; i <= K; ++i) {
        const uint64_t step = t0 + i;
        CK(gck_h_generate(4, 1, 42, step, 0, n, 4, g, NULL));      /* the step's "backward" */
        if (i == K) CK(gck_sync_snapshot(ctx, NULL, snap_p, snap_m, snap_v));  /* S(T) reference */
        gck_step_args a = {step, step, 1e-3, 1.0, 0, g};
        CK(gck_submit(ctx, i, &a, NULL));
    }
    gck_checkpoint ck;
    CK(gck_finalize(ctx, &ck));
    const int ok = ck.step == t0 + K - 1 && memcmp(ck.master, snap_p, n * 4) == 0 &&
                   memcmp(ck.exp_avg, snap_m, n * 4) == 0 && memcmp(ck.exp_avg_sq, snap_v, n * 4) == 0;
    gck_stats s;
    CK(gck_get_stats(ctx, &s));
    printf("c_api_demo: n=%llu K=%u checkpoint S(%llu) %s the synchronous snapshot; d2h %.2f GB in %.2f ms, "
           "host replay %.2f ms\n",
           (unsigned long long)n, K, (unsigned long long)ck.step, ok ? "==" : "!=", s.d2h_bytes / 1e9,
           s.last_session_d2h_ms, s.last_replay_ms);
    CK(gck_release(ctx));
    CK(gck_destroy(ctx));
    free(snap_p);
    free(snap_m);
    free(snap_v);
    return ok ? 0 : 4;
}

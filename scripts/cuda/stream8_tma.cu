// Measurement aid (not the product): the 8-stream pattern of fused_adamw_pack (read p, m, v fp32
// + g bf16, write p, m, v + bf16 out: 28 B/element) moved entirely by the bulk-copy engine:
// one lane per CTA bulk-loads 2048-element tiles into a kStages-deep smem ring (UBLKCP.S.G,
// mbarrier completion) and a second lane bulk-stores each landed tile back (UBLKCP.G.S), releasing
// a stage once the store has read it. No arithmetic, no LDS/STG: the ceiling of a TMA-store
// variant of the fused kernel.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\nW8:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W8;\n}"
                 ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g2s(void *d, const void *s, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(d)), "l"(s), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void s2g(void *d, const void *s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(smem_u32(s)), "r"(bytes)
                 : "memory");
}
}  // namespace

template <int kStages, int kTile, int kLag>
__global__ void __launch_bounds__(64, 1) tma8(float *p, float *m, float *v, const uint16_t *g, uint16_t *out,
                                              uint64_t n) {
    constexpr int kStageBytes = kTile * 14;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes);
    uint64_t *empty = full + kStages;
    const uint64_t n_tiles = n / kTile;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // loader
        uint32_t k = 0;
        for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
            const int s = k % kStages;
            mbar_wait(&empty[s], ((k / kStages) & 1u) ^ 1u);
            mbar_expect_tx(&full[s], kStageBytes);
            uint8_t *st = smem + s * kStageBytes;
            const uint64_t b = t * kTile;
            g2s(st, p + b, kTile * 4, &full[s]);
            g2s(st + kTile * 4, m + b, kTile * 4, &full[s]);
            g2s(st + kTile * 8, v + b, kTile * 4, &full[s]);
            g2s(st + kTile * 12, g + b, kTile * 2, &full[s]);
        }
    } else if (threadIdx.x == 32) {  // storer
        uint32_t k = 0;
        int pend[kLag + 1];
        int np = 0;
        for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
            const int s = k % kStages;
            mbar_wait(&full[s], (k / kStages) & 1u);
            const uint8_t *st = smem + s * kStageBytes;
            const uint64_t b = t * kTile;
            s2g(p + b, st, kTile * 4);
            s2g(m + b, st + kTile * 4, kTile * 4);
            s2g(v + b, st + kTile * 8, kTile * 4);
            s2g(out + b, st + kTile * 12, kTile * 2);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            pend[np++] = s;
            if (np > kLag) {  // keep kLag groups reading; release the oldest once it has been read
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kLag) : "memory");
                mbar_arrive(&empty[pend[0]]);
                for (int i = 1; i < np; ++i) pend[i - 1] = pend[i];
                --np;
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

template <int S, int T, int L>
static int launch(float *p, float *m, float *v, const uint16_t *g, uint16_t *o, uint64_t n, int blocks, void *st) {
    const int smem = S * T * 14 + 2 * S * 8;
    cudaFuncSetAttribute(tma8<S, T, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma8<S, T, L><<<blocks, 64, smem, (cudaStream_t)st>>>(p, m, v, g, o, n);
    return (int)cudaGetLastError();
}

extern "C" int run_tma8(float *p, float *m, float *v, const uint16_t *g, uint16_t *out, uint64_t n, int blocks,
                        int cfg, void *stream) {
    switch (cfg) {
        case 0: return launch<4, 2048, 1>(p, m, v, g, out, n, blocks, stream);
        case 1: return launch<6, 2048, 2>(p, m, v, g, out, n, blocks, stream);
        case 2: return launch<7, 2048, 3>(p, m, v, g, out, n, blocks, stream);
        case 3: return launch<3, 4096, 1>(p, m, v, g, out, n, blocks, stream);
        case 4: return launch<3, 2048, 1>(p, m, v, g, out, n, blocks, stream);  // 2 CTAs/SM
        default: return -1;
    }
}

// Measurement aid (not the product): the achievable HBM bandwidth for fused_adamw_pack's exact
// access pattern without its arithmetic — read p, m, v (fp32) + g (bf16), write p, m, v + bf16
// (28 B/element, 8 concurrent streams), as a persistent grid-stride 16-B vector copy kernel.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(512) stream8(float *p, float *m, float *v, const uint16_t *g, uint16_t *out,
                                              uint64_t n) {
    const uint64_t nq = n / 8;  // 8 elements per iteration: 2 float4 of each fp32 array, 1 uint4 of bf16
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nq; i += (uint64_t)gridDim.x * blockDim.x) {
        float4 *P = reinterpret_cast<float4 *>(p) + 2 * i, *M = reinterpret_cast<float4 *>(m) + 2 * i,
               *V = reinterpret_cast<float4 *>(v) + 2 * i;
        float4 p0 = P[0], p1 = P[1], m0 = M[0], m1 = M[1], v0 = V[0], v1 = V[1];
        uint4 gg = reinterpret_cast<const uint4 *>(g)[i];
        // trivial data dependence so nothing is elided; bytes identical to the real kernel
        p0.x += 1.0f; m0.x += 1.0f; v0.x += 1.0f;
        P[0] = p0; P[1] = p1; M[0] = m0; M[1] = m1; V[0] = v0; V[1] = v1;
        reinterpret_cast<uint4 *>(out)[i] = gg;
    }
}

extern "C" int run_stream8(float *p, float *m, float *v, const uint16_t *g, uint16_t *out, uint64_t n, int blocks,
                           void *stream) {
    stream8<<<blocks, 512, 0, (cudaStream_t)stream>>>(p, m, v, g, out, n);
    return (int)cudaGetLastError();
}

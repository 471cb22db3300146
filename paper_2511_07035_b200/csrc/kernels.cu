// sm_100a kernels of the GoCkpt hot path (arXiv 2511.07035). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo (no --use_fast_math: IEEE
//   division/sqrt and denormals are part of the normative update, R6/R13).
//
//  fused_adamw_pack  a2: one pass over the shard per training step. Loads p, m, v (fp32)
//                    and g (bf16); in a session, stores the PRE-update p, m, v of part i
//                    and the raw g bits of the prefix [0, hi_i) into the HBM staging slot
//                    (§4.2.1); applies the normative AdamW; stores p', m', v' and
//                    RNE_bf16(p'). HBM-bound: 28 B/element + the slot bytes.
//  replay            a5 (GPU variant): brings each staged part j < K from S(t0+j-1) to
//                    S(t0+K-1) by applying updates t0+j..t0+K-1 (§4.3.1).
//  zerocopy_drain    a3 variant: 16-B SM stores from the slot into mapped pinned memory.
//  generate          harness only (NOT the method): the counter-hash input generator of
//                    gockpt_inputs.py, bit-identical to the numpy side.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace gck {
namespace {

struct Rec {
    float b1, c1, b2, c2, bc1, bc2, lr, eps, wd, gs;
};

__device__ __forceinline__ Rec to_rec(const gck_step_record &s) {
    return Rec{s.b1, s.c1, s.b2, s.c2, s.bc1, s.bc2, s.lr, s.eps, s.wd, s.gs};
}

// The normative update; every op is a correctly rounded
// binary32 op with no contraction (the _rn intrinsics are never fused into FMA).
__device__ __forceinline__ void adamw_elem(float &p, float &m, float &v, uint32_t gbits, const Rec &r) {
    const float g = __fmul_rn(__uint_as_float(gbits << 16), r.gs);
    m = __fadd_rn(__fmul_rn(r.b1, m), __fmul_rn(r.c1, g));
    v = __fadd_rn(__fmul_rn(r.b2, v), __fmul_rn(r.c2, __fmul_rn(g, g)));
    const float mh = __fdiv_rn(m, r.bc1);
    const float vh = __fdiv_rn(v, r.bc2);
    const float u = __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), r.eps));
    p = __fsub_rn(p, __fmul_rn(r.lr, __fadd_rn(u, __fmul_rn(r.wd, p))));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // cvt.rn.bf16x2.f32: RNE
    return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ uint32_t bf16_lane(const uint4 &q, int k) {
    const uint32_t w = (k < 2) ? q.x : (k < 4) ? q.y : (k < 6) ? q.z : q.w;
    return (k & 1) ? (w >> 16) : (w & 0xFFFFu);
}

struct Vec8 {
    float x[8];
};

__device__ __forceinline__ Vec8 ld8(const float *ptr) {
    const float4 a = *reinterpret_cast<const float4 *>(ptr);
    const float4 b = *reinterpret_cast<const float4 *>(ptr + 4);
    return Vec8{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
}

__device__ __forceinline__ void st8(float *ptr, const Vec8 &v) {
    *reinterpret_cast<float4 *>(ptr) = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
    *reinterpret_cast<float4 *>(ptr + 4) = make_float4(v.x[4], v.x[5], v.x[6], v.x[7]);
}

template <bool PACK>
__global__ void __launch_bounds__(256) fused_adamw_pack_kernel(const FusedArgs a) {
    const Rec r = to_rec(a.rec);
    const bool skip = a.rec.skip != 0;
    const uint64_t ngroups = a.n >> 3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
        const uint64_t e = gi << 3;
        Vec8 p = ld8(a.p + e), m = ld8(a.m + e), v = ld8(a.v + e);
        const uint4 gq = *reinterpret_cast<const uint4 *>(a.g + e);
        if (PACK) {
            if (e >= a.lo && e < a.hi) {  // lo, hi are multiples of 8 (A % 8 == 0) or hi == n
                const uint64_t o = e - a.lo;
                st8(a.sp + o, p);
                st8(a.sm + o, m);
                st8(a.sv + o, v);
            }
            if (e < a.ghi) *reinterpret_cast<uint4 *>(a.sg + e) = gq;
        }
        if (!skip) {
#pragma unroll
            for (int k = 0; k < 8; ++k) adamw_elem(p.x[k], m.x[k], v.x[k], bf16_lane(gq, k), r);
            st8(a.p + e, p);
            st8(a.m + e, m);
            st8(a.v + e, v);
        }
        if (a.out) {
            uint4 o;
            o.x = pack_bf16x2(p.x[0], p.x[1]);
            o.y = pack_bf16x2(p.x[2], p.x[3]);
            o.z = pack_bf16x2(p.x[4], p.x[5]);
            o.w = pack_bf16x2(p.x[6], p.x[7]);
            *reinterpret_cast<uint4 *>(a.out + e) = o;
        }
    }
    // ragged tail: n % 8 elements, scalar
    const uint64_t tail0 = ngroups << 3;
    if (blockIdx.x == 0 && threadIdx.x < (a.n - tail0)) {
        const uint64_t e = tail0 + threadIdx.x;
        float p = a.p[e], m = a.m[e], v = a.v[e];
        const uint32_t g = a.g[e];
        if (PACK) {
            if (e >= a.lo && e < a.hi) {
                a.sp[e - a.lo] = p;
                a.sm[e - a.lo] = m;
                a.sv[e - a.lo] = v;
            }
            if (e < a.ghi) a.sg[e] = (uint16_t)g;
        }
        if (!skip) {
            adamw_elem(p, m, v, g, r);
            a.p[e] = p;
            a.m[e] = m;
            a.v[e] = v;
        }
        if (a.out) a.out[e] = (uint16_t)(pack_bf16x2(p, 0.f) & 0xFFFFu);
    }
}

__device__ __forceinline__ uint32_t part_of(const ReplayArgs &a, uint64_t e) {
    uint32_t j = 0;
    while (j + 1 < a.K && e >= a.hi[j]) ++j;
    return j;  // 0-based part index
}

__global__ void __launch_bounds__(256) replay_kernel(const ReplayArgs a) {
    const uint64_t ngroups = (a.n_replay + 7) >> 3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
        const uint64_t e = gi << 3;
        const uint32_t j = part_of(a, e);
        const bool full = (e + 8 <= a.hi[j]) && (e + 8 <= a.n_replay);
        if (full) {
            Vec8 p = ld8(a.p + e), m = ld8(a.m + e), v = ld8(a.v + e);
            for (uint32_t i = j; i + 1 < a.K; ++i) {  // updates t0+j+1 .. t0+K-1 (1-based: j+1..K-1)
                if (a.rec[i].skip) continue;
                const Rec r = to_rec(a.rec[i]);
                const uint4 gq = *reinterpret_cast<const uint4 *>(a.glog[i] + e);
#pragma unroll
                for (int k = 0; k < 8; ++k) adamw_elem(p.x[k], m.x[k], v.x[k], bf16_lane(gq, k), r);
            }
            st8(a.p + e, p);
            st8(a.m + e, m);
            st8(a.v + e, v);
        } else {
            for (uint64_t q = e; q < e + 8 && q < a.n_replay; ++q) {
                const uint32_t jq = part_of(a, q);
                float p = a.p[q], m = a.m[q], v = a.v[q];
                for (uint32_t i = jq; i + 1 < a.K; ++i) {
                    if (a.rec[i].skip) continue;
                    adamw_elem(p, m, v, a.glog[i][q], to_rec(a.rec[i]));
                }
                a.p[q] = p;
                a.m[q] = m;
                a.v[q] = v;
            }
        }
    }
}

__global__ void __launch_bounds__(512) zerocopy_drain_kernel(const ZcArgs a) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (int s = 0; s < a.count; ++s) {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.src[s]);
        uint4 *dst = reinterpret_cast<uint4 *>(a.dst[s]);
        const uint64_t nv = a.bytes[s] >> 4;
        uint64_t i = tid;
        for (; i + 3 * stride < nv; i += 4 * stride) {  // 4 independent 16-B loads in flight
            const uint4 x0 = src[i], x1 = src[i + stride], x2 = src[i + 2 * stride], x3 = src[i + 3 * stride];
            dst[i] = x0;
            dst[i + stride] = x1;
            dst[i + 2 * stride] = x2;
            dst[i + 3 * stride] = x3;
        }
        for (; i < nv; i += stride) dst[i] = src[i];
        const uint64_t tail = a.bytes[s] & 15;
        if (tid < tail) {
            reinterpret_cast<uint8_t *>(a.dst[s])[(nv << 4) + tid] =
                reinterpret_cast<const uint8_t *>(a.src[s])[(nv << 4) + tid];
        }
    }
}

// ---- harness-only generator (gockpt_inputs.py) ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__global__ void generate_kernel(int kind, int mode, uint64_t key, uint64_t offset, uint64_t n,
                                uint32_t zero_per_256, void *out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint64_t h = mix64(key ^ (offset + k));
        if (kind == 4) {
            uint16_t bits;
            if (mode == 0) {
                const int64_t q = (int64_t)(h >> 57) - 64;
                const float f = __fmul_rn((float)q, 0.015625f);  // exact
                bits = (uint16_t)(__float_as_uint(f) >> 16);
            } else {
                const uint32_t sign = (uint32_t)(h >> 63) & 1u;
                const uint32_t ex = (uint32_t)(h >> 56) & 15u;
                const uint32_t mant = (uint32_t)(h >> 40) & 0x7Fu;
                bits = (uint16_t)((sign << 15) | ((127u - 6u - ex) << 7) | mant);
                if (((h >> 32) & 0xFFu) < zero_per_256) bits = 0;
            }
            static_cast<uint16_t *>(out)[k] = bits;
        } else {
            const uint64_t u24 = h >> 40;
            float f;
            if (kind == 3) {
                f = __fmul_rn((float)(u24 + 1), 5.684341886080802e-14f);  // 2^-44
            } else {
                const float c = (float)((int64_t)u24 - (1ll << 23));
                const float sc = (kind == 2) ? 1.1641532182693481e-10f                // 2^-33
                                             : (mode == 0 ? 1.1920928955078125e-07f  // 2^-23
                                                          : 1.862645149230957e-09f);  // 2^-29
                f = __fmul_rn(c, sc);
            }
            static_cast<float *>(out)[k] = f;
        }
    }
}

inline unsigned grid_for(uint64_t work_items, unsigned block, int num_sms, unsigned per_sm) {
    const uint64_t need = (work_items + block - 1) / block;
    const uint64_t cap = (uint64_t)(num_sms > 0 ? num_sms : 148) * per_sm;
    const uint64_t g = need < cap ? need : cap;
    return (unsigned)(g > 0 ? g : 1);
}

}  // namespace

int launch_fused(const FusedArgs &a, bool pack, void *stream, int num_sms) {
    const unsigned grid = grid_for(a.n >> 3, 256, num_sms, 8);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (pack)
        fused_adamw_pack_kernel<true><<<grid, 256, 0, s>>>(a);
    else
        fused_adamw_pack_kernel<false><<<grid, 256, 0, s>>>(a);
    return (int)cudaGetLastError();
}

int launch_replay(const ReplayArgs &a, void *stream, int num_sms) {
    if (a.n_replay == 0) return 0;
    const unsigned grid = grid_for((a.n_replay + 7) >> 3, 256, num_sms, 8);
    replay_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
    return (int)cudaGetLastError();
}

int launch_zerocopy_drain(const ZcArgs &a, int ctas, void *stream) {
    zerocopy_drain_kernel<<<ctas > 0 ? ctas : 32, 512, 0, static_cast<cudaStream_t>(stream)>>>(a);
    return (int)cudaGetLastError();
}

int launch_generate(int kind, int mode, uint64_t seed, uint64_t step, uint64_t offset, uint64_t n,
                    uint32_t zero_per_256, void *out, void *stream, int num_sms) {
    if (n == 0) return 0;
    // key = mix(mix(seed ^ stream*GOLD) ^ step), stream = kind (gockpt_inputs.py)
    auto mixh = [](uint64_t z) {
        z ^= z >> 30;
        z *= 0xBF58476D1CE4E5B9ull;
        z ^= z >> 27;
        z *= 0x94D049BB133111EBull;
        z ^= z >> 31;
        return z;
    };
    const uint64_t key = mixh(mixh(seed ^ ((uint64_t)kind * 0x9E3779B97F4A7C15ull)) ^ step);
    const unsigned grid = grid_for(n, 256, num_sms, 8);
    generate_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(kind, mode, key, offset, n, zero_per_256,
                                                                          out);
    return (int)cudaGetLastError();
}

}  // namespace gck

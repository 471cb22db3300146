// sm_100a kernels of the GoCkpt hot path (arXiv 2511.07035). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo (no --use_fast_math: IEEE
//   division/sqrt and denormals are part of the normative update, R6/R13).
//
//  fused_adamw_pack  a2: one pass over the shard per training step (two forms: the TMA-pipelined
//                    kernel, default for n >= 2^18, on the branch-free fast paths of
//                    adamw_math.cuh; and a plain grid-stride kernel on the reference intrinsics). Loads p, m, v (fp32)
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

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "adamw_math.cuh"
#include "internal.h"

namespace gck {
namespace {

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

// ---- TMA-pipelined variant of a2 with STG stores (GCK_FUSED_IMPL=t; the bulk-store variant below is the default) ----
// Persistent CTAs (default: 1 per SM, 4 stages, 16 consumer warps; GCK_TMA_CFG selects other
// instantiations for experiments). One producer warp streams 2048-element tiles of p, m, v
// (fp32) and g (bf16) into a kStages-deep shared-memory ring with 1-D bulk async copies
// (cp.async.bulk, SASS UBLKCP.S.G) completing on mbarriers; the consumer warps compute from
// shared memory (adamw_group_fast) and store p', m', v', bf16(p') with 16-B STG; in a session a
// pack warp bulk-stores the staged pre-update tile into the ring slot (UBLKCP.G.S). Bytes in
// flight per SM no longer depend on registers: up to kStages x 28 KiB.
constexpr uint64_t kTmaMinElems = 1u << 18;
constexpr int tma_smem(int stages, int tile) { return stages * tile * 14 + 2 * stages * 8; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "GCK_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra GCK_WAIT;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("fence.proxy.async.shared::cta;\n\t"
                 "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void process4(const FusedArgs &a, const RecF &r, bool skip, bool pack, uint64_t e,
                                         float4 p4, float4 m4, float4 v4, uint2 g2) {
    float p[4] = {p4.x, p4.y, p4.z, p4.w}, m[4] = {m4.x, m4.y, m4.z, m4.w}, v[4] = {v4.x, v4.y, v4.z, v4.w};
    if (pack) {
        if (e >= a.lo && e < a.hi) {  // part boundaries are multiples of A (a multiple of 8)
            const uint64_t o = e - a.lo;
            *reinterpret_cast<float4 *>(a.sp + o) = p4;
            *reinterpret_cast<float4 *>(a.sm + o) = m4;
            *reinterpret_cast<float4 *>(a.sv + o) = v4;
        }
        if (e < a.ghi) *reinterpret_cast<uint2 *>(a.sg + e) = g2;
    }
    if (!skip) {
        const uint32_t gb[4] = {g2.x & 0xFFFFu, g2.x >> 16, g2.y & 0xFFFFu, g2.y >> 16};
        adamw_group_fast(p, m, v, gb, r);
        *reinterpret_cast<float4 *>(a.p + e) = make_float4(p[0], p[1], p[2], p[3]);
        *reinterpret_cast<float4 *>(a.m + e) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4 *>(a.v + e) = make_float4(v[0], v[1], v[2], v[3]);
    }
    if (a.out) *reinterpret_cast<uint2 *>(a.out + e) = make_uint2(pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]));
}

template <bool PACK, int kStages, int kMinBlocks, int kCW, int kTile>
__global__ void __launch_bounds__((kCW + 2) * 32, kMinBlocks) fused_adamw_pack_tma_kernel(const FusedArgs a) {
    // Warps 0..kCW-1 consume (kQ float4 groups of the tile per thread: elements
    // [4(c + q*kCW*32), +4)); warp kCW produces (bulk loads); warp kCW+1 packs in a session
    // (bulk stores of the staged tile straight into the ring slot) and idles otherwise.
    constexpr int kThreads = kCW * 32;
    constexpr int kStageBytes = kTile * 14;  // p, m, v fp32 + g bf16
    constexpr int kQ = kTile / 4 / kThreads;
    static_assert(kQ * kThreads * 4 == kTile, "tile must split evenly");
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes);
    uint64_t *empty = full + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t n_tiles = a.n / kTile;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCW + (PACK ? 1 : 0));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kCW) {  // producer warp: one elected lane issues the bulk copies
        if (lane == 0) {
            uint32_t k = 0;
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
                const int s = k % kStages;
                const uint32_t ph = (k / kStages) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_expect_tx(&full[s], kStageBytes);
                uint8_t *st = smem + s * kStageBytes;
                const uint64_t base = tile * kTile;
                bulk_g2s(st, a.p + base, kTile * 4, &full[s]);
                bulk_g2s(st + kTile * 4, a.m + base, kTile * 4, &full[s]);
                bulk_g2s(st + kTile * 8, a.v + base, kTile * 4, &full[s]);
                bulk_g2s(st + kTile * 12, a.g + base, kTile * 2, &full[s]);
            }
        }
        return;
    }
    if (warp == kCW + 1) {  // pack warp (session launches only)
        if (PACK && lane == 0) {
            uint32_t k = 0;
            int prev_s = -1;
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
                const int s = k % kStages;
                const uint32_t ph = (k / kStages) & 1u;
                mbar_wait(&full[s], ph);
                const uint8_t *st = smem + s * kStageBytes;
                const uint64_t base = tile * kTile;
                // the pre-update p, m, v of the tile's overlap with [lo, hi); g of its overlap with [0, ghi)
                const uint64_t olo = base > a.lo ? base : a.lo;
                const uint64_t ohi = (base + kTile) < a.hi ? (base + kTile) : a.hi;
                const uint64_t ghi = (base + kTile) < a.ghi ? (base + kTile) : a.ghi;
                bool issued = false;
                if (olo < ohi) {
                    const uint32_t off = (uint32_t)(olo - base), bytes = (uint32_t)(ohi - olo) * 4;
                    bulk_s2g(a.sp + (olo - a.lo), st + off * 4, bytes);
                    bulk_s2g(a.sm + (olo - a.lo), st + kTile * 4 + off * 4, bytes);
                    bulk_s2g(a.sv + (olo - a.lo), st + kTile * 8 + off * 4, bytes);
                    issued = true;
                }
                if (base < ghi) {
                    bulk_s2g(a.sg + base, st + kTile * 12, (uint32_t)(ghi - base) * 2);
                    issued = true;
                }
                // one bulk group per tile (possibly empty); keep one group's smem reads in flight
                // while the next tile arrives, and release a stage only once its group has read it
                bulk_commit();
                (void)issued;
                bulk_wait_read_1();
                if (prev_s >= 0) mbar_arrive(&empty[prev_s]);
                prev_s = s;
            }
            bulk_wait_read();
            if (prev_s >= 0) mbar_arrive(&empty[prev_s]);
            bulk_wait_all();  // slot writes complete before the CTA retires
        }
        return;
    }
    const RecF r = to_recf(a.rec);
    const bool skip = a.rec.skip != 0;
    const int c = threadIdx.x;
    uint32_t k = 0;
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int s = k % kStages;
        const uint32_t ph = (k / kStages) & 1u;
        mbar_wait(&full[s], ph);
        const uint8_t *st = smem + s * kStageBytes;
        const uint64_t base = tile * kTile;
        const float4 *sp = reinterpret_cast<const float4 *>(st);
        const float4 *sm = reinterpret_cast<const float4 *>(st + kTile * 4);
        const float4 *sv = reinterpret_cast<const float4 *>(st + kTile * 8);
        const uint2 *sg = reinterpret_cast<const uint2 *>(st + kTile * 12);
        float4 pq[kQ], mq[kQ], vq[kQ];
        uint2 gq[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            pq[q] = sp[c + q * kThreads];
            mq[q] = sm[c + q * kThreads];
            vq[q] = sv[c + q * kThreads];
            gq[q] = sg[c + q * kThreads];
        }
        // Release the stage only once every lane's shared-memory loads have landed in registers:
        // a dependent instruction on all loaded values makes the scoreboard wait for the LDS
        // results, __syncwarp orders the lanes before lane 0's arrive, and the proxy fence orders
        // these generic-proxy reads before the async-proxy (TMA) refill of the same bytes (WAR).
        // (one component per LDS suffices: an LDS writes all its destination registers under one
        // scoreboard entry, so a use of .x waits for the whole vector)
        uint32_t dep = 0;
#pragma unroll
        for (int q = 0; q < kQ; ++q)
            dep ^= __float_as_uint(pq[q].x) ^ __float_as_uint(mq[q].x) ^ __float_as_uint(vq[q].x) ^ gq[q].x;
        asm volatile("" : "+r"(dep));
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&empty[s]);  // the stage may be refilled while we compute
        }
#pragma unroll
        for (int q = 0; q < kQ; ++q)
            process4(a, r, skip, false, base + 4 * (uint64_t)(c + q * kThreads), pq[q], mq[q], vq[q], gq[q]);
    }
    // ragged tail [n_tiles*kTile, n): block 0's consumers, plain loads
    if (blockIdx.x == 0) {
        for (uint64_t e = n_tiles * kTile + (uint64_t)c; e < a.n; e += kThreads) {
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
                adamw_elem_fast(p, m, v, g, r);
                a.p[e] = p;
                a.m[e] = m;
                a.v[e] = v;
            }
            if (a.out) a.out[e] = (uint16_t)(pack_bf16x2(p, 0.f) & 0xFFFFu);
        }
    }
}

// ---- a2 with bulk stores too (GCK_FUSED_IMPL=x): loads AND stores through the bulk-copy engine ----
// As fused_adamw_pack_tma_kernel, but the consumers write p', m', v', bf16(p') into a kOut-deep
// shared-memory OUTPUT ring and a store warp bulk-copies each finished tile to global memory
// (UBLKCP.G.S), so no STG is issued on the steady-state path. An all-bulk copy of this 8-stream
// pattern holds 6.23 TB/s after a GEMM burst where the LDG/STG copy drops to 5.7
// (profiles/r01_tma8_ceiling.txt): the stores no longer depend on the SM clock. The input stage
// is not written (the pack warp still bulk-stores the pre-update bytes from it).
constexpr int tmast_smem(int stages, int outs, int tile) { return (stages + outs) * tile * 14 + 2 * (stages + outs) * 8; }

template <bool PACK, int kStages, int kOut, int kCW, int kTile>
__global__ void __launch_bounds__((kCW + 3) * 32, 1) fused_adamw_pack_tmast_kernel(const FusedArgs a) {
    // warps 0..kCW-1 consume; warp kCW loads; warp kCW+1 packs (session); warp kCW+2 stores
    constexpr int kThreads = kCW * 32;
    constexpr int kStageBytes = kTile * 14;
    constexpr int kQ = kTile / 4 / kThreads;
    static_assert(kQ * kThreads * 4 == kTile, "tile must split evenly");
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *obuf = smem + kStages * kStageBytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(obuf + kOut * kStageBytes);
    uint64_t *empty = full + kStages;
    uint64_t *ofull = empty + kStages;
    uint64_t *oempty = ofull + kOut;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t n_tiles = a.n / kTile;
    const bool skip = a.rec.skip != 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCW + (PACK ? 1 : 0));
        }
        for (int o = 0; o < kOut; ++o) {
            mbar_init(&ofull[o], kCW);
            mbar_init(&oempty[o], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kCW) {  // loads (as the STG variant)
        if (lane == 0) {
            uint32_t k = 0;
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
                const int s = k % kStages;
                mbar_wait(&empty[s], ((k / kStages) & 1u) ^ 1u);
                mbar_expect_tx(&full[s], kStageBytes);
                uint8_t *st = smem + s * kStageBytes;
                const uint64_t base = tile * kTile;
                bulk_g2s(st, a.p + base, kTile * 4, &full[s]);
                bulk_g2s(st + kTile * 4, a.m + base, kTile * 4, &full[s]);
                bulk_g2s(st + kTile * 8, a.v + base, kTile * 4, &full[s]);
                bulk_g2s(st + kTile * 12, a.g + base, kTile * 2, &full[s]);
            }
        }
        return;
    }
    if (warp == kCW + 1) {  // pack (session launches only): pre-update bytes from the input stage
        if (PACK && lane == 0) {
            uint32_t k = 0;
            int prev_s = -1;
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
                const int s = k % kStages;
                mbar_wait(&full[s], (k / kStages) & 1u);
                const uint8_t *st = smem + s * kStageBytes;
                const uint64_t base = tile * kTile;
                const uint64_t olo = base > a.lo ? base : a.lo;
                const uint64_t ohi = (base + kTile) < a.hi ? (base + kTile) : a.hi;
                const uint64_t ghi = (base + kTile) < a.ghi ? (base + kTile) : a.ghi;
                if (olo < ohi) {
                    const uint32_t off = (uint32_t)(olo - base), bytes = (uint32_t)(ohi - olo) * 4;
                    bulk_s2g(a.sp + (olo - a.lo), st + off * 4, bytes);
                    bulk_s2g(a.sm + (olo - a.lo), st + kTile * 4 + off * 4, bytes);
                    bulk_s2g(a.sv + (olo - a.lo), st + kTile * 8 + off * 4, bytes);
                }
                if (base < ghi) bulk_s2g(a.sg + base, st + kTile * 12, (uint32_t)(ghi - base) * 2);
                bulk_commit();
                bulk_wait_read_1();
                if (prev_s >= 0) mbar_arrive(&empty[prev_s]);
                prev_s = s;
            }
            bulk_wait_read();
            if (prev_s >= 0) mbar_arrive(&empty[prev_s]);
            bulk_wait_all();
        }
        return;
    }
    if (warp == kCW + 2) {  // stores: finished output tiles -> global, one bulk group per tile
        if (lane == 0) {
            uint32_t k = 0;
            int prev_o = -1;
            for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
                const int o = k % kOut;
                mbar_wait(&ofull[o], (k / kOut) & 1u);
                const uint8_t *ot = obuf + o * kStageBytes;
                const uint64_t base = tile * kTile;
                if (!skip) {
                    bulk_s2g(a.p + base, ot, kTile * 4);
                    bulk_s2g(a.m + base, ot + kTile * 4, kTile * 4);
                    bulk_s2g(a.v + base, ot + kTile * 8, kTile * 4);
                }
                if (a.out) bulk_s2g(a.out + base, ot + kTile * 12, kTile * 2);
                bulk_commit();
                bulk_wait_read_1();  // the previous tile's group has read its buffer: release it
                if (prev_o >= 0) mbar_arrive(&oempty[prev_o]);
                prev_o = o;
            }
            bulk_wait_read();
            if (prev_o >= 0) mbar_arrive(&oempty[prev_o]);
            bulk_wait_all();  // every store performed before the CTA retires
        }
        return;
    }
    const RecF r = to_recf(a.rec);
    const int c = threadIdx.x;
    uint32_t k = 0;
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int s = k % kStages;
        mbar_wait(&full[s], (k / kStages) & 1u);
        const uint8_t *st = smem + s * kStageBytes;
        const float4 *sp = reinterpret_cast<const float4 *>(st);
        const float4 *sm = reinterpret_cast<const float4 *>(st + kTile * 4);
        const float4 *sv = reinterpret_cast<const float4 *>(st + kTile * 8);
        const uint2 *sg = reinterpret_cast<const uint2 *>(st + kTile * 12);
        float4 pq[kQ], mq[kQ], vq[kQ];
        uint2 gq[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            pq[q] = sp[c + q * kThreads];
            mq[q] = sm[c + q * kThreads];
            vq[q] = sv[c + q * kThreads];
            gq[q] = sg[c + q * kThreads];
        }
        // release the input stage once every lane's LDS has landed (see the STG variant)
        uint32_t dep = 0;
#pragma unroll
        for (int q = 0; q < kQ; ++q)
            dep ^= __float_as_uint(pq[q].x) ^ __float_as_uint(mq[q].x) ^ __float_as_uint(vq[q].x) ^ gq[q].x;
        asm volatile("" : "+r"(dep));
        __syncwarp();
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&empty[s]);
        }
        // compute, then write the tile's results into output buffer o once the store warp has
        // finished reading its previous contents
        const int o = k % kOut;
        mbar_wait(&oempty[o], ((k / kOut) & 1u) ^ 1u);
        uint8_t *ot = obuf + o * kStageBytes;
        float4 *op = reinterpret_cast<float4 *>(ot);
        float4 *om = reinterpret_cast<float4 *>(ot + kTile * 4);
        float4 *ov = reinterpret_cast<float4 *>(ot + kTile * 8);
        uint2 *og = reinterpret_cast<uint2 *>(ot + kTile * 12);
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            float p[4] = {pq[q].x, pq[q].y, pq[q].z, pq[q].w}, m[4] = {mq[q].x, mq[q].y, mq[q].z, mq[q].w},
                  v[4] = {vq[q].x, vq[q].y, vq[q].z, vq[q].w};
            if (!skip) {
                const uint32_t gb[4] = {gq[q].x & 0xFFFFu, gq[q].x >> 16, gq[q].y & 0xFFFFu, gq[q].y >> 16};
                adamw_group_fast(p, m, v, gb, r);
                op[c + q * kThreads] = make_float4(p[0], p[1], p[2], p[3]);
                om[c + q * kThreads] = make_float4(m[0], m[1], m[2], m[3]);
                ov[c + q * kThreads] = make_float4(v[0], v[1], v[2], v[3]);
            }
            og[c + q * kThreads] = make_uint2(pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]));
        }
        // generic-proxy smem writes -> visible to the async proxy (the bulk store), then arrive
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&ofull[o]);
    }
    // ragged tail [n_tiles*kTile, n): block 0's consumers, plain loads and stores
    if (blockIdx.x == 0) {
        for (uint64_t e = n_tiles * kTile + (uint64_t)c; e < a.n; e += kThreads) {
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
                adamw_elem_fast(p, m, v, g, r);
                a.p[e] = p;
                a.m[e] = m;
                a.v[e] = v;
            }
            if (a.out) a.out[e] = (uint16_t)(pack_bf16x2(p, 0.f) & 0xFFFFu);
        }
    }
}

struct __align__(16) RecP {
    RecF f;
};

__device__ __forceinline__ uint32_t part_of(const ReplayArgs &a, uint64_t e) {
    uint32_t j = 0;
    while (j + 1 < a.K && e >= a.hi[j]) ++j;
    return j;  // 0-based part index
}

// a5 GPU replay, general form: any part boundaries (per-element path where a group of 8 straddles a
// boundary), skipped records tested per step. Used only when replay_kernel's preconditions fail.
__global__ void __launch_bounds__(256) replay_generic_kernel(const ReplayArgs a) {
    // the K step records with their hoisted reciprocals, computed once per CTA
    __shared__ RecF srec[GCK_K_LIMIT];
    __shared__ int sskip[GCK_K_LIMIT];
    for (uint32_t i = threadIdx.x; i < a.K; i += blockDim.x) {
        srec[i] = to_recf(a.rec[i]);
        sskip[i] = a.rec[i].skip;
    }
    __syncthreads();
    const uint64_t ngroups = (a.n_replay + 7) >> 3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
        const uint64_t e = gi << 3;
        const uint32_t j = part_of(a, e);
        const bool full = (e + 8 <= a.hi[j]) && (e + 8 <= a.n_replay);
        if (full) {
            Vec8 p = ld8(a.p + e), m = ld8(a.m + e), v = ld8(a.v + e);
            // software pipeline: the next step's gradient vector is in flight while this step computes
            uint4 gnext = (j + 1 < a.K) ? *reinterpret_cast<const uint4 *>(a.glog[j] + e) : make_uint4(0, 0, 0, 0);
            for (uint32_t i = j; i + 1 < a.K; ++i) {  // updates t0+j+1 .. t0+K-1 (1-based: j+1..K-1)
                const uint4 gq = gnext;
                if (i + 2 < a.K) gnext = *reinterpret_cast<const uint4 *>(a.glog[i + 1] + e);
                if (sskip[i]) continue;
                uint32_t gb[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) gb[k] = bf16_lane(gq, k);
                adamw_group_fast(p.x, m.x, v.x, gb, srec[i]);
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
                    adamw_elem_fast(p, m, v, a.glog[i][q], to_recf(a.rec[i]));
                }
                a.p[q] = p;
                a.m[q] = m;
                a.v[q] = v;
            }
        }
    }
}

// a5 GPU replay (default): brings each stale part j < K-1 (0-based) from S(t0+j) to S(T) with the
// compacted non-skipped StepRecords j .. K-2 (ReplayPlan, built on the host). One thread owns 8
// consecutive elements (two 16-B vectors of p, m, v), keeps them in registers across all of their
// pending updates — the next step's gradient vector in flight while this step computes — and stores
// them once: 24 B + 2 B per pending update per element, the algorithmic minimum. Grid-stride over
// the groups with the part index tracked monotonically (one compare per group); every group lies in
// one part (boundaries are multiples of 8, checked on the host). The update is adamw_group_mm:
// the fused kernel's op sequence, one min/max guard per group and step.
template <bool kUnitGs, bool kAllFast, bool kPacked, int kMinB = 1, bool kMixed = false>
__global__ void __launch_bounds__(256, kMinB) replay_kernel(const ReplayPlan a) {
    __shared__ RecP srec[GCK_K_LIMIT];
    __shared__ __align__(16) RecF2 srec2[GCK_K_LIMIT];
    for (uint32_t q = threadIdx.x; q < a.nact; q += blockDim.x) {
        srec[q].f = to_recf(a.rec[q]);
        srec2[q] = to_recf2(srec[q].f, a.neg_zero);
    }
    __syncthreads();
    const uint64_t ngroups = kMixed ? (a.seg_u0[a.nseg] << 5) : (a.n_replay >> 3);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t j = 0, sg = 0;
    for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
        uint64_t e;
        if (kMixed) {  // warp-uniform 32-group units, heavy and light parts alternating
            const uint64_t u = gi >> 5;
            while (u >= a.seg_u0[sg + 1]) ++sg;
            const uint64_t l = u - a.seg_u0[sg], na = a.seg_na[sg], nb = a.seg_nb[sg];
            const uint64_t both = 2 * (na < nb ? na : nb);
            uint64_t ui;
            if (l < both) {
                j = (l & 1) ? a.seg_b[sg] : a.seg_a[sg];
                ui = l >> 1;
            } else {
                j = na > nb ? a.seg_a[sg] : a.seg_b[sg];
                ui = both / 2 + (l - both);
            }
            e = (j ? a.hi[j - 1] : 0) + ((ui << 5) + (gi & 31)) * 8;
            if (e >= a.hi[j]) continue;  // the part's last unit is partial
        } else {
            e = gi << 3;
            while (e >= a.hi[j]) ++j;  // e only grows: amortised O(1)
        }
        const uint32_t q0 = a.first[j];
        if (q0 >= a.nact) continue;  // every pending update of this part was skipped: already S(T)
        Vec8 p = ld8(a.p + e), m = ld8(a.m + e), v = ld8(a.v + e);
        uint4 gnext = *reinterpret_cast<const uint4 *>(a.glog[q0] + e);
        for (uint32_t q = q0; q < a.nact; ++q) {
            const uint4 gq = gnext;
            if (q + 1 < a.nact) gnext = *reinterpret_cast<const uint4 *>(a.glog[q + 1] + e);
            const uint32_t gb[8] = {gq.x & 0xFFFFu, gq.x >> 16, gq.y & 0xFFFFu, gq.y >> 16,
                                    gq.z & 0xFFFFu, gq.z >> 16, gq.w & 0xFFFFu, gq.w >> 16};
            if (kPacked)
                adamw_group_p2<8, kUnitGs, kAllFast>(p.x, m.x, v.x, gb, srec[q].f, srec2[q]);
            else
                adamw_group_mm<8, kUnitGs, kAllFast>(p.x, m.x, v.x, gb, srec[q].f);
        }
        st8(a.p + e, p);
        st8(a.m + e, m);
        st8(a.v + e, v);
    }
}

// ---- replay_kernel with a per-thread asynchronous prefetch ring (default) ----
// The same per-thread work as replay_kernel, but the loads it waits for are issued early into a
// per-thread shared-memory ring with cp.async (LDGSTS, 16 B each; no registers held in flight):
//   - the next group's p, m, v and its first D gradient vectors, right after this group's state has
//     been read into registers (one group of lead time: the long-scoreboard stall at every group
//     start of replay_kernel);
//   - inside a group, the gradient of step k + D while step k computes (replay_kernel's one-step
//     lead did not cover the HBM latency under load; ncu: 32% of warp samples waited there).
// Every step commits exactly one cp.async group, so "the data of step k" is always the group
// committed D steps earlier: cp.async.wait_group(D-1). Slots are [slot][thread] 16-B entries
// (conflict-free LDS.128). A slot is refilled only after its previous value was consumed in a
// register (a dependent instruction first), so the async write never races the LDS.
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int D>
struct ReplayRing {
    static constexpr int kSlots = 6 + 2 * D;  // p0 p1 m0 m1 v0 v1 | gradients: 2 areas x D
    static constexpr int smem(int threads) { return kSlots * 16 * threads; }
};

template <bool kUnitGs, int D>
__global__ void __launch_bounds__(256, 4) replay_ring_kernel(const ReplayPlan a) {
    extern __shared__ __align__(16) uint4 ring[];
    __shared__ RecP srec[GCK_K_LIMIT];
    __shared__ __align__(16) RecF2 srec2[GCK_K_LIMIT];
    for (uint32_t q = threadIdx.x; q < a.nact; q += blockDim.x) {
        srec[q].f = to_recf(a.rec[q]);
        srec2[q] = to_recf2(srec[q].f, a.neg_zero);
    }
    __syncthreads();
    const uint32_t T = blockDim.x;
    uint4 *slot = ring + threadIdx.x;  // slot s of this thread: slot[s * T]
    const uint64_t ngroups = a.n_replay >> 3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // issue the state + first D gradients of group gi into gradient area `area`; one commit
    uint32_t jn = 0;  // part tracker of the prefetch cursor (groups only grow)
    auto issue_group = [&](uint64_t gi, int area) {
        if (gi < ngroups) {
            const uint64_t e = gi << 3;
            while (e >= a.hi[jn]) ++jn;
            const uint32_t q0 = a.first[jn];
            if (q0 < a.nact) {
                cp_async16(&slot[0 * T], a.p + e);
                cp_async16(&slot[1 * T], a.p + e + 4);
                cp_async16(&slot[2 * T], a.m + e);
                cp_async16(&slot[3 * T], a.m + e + 4);
                cp_async16(&slot[4 * T], a.v + e);
                cp_async16(&slot[5 * T], a.v + e + 4);
                const uint32_t nst = a.nact - q0;
#pragma unroll
                for (int k = 0; k < D; ++k)
                    if ((uint32_t)k < nst) cp_async16(&slot[(6 + area * D + k) * T], a.glog[q0 + k] + e);
            }
        }
        cp_async_commit();
    };
    uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    issue_group(gi, 0);
    uint32_t j = 0;
    int area = 0;
    for (; gi < ngroups; gi += stride, area ^= 1) {
        const uint64_t e = gi << 3;
        while (e >= a.hi[j]) ++j;
        const uint32_t q0 = a.first[j];
        cp_async_wait<0>();  // this group's batch (issued one group ago) has landed
        float p[8], m[8], v[8];
        const bool live = q0 < a.nact;
        if (live) {
            const uint4 s0 = slot[0 * T], s1 = slot[1 * T], s2 = slot[2 * T], s3 = slot[3 * T], s4 = slot[4 * T],
                        s5 = slot[5 * T];
            const uint4 q4[6] = {s0, s1, s2, s3, s4, s5};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                p[4 * h] = __uint_as_float(q4[h].x), p[4 * h + 1] = __uint_as_float(q4[h].y);
                p[4 * h + 2] = __uint_as_float(q4[h].z), p[4 * h + 3] = __uint_as_float(q4[h].w);
                m[4 * h] = __uint_as_float(q4[2 + h].x), m[4 * h + 1] = __uint_as_float(q4[2 + h].y);
                m[4 * h + 2] = __uint_as_float(q4[2 + h].z), m[4 * h + 3] = __uint_as_float(q4[2 + h].w);
                v[4 * h] = __uint_as_float(q4[4 + h].x), v[4 * h + 1] = __uint_as_float(q4[4 + h].y);
                v[4 * h + 2] = __uint_as_float(q4[4 + h].z), v[4 * h + 3] = __uint_as_float(q4[4 + h].w);
            }
            uint32_t dep = s0.x ^ s1.x ^ s2.x ^ s3.x ^ s4.x ^ s5.x;  // the state slots are read: refill them
            asm volatile("" : "+r"(dep)::"memory");
        }
        issue_group(gi + stride, area ^ 1);
        if (!live) continue;  // every pending update of this part was skipped: already S(T)
        const uint32_t nst = a.nact - q0;
        for (uint32_t k = 0; k < nst; ++k) {
            if (k >= (uint32_t)D) cp_async_wait<D - 1>();  // step k's gradient: committed D steps ago
            uint4 *gs = &slot[(6 + area * D + (k % D)) * T];
            const uint4 gq = *gs;
            if (k + D < nst) {
                uint32_t dep = gq.x;
                asm volatile("" : "+r"(dep)::"memory");
                cp_async16(gs, a.glog[q0 + k + D] + e);
            }
            cp_async_commit();
            const uint32_t gb[8] = {gq.x & 0xFFFFu, gq.x >> 16, gq.y & 0xFFFFu, gq.y >> 16,
                                    gq.z & 0xFFFFu, gq.z >> 16, gq.w & 0xFFFFu, gq.w >> 16};
            adamw_group_p2<8, kUnitGs, false>(p, m, v, gb, srec[q0 + k].f, srec2[q0 + k]);
        }
        *reinterpret_cast<float4 *>(a.p + e) = make_float4(p[0], p[1], p[2], p[3]);
        *reinterpret_cast<float4 *>(a.p + e + 4) = make_float4(p[4], p[5], p[6], p[7]);
        *reinterpret_cast<float4 *>(a.m + e) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4 *>(a.m + e + 4) = make_float4(m[4], m[5], m[6], m[7]);
        *reinterpret_cast<float4 *>(a.v + e) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(a.v + e + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
    cp_async_wait<0>();
}

// ---- replay_kernel, 3-way unrolled step loop (default) ----
// As replay_kernel, with the gradient vectors in three rotating register sets: step k computes with
// set k % 3 while the loads of steps k+1 and k+2 are in flight (two steps of lead instead of one;
// ncu showed replay_kernel's warps waiting on the one-step prefetch at the end of every step), and
// no register moves between steps. kPrefState: the next group's p, m, v are prefetched into a
// per-thread shared-memory slot with cp.async while this group computes (the other long-scoreboard
// wait of replay_kernel: the state loads at every group start).
template <bool kUnitGs, bool kAllFast, bool kPrefState, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) replay3_kernel(const ReplayPlan a) {
    extern __shared__ __align__(16) uint4 sstate[];  // kPrefState: [6][blockDim] 16-B slots
    __shared__ RecP srec[GCK_K_LIMIT];
    __shared__ __align__(16) RecF2 srec2[GCK_K_LIMIT];
    for (uint32_t q = threadIdx.x; q < a.nact; q += blockDim.x) {
        srec[q].f = to_recf(a.rec[q]);
        srec2[q] = to_recf2(srec[q].f, a.neg_zero);
    }
    __syncthreads();
    const uint32_t T = blockDim.x;
    uint4 *slot = sstate + threadIdx.x;
    const uint64_t ngroups = a.n_replay >> 3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t j = 0, jn = 0;
    auto pref = [&](uint64_t gi) {  // next group's state -> slot (kPrefState); one commit
        if (gi < ngroups) {
            const uint64_t e = gi << 3;
            while (e >= a.hi[jn]) ++jn;
            if (a.first[jn] < a.nact) {
                cp_async16(&slot[0 * T], a.p + e);
                cp_async16(&slot[1 * T], a.p + e + 4);
                cp_async16(&slot[2 * T], a.m + e);
                cp_async16(&slot[3 * T], a.m + e + 4);
                cp_async16(&slot[4 * T], a.v + e);
                cp_async16(&slot[5 * T], a.v + e + 4);
            }
        }
        cp_async_commit();
    };
    uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (kPrefState) pref(gi);
    for (; gi < ngroups; gi += stride) {
        const uint64_t e = gi << 3;
        while (e >= a.hi[j]) ++j;
        const uint32_t q0 = a.first[j];
        const bool live = q0 < a.nact;
        float p[8], m[8], v[8];
        if (kPrefState) {
            cp_async_wait<0>();
            if (live) {
                const uint4 s0 = slot[0 * T], s1 = slot[1 * T], s2 = slot[2 * T], s3 = slot[3 * T],
                            s4 = slot[4 * T], s5 = slot[5 * T];
                const uint4 q4[6] = {s0, s1, s2, s3, s4, s5};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    p[4 * h] = __uint_as_float(q4[h].x), p[4 * h + 1] = __uint_as_float(q4[h].y);
                    p[4 * h + 2] = __uint_as_float(q4[h].z), p[4 * h + 3] = __uint_as_float(q4[h].w);
                    m[4 * h] = __uint_as_float(q4[2 + h].x), m[4 * h + 1] = __uint_as_float(q4[2 + h].y);
                    m[4 * h + 2] = __uint_as_float(q4[2 + h].z), m[4 * h + 3] = __uint_as_float(q4[2 + h].w);
                    v[4 * h] = __uint_as_float(q4[4 + h].x), v[4 * h + 1] = __uint_as_float(q4[4 + h].y);
                    v[4 * h + 2] = __uint_as_float(q4[4 + h].z), v[4 * h + 3] = __uint_as_float(q4[4 + h].w);
                }
                uint32_t dep = s0.x ^ s1.x ^ s2.x ^ s3.x ^ s4.x ^ s5.x;  // slots read: refill them
                asm volatile("" : "+r"(dep)::"memory");
            }
            pref(gi + stride);
        }
        if (!live) continue;  // every pending update of this part was skipped: already S(T)
        const uint32_t nst = a.nact - q0;
        const uint16_t *const *gl = a.glog + q0;
        const RecP *rr = srec + q0;
        uint4 g0 = *reinterpret_cast<const uint4 *>(gl[0] + e), g1 = make_uint4(0, 0, 0, 0), g2 = g1;
        if (nst > 1) g1 = *reinterpret_cast<const uint4 *>(gl[1] + e);
        if (!kPrefState) {
            const Vec8 pv = ld8(a.p + e), mv = ld8(a.m + e), vv = ld8(a.v + e);
#pragma unroll
            for (int k = 0; k < 8; ++k) p[k] = pv.x[k], m[k] = mv.x[k], v[k] = vv.x[k];
        }
        const RecF2 *rr2 = srec2 + q0;
        auto step = [&](const uint4 &gq, const RecF &r, const RecF2 &c) {
            const uint32_t gb[8] = {gq.x & 0xFFFFu, gq.x >> 16, gq.y & 0xFFFFu, gq.y >> 16,
                                    gq.z & 0xFFFFu, gq.z >> 16, gq.w & 0xFFFFu, gq.w >> 16};
            adamw_group_p2<8, kUnitGs, kAllFast>(p, m, v, gb, r, c);
        };
        uint32_t k = 0;
        for (; k + 3 <= nst; k += 3) {  // sets: step k -> g0, k+1 -> g1, k+2 -> g2
            if (k + 2 < nst) g2 = *reinterpret_cast<const uint4 *>(gl[k + 2] + e);
            step(g0, rr[k].f, rr2[k]);
            if (k + 3 < nst) g0 = *reinterpret_cast<const uint4 *>(gl[k + 3] + e);
            step(g1, rr[k + 1].f, rr2[k + 1]);
            if (k + 4 < nst) g1 = *reinterpret_cast<const uint4 *>(gl[k + 4] + e);
            step(g2, rr[k + 2].f, rr2[k + 2]);
        }
        if (k < nst) {  // 1 or 2 steps left, in g0 (and g1)
            step(g0, rr[k].f, rr2[k]);
            if (k + 1 < nst) step(g1, rr[k + 1].f, rr2[k + 1]);
        }
        *reinterpret_cast<float4 *>(a.p + e) = make_float4(p[0], p[1], p[2], p[3]);
        *reinterpret_cast<float4 *>(a.p + e + 4) = make_float4(p[4], p[5], p[6], p[7]);
        *reinterpret_cast<float4 *>(a.m + e) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4 *>(a.m + e + 4) = make_float4(m[4], m[5], m[6], m[7]);
        *reinterpret_cast<float4 *>(a.v + e) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(a.v + e + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (kPrefState) cp_async_wait<0>();
}

// ---- a5 GPU replay, TMA-pipelined (GCK_REPLAY_IMPL=b) ----
// Persistent CTAs, one per SM. The stale range is cut into tiles of kTile elements that never
// straddle a part. A load warp bulk-copies each tile's p, m, v into a state stage (kS deep) and the
// tile's gradient slices, kGS steps per gradient chunk (kGd deep); kCW consumer warps read the stage
// into registers, apply every pending update (adamw_group_p2) and write the results back into the
// stage; a store warp bulk-stores the finished stage. Each CTA walks its round-robin tiles
// alternately from the front (part 1: K-1 updates) and the back (part K-1: one update) so the ALU-
// and HBM-heavy tiles overlap in the pipeline.
template <int kTile, int kCW, int kS, int kGd, int kGS>
struct ReplayTma {
    static constexpr int kThreads = kCW * 32;
    static constexpr int kQ = kTile / 4 / kThreads;  // float4 groups per consumer thread
    static constexpr int kStateBytes = kTile * 12;
    static constexpr int kChunkBytes = kTile * 2 * kGS;
    static constexpr int smem() { return kS * kStateBytes + kGd * kChunkBytes + (3 * kS + 2 * kGd) * 8; }
    static_assert(kQ * kThreads * 4 == kTile, "tile must split evenly");
};

struct ReplayTiles {  // per-CTA schedule in shared memory
    uint32_t tstart[GCK_K_LIMIT + 1];  // tiles before part j (parts with no pending update: 0 tiles)
    uint32_t nparts;
};

__device__ __forceinline__ uint32_t tile_part(const ReplayTiles &s, uint32_t t) {
    uint32_t lo = 0, hi = s.nparts;  // largest j with tstart[j] <= t
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s.tstart[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t cta_tile(uint32_t k, uint32_t nq) {
    const uint32_t q = (k & 1u) ? (nq - 1u - (k >> 1)) : (k >> 1);
    return blockIdx.x + q * gridDim.x;
}

template <int kTile, int kCW, int kS, int kGd, int kGS, bool kUnitGs>
__global__ void __launch_bounds__((kCW + 2) * 32, 1) replay_tma_kernel(const ReplayPlan a) {
    using C = ReplayTma<kTile, kCW, kS, kGd, kGS>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *gbuf = smem + kS * C::kStateBytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(gbuf + kGd * C::kChunkBytes);
    uint64_t *done = full + kS;
    uint64_t *empty = done + kS;
    uint64_t *gfull = empty + kS;
    uint64_t *gempty = gfull + kGd;
    __shared__ RecP srec[GCK_K_LIMIT];
    __shared__ __align__(16) RecF2 srec2[GCK_K_LIMIT];
    __shared__ ReplayTiles sch;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t nparts = 0;
    while (nparts < GCK_K_LIMIT && (nparts == 0 || a.hi[nparts - 1] < a.n_replay)) ++nparts;
    if (threadIdx.x == 0) {
        uint32_t tiles = 0;
        for (uint32_t j = 0; j < nparts; ++j) {
            sch.tstart[j] = tiles;
            const uint64_t lo = j ? a.hi[j - 1] : 0;
            if (a.first[j] < a.nact) tiles += (uint32_t)((a.hi[j] - lo + kTile - 1) / kTile);
        }
        sch.tstart[nparts] = tiles;
        sch.nparts = nparts;
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], kCW);
            mbar_init(&empty[s], 1);
        }
        for (int g = 0; g < kGd; ++g) {
            mbar_init(&gfull[g], 1);
            mbar_init(&gempty[g], kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t q = threadIdx.x; q < a.nact; q += blockDim.x) {
        srec[q].f = to_recf(a.rec[q]);
        srec2[q] = to_recf2(srec[q].f, a.neg_zero);
    }
    __syncthreads();
    const uint32_t ntiles = sch.tstart[nparts];
    const uint32_t nq = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto tile_of = [&](uint32_t k, uint32_t &j, uint64_t &base, uint32_t &len) {
        const uint32_t t = cta_tile(k, nq);
        j = tile_part(sch, t);
        const uint64_t lo = j ? a.hi[j - 1] : 0;
        base = lo + (uint64_t)(t - sch.tstart[j]) * kTile;
        const uint64_t rem = a.hi[j] - base;
        len = (uint32_t)(rem < (uint64_t)kTile ? rem : (uint64_t)kTile);
    };
    if (warp == kCW) {  // load warp
        if (lane == 0) {
            uint32_t gc = 0;
            for (uint32_t k = 0; k < nq; ++k) {
                uint32_t j, len;
                uint64_t base;
                tile_of(k, j, base, len);
                const int s = k % kS;
                mbar_wait(&empty[s], ((k / kS) & 1u) ^ 1u);
                mbar_expect_tx(&full[s], len * 12);
                uint8_t *st = smem + s * C::kStateBytes;
                bulk_g2s(st, a.p + base, len * 4, &full[s]);
                bulk_g2s(st + kTile * 4, a.m + base, len * 4, &full[s]);
                bulk_g2s(st + kTile * 8, a.v + base, len * 4, &full[s]);
                for (uint32_t q0 = a.first[j]; q0 < a.nact; q0 += kGS, ++gc) {
                    const uint32_t nst = umin((uint32_t)kGS, a.nact - q0);
                    const int g = gc % kGd;
                    mbar_wait(&gempty[g], ((gc / kGd) & 1u) ^ 1u);
                    mbar_expect_tx(&gfull[g], len * 2 * nst);
                    uint8_t *gb = gbuf + g * C::kChunkBytes;
                    for (uint32_t q = 0; q < nst; ++q)
                        bulk_g2s(gb + q * kTile * 2, a.glog[q0 + q] + base, len * 2, &gfull[g]);
                }
            }
        }
        return;
    }
    if (warp == kCW + 1) {  // store warp
        if (lane == 0) {
            int prev = -1;
            for (uint32_t k = 0; k < nq; ++k) {
                uint32_t j, len;
                uint64_t base;
                tile_of(k, j, base, len);
                const int s = k % kS;
                mbar_wait(&done[s], (k / kS) & 1u);
                const uint8_t *st = smem + s * C::kStateBytes;
                bulk_s2g(a.p + base, st, len * 4);
                bulk_s2g(a.m + base, st + kTile * 4, len * 4);
                bulk_s2g(a.v + base, st + kTile * 8, len * 4);
                bulk_commit();
                bulk_wait_read_1();
                if (prev >= 0) mbar_arrive(&empty[prev]);
                prev = s;
            }
            bulk_wait_read();
            if (prev >= 0) mbar_arrive(&empty[prev]);
            bulk_wait_all();
        }
        return;
    }
    const int c = threadIdx.x;
    uint32_t gc = 0;
    for (uint32_t k = 0; k < nq; ++k) {
        uint32_t j, len;
        uint64_t base;
        tile_of(k, j, base, len);
        const int s = k % kS;
        mbar_wait(&full[s], (k / kS) & 1u);
        uint8_t *st = smem + s * C::kStateBytes;
        float4 *sp = reinterpret_cast<float4 *>(st);
        float4 *sm = reinterpret_cast<float4 *>(st + kTile * 4);
        float4 *sv = reinterpret_cast<float4 *>(st + kTile * 8);
        float p[4 * C::kQ], m[4 * C::kQ], v[4 * C::kQ];
#pragma unroll
        for (int q = 0; q < C::kQ; ++q) {
            const int f = c + q * C::kThreads;
            const float4 p4 = sp[f], m4 = sm[f], v4 = sv[f];  // lanes past len hold stale bytes, never stored
            p[4 * q] = p4.x, p[4 * q + 1] = p4.y, p[4 * q + 2] = p4.z, p[4 * q + 3] = p4.w;
            m[4 * q] = m4.x, m[4 * q + 1] = m4.y, m[4 * q + 2] = m4.z, m[4 * q + 3] = m4.w;
            v[4 * q] = v4.x, v[4 * q + 1] = v4.y, v[4 * q + 2] = v4.z, v[4 * q + 3] = v4.w;
        }
        for (uint32_t q0 = a.first[j]; q0 < a.nact; q0 += kGS, ++gc) {
            const uint32_t nst = umin((uint32_t)kGS, a.nact - q0);
            const int g = gc % kGd;
            mbar_wait(&gfull[g], (gc / kGd) & 1u);
            const uint8_t *gbp = gbuf + g * C::kChunkBytes;
            uint32_t dep = 0;
            for (uint32_t q = 0; q < nst; ++q) {
                const uint2 *gq = reinterpret_cast<const uint2 *>(gbp + q * kTile * 2);
                uint32_t gbits[4 * C::kQ];
#pragma unroll
                for (int h = 0; h < C::kQ; ++h) {
                    const uint2 g2 = gq[c + h * C::kThreads];
                    dep ^= g2.x;
                    gbits[4 * h] = g2.x & 0xFFFFu, gbits[4 * h + 1] = g2.x >> 16;
                    gbits[4 * h + 2] = g2.y & 0xFFFFu, gbits[4 * h + 3] = g2.y >> 16;
                }
                adamw_group_p2<4 * C::kQ, kUnitGs, false>(p, m, v, gbits, srec[q0 + q].f, srec2[q0 + q]);
            }
            asm volatile("" : "+r"(dep));
            __syncwarp();
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&gempty[g]);
            }
        }
#pragma unroll
        for (int q = 0; q < C::kQ; ++q) {
            const int f = c + q * C::kThreads;
            if (4u * (uint32_t)f < len) {
                sp[f] = make_float4(p[4 * q], p[4 * q + 1], p[4 * q + 2], p[4 * q + 3]);
                sm[f] = make_float4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
                sv[f] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[s]);
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


// ---- drain verification (a3): checksums of the staged sections before the copy ----
// Over the little-endian 32-bit words w_i of each section (a partial last word zero-padded):
// A = sum w_i, B = sum (i+1) w_i, both mod 2^64 (checksum_host in replay_host.cpp computes the same
// on the landed bytes). A single corrupted byte changes A; transposed words change B.
__device__ __forceinline__ void sum_pair_reduce(uint64_t a, uint64_t b, unsigned long long *out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0 && (a | b)) {
        atomicAdd(out, (unsigned long long)a);
        atomicAdd(out + 1, (unsigned long long)b);
    }
}

__global__ void __launch_bounds__(256) checksum_kernel(const ZcArgs a, unsigned long long *out) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (int s = 0; s < a.count; ++s) {
        const uint8_t *src = static_cast<const uint8_t *>(a.src[s]);
        const uint64_t bytes = a.bytes[s];
        uint64_t A = 0, B = 0;
        // the 16-byte vectors of the section (src is 16-byte aligned: slot sections 256 B, live
        // state at lo_i = a multiple of A >= 8 elements, the gradient buffer 16 B)
        const uint64_t nv = bytes >> 4;
        const uint4 *v4 = reinterpret_cast<const uint4 *>(src);
        for (uint64_t v = tid; v < nv; v += stride) {
            const uint4 q = v4[v];
            const uint64_t sw = (uint64_t)q.x + q.y + q.z + q.w;
            A += sw;
            B += (4 * v + 1) * sw + (uint64_t)q.y + 2ull * q.z + 3ull * q.w;
        }
        // tail words (bytes % 16), the last one zero-padded
        const uint64_t w0 = nv << 2, nw = (bytes + 3) >> 2;
        if (tid < nw - w0) {
            const uint64_t i = w0 + tid;
            uint32_t w = 0;
            for (uint64_t b = 0; b < 4 && 4 * i + b < bytes; ++b) w |= (uint32_t)src[4 * i + b] << (8 * b);
            A += w;
            B += (i + 1) * (uint64_t)w;
        }
        sum_pair_reduce(A, B, out + 2 * s);
    }
}

// Test hook (GCK_FAULT_FLIP): XOR one byte of device memory.
__global__ void flip_byte_kernel(uint8_t *p) { *p ^= 0x10u; }

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

__global__ void cast_bf16_kernel(const float *src, uint16_t *dst, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = (uint16_t)(pack_bf16x2(src[i], 0.f) & 0xFFFFu);
}

inline unsigned grid_for(uint64_t work_items, unsigned block, int num_sms, unsigned per_sm) {
    const uint64_t need = (work_items + block - 1) / block;
    const uint64_t cap = (uint64_t)(num_sms > 0 ? num_sms : 148) * per_sm;
    const uint64_t g = need < cap ? need : cap;
    return (unsigned)(g > 0 ? g : 1);
}

}  // namespace

template <int S, int B, int CW, int TL = 2048>
int launch_tma(const FusedArgs &a, bool pack, cudaStream_t s, int num_sms) {
    static std::atomic<uint64_t> attr_set_devices{0};  // the smem opt-in is per device
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set_devices.load() & bit)) {
        cudaFuncSetAttribute(fused_adamw_pack_tma_kernel<true, S, B, CW, TL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem(S, TL));
        cudaFuncSetAttribute(fused_adamw_pack_tma_kernel<false, S, B, CW, TL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem(S, TL));
        attr_set_devices.fetch_or(bit);
    }
    const uint64_t tiles = a.n / TL;
    const uint64_t cap = (uint64_t)(num_sms > 0 ? num_sms : 148) * B;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, cap));
    const unsigned block = (CW + 2) * 32;
    if (pack)
        fused_adamw_pack_tma_kernel<true, S, B, CW, TL><<<grid, block, tma_smem(S, TL), s>>>(a);
    else
        fused_adamw_pack_tma_kernel<false, S, B, CW, TL><<<grid, block, tma_smem(S, TL), s>>>(a);
    return (int)cudaGetLastError();
}

template <int S, int O, int CW, int TL = 2048>
int launch_tmast(const FusedArgs &a, bool pack, cudaStream_t s, int num_sms) {
    static std::atomic<uint64_t> attr_set_devices{0};  // the smem opt-in is per device
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set_devices.load() & bit)) {
        cudaFuncSetAttribute(fused_adamw_pack_tmast_kernel<true, S, O, CW, TL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, tmast_smem(S, O, TL));
        cudaFuncSetAttribute(fused_adamw_pack_tmast_kernel<false, S, O, CW, TL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, tmast_smem(S, O, TL));
        attr_set_devices.fetch_or(bit);
    }
    const uint64_t tiles = a.n / TL;
    const uint64_t cap = (uint64_t)(num_sms > 0 ? num_sms : 148);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, cap));
    const unsigned block = (CW + 3) * 32;
    if (pack)
        fused_adamw_pack_tmast_kernel<true, S, O, CW, TL><<<grid, block, tmast_smem(S, O, TL), s>>>(a);
    else
        fused_adamw_pack_tmast_kernel<false, S, O, CW, TL><<<grid, block, tmast_smem(S, O, TL), s>>>(a);
    return (int)cudaGetLastError();
}

int fused_impl_default() {
    const char *e = getenv("GCK_FUSED_IMPL");
    if (e && e[0] == 's') return 1;
    if (e && e[0] == 't') return 2;
    if (e && e[0] == 'x') return 3;
    return 0;
}

int launch_fused(const FusedArgs &a, bool pack, void *stream, int num_sms) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int impl = fused_impl_default();
    const bool aligned = ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                           reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.g)) & 15u) == 0;
    const bool out_aligned = (reinterpret_cast<uintptr_t>(a.out) & 15u) == 0;
    // default for n >= 2^18: the bulk-store variant (3 input + 3 output stages); GCK_FUSED_IMPL=t
    // selects the STG-store TMA kernel, s the plain grid-stride kernel
    if (aligned && out_aligned && (impl == 3 ? a.n >= 2048 : (impl == 0 && a.n >= kTmaMinElems))) {
        const char *e = getenv("GCK_TMAST_CFG");
        int st = 3, o = 3, cw = 16;
        if (e) sscanf(e, "%d,%d,%d", &st, &o, &cw);
        const int cfg = st * 100 + o * 10 + (cw == 8 ? 1 : 0);
        switch (cfg) {
            case 330: return launch_tmast<3, 3, 16>(a, pack, s, num_sms);
            case 340: return launch_tmast<3, 4, 16>(a, pack, s, num_sms);
            case 350: return launch_tmast<3, 5, 16>(a, pack, s, num_sms);
            case 440: return launch_tmast<4, 4, 16>(a, pack, s, num_sms);
            case 240: return launch_tmast<2, 4, 16>(a, pack, s, num_sms);
            case 420: return launch_tmast<4, 2, 16>(a, pack, s, num_sms);
            case 421: return launch_tmast<4, 2, 8>(a, pack, s, num_sms);
            case 430: return launch_tmast<4, 3, 16>(a, pack, s, num_sms);
            case 520: return launch_tmast<5, 2, 16>(a, pack, s, num_sms);
            default: return launch_tmast<3, 3, 16>(a, pack, s, num_sms);
        }
    }
    if (aligned && (impl == 2 || (impl == 0 && a.n >= kTmaMinElems))) {
        const int cfg = [] {
            const char *e = getenv("GCK_TMA_CFG");
            if (!e) return 4116;
            int st = 0, b = 0, cw = 0;
            if (sscanf(e, "%d,%d,%d", &st, &b, &cw) != 3) return 4116;
            return st * 1000 + b * 100 + cw;
        }();
        switch (cfg) {
            case 6108: return launch_tma<6, 1, 8>(a, pack, s, num_sms);
            case 6116: return launch_tma<6, 1, 16>(a, pack, s, num_sms);
            case 4116: return launch_tma<4, 1, 16>(a, pack, s, num_sms);
            case 8116: return launch_tma<8, 1, 16>(a, pack, s, num_sms);
            case 3208: return launch_tma<3, 2, 8>(a, pack, s, num_sms);
            case 3216: return launch_tma<3, 2, 16>(a, pack, s, num_sms);
            case 3108: return launch_tma<3, 1, 8>(a, pack, s, num_sms);
            case 4124: return launch_tma<4, 1, 24, 3072>(a, pack, s, num_sms);
            case 3130: return launch_tma<3, 1, 30, 3840>(a, pack, s, num_sms);
            default: return launch_tma<4, 1, 16>(a, pack, s, num_sms);
        }
    }
    const unsigned grid = grid_for(a.n >> 3, 256, num_sms, 8);
    if (pack)
        fused_adamw_pack_kernel<true><<<grid, 256, 0, s>>>(a);
    else
        fused_adamw_pack_kernel<false><<<grid, 256, 0, s>>>(a);
    return (int)cudaGetLastError();
}

// replay_kernel's preconditions: every stale part boundary a multiple of 8 elements (plans from
// plan_parts always qualify: A % 8 == 0) and 16-byte aligned arrays; else replay_generic_kernel.
static bool replay_plan(const ReplayArgs &a, ReplayPlan *rp, bool *unit_gs) {
    uintptr_t al = reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                   reinterpret_cast<uintptr_t>(a.v);
    std::memset(rp, 0, sizeof(*rp));
    rp->p = a.p;
    rp->m = a.m;
    rp->v = a.v;
    rp->n_replay = a.n_replay;
    rp->neg_zero = -0.0f;
    *unit_gs = true;
    for (uint32_t i = 0; i + 1 < a.K; ++i) {
        if ((a.lo[i] | a.hi[i]) & 7u) return false;
        al |= reinterpret_cast<uintptr_t>(a.glog[i]);
        rp->hi[i] = a.hi[i];
        if (a.rec[i].skip) continue;
        rp->glog[rp->nact] = a.glog[i];
        rp->rec[rp->nact] = a.rec[i];
        *unit_gs = *unit_gs && a.rec[i].gs == 1.0f;
        rp->nact++;
    }
    {  // first[j]: the first compacted record with original index >= j (compaction keeps the order)
        uint32_t q = 0, idx[GCK_K_LIMIT];
        for (uint32_t i = 0, c = 0; i + 1 < a.K; ++i)
            if (!a.rec[i].skip) idx[c++] = i;
        for (uint32_t j = 0; j + 1 < a.K; ++j) {
            while (q < rp->nact && idx[q] < j) ++q;
            rp->first[j] = q;
        }
    }
    {  // mixed schedule: pair part a with part K-2-a (a+1 and K-1-a pending updates: K per pair)
        const uint32_t P = a.K - 1;
        uint64_t u = 0;
        rp->nseg = 0;
        for (uint32_t x = 0, y = P - 1; x <= y && P; ++x, --y) {
            const uint32_t s = rp->nseg++;
            auto units = [&](uint32_t jj) -> uint64_t {
                if (rp->first[jj] >= rp->nact) return 0;
                const uint64_t lo = jj ? a.hi[jj - 1] : 0;
                return ((a.hi[jj] - lo) / 8 + 31) / 32;
            };
            rp->seg_a[s] = x;
            rp->seg_b[s] = y;
            rp->seg_na[s] = (uint32_t)units(x);
            rp->seg_nb[s] = x == y ? 0 : (uint32_t)units(y);
            rp->seg_u0[s] = u;
            u += rp->seg_na[s] + rp->seg_nb[s];
            if (y == 0) break;
        }
        rp->seg_u0[rp->nseg] = u;
    }
    const char *e = getenv("GCK_REPLAY_IMPL");
    return (al & 15u) == 0 && !(e && e[0] == 's');
}

template <int kTile, int kCW, int kS, int kGd, int kGS>
int launch_replay_tma(const ReplayPlan &rp, bool unit_gs, cudaStream_t s, int num_sms) {
    using C = ReplayTma<kTile, kCW, kS, kGd, kGS>;
    static std::atomic<uint64_t> attr_set_devices{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set_devices.load() & bit)) {
        cudaFuncSetAttribute(replay_tma_kernel<kTile, kCW, kS, kGd, kGS, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem());
        cudaFuncSetAttribute(replay_tma_kernel<kTile, kCW, kS, kGd, kGS, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem());
        attr_set_devices.fetch_or(bit);
    }
    uint64_t tiles = 0, lo = 0;
    for (uint32_t j = 0; lo < rp.n_replay; ++j) {
        if (rp.first[j] < rp.nact) tiles += (rp.hi[j] - lo + kTile - 1) / kTile;
        lo = rp.hi[j];
    }
    if (!tiles) return 0;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, num_sms > 0 ? num_sms : 148));
    if (unit_gs)
        replay_tma_kernel<kTile, kCW, kS, kGd, kGS, true><<<grid, (kCW + 2) * 32, C::smem(), s>>>(rp);
    else
        replay_tma_kernel<kTile, kCW, kS, kGd, kGS, false><<<grid, (kCW + 2) * 32, C::smem(), s>>>(rp);
    return (int)cudaGetLastError();
}

// the host mirror of to_recf's `fast` test for every record of the plan (kAllFast)
static bool all_fast(const ReplayPlan &rp) {
    for (uint32_t q = 0; q < rp.nact; ++q) {
        const gck_step_record &r = rp.rec[q];
        if (!(r.bc1 >= 9.5367431640625e-07f && r.bc1 <= 1.0f && r.bc2 >= 9.5367431640625e-07f && r.bc2 <= 1.0f &&
              r.eps >= 0.0f && r.eps <= 1.0f))
            return false;
    }
    return true;
}

template <bool U, bool F, bool P, int B>
int launch_replay3_b(const ReplayPlan &rp, cudaStream_t s, int num_sms) {
    const int smem = P ? 6 * 16 * 256 : 0;  // 24 KiB: below the 48 KiB default, no opt-in needed
    replay3_kernel<U, F, P, B><<<grid_for(rp.n_replay >> 3, 256, num_sms, B), 256, smem, s>>>(rp);
    return (int)cudaGetLastError();
}

template <bool U, bool F, bool P>
int launch_replay3_t(const ReplayPlan &rp, cudaStream_t s, int num_sms) {
    const char *e = getenv("GCK_REPLAY_MINB");
    return (e && e[0] == '4') ? launch_replay3_b<U, F, P, 4>(rp, s, num_sms) : launch_replay3_b<U, F, P, 3>(rp, s, num_sms);
}

static int launch_replay3(const ReplayPlan &rp, bool unit_gs, bool fast, bool pref_state, cudaStream_t s,
                          int num_sms) {
    const int sel = (unit_gs ? 4 : 0) | (fast ? 2 : 0) | (pref_state ? 1 : 0);
    switch (sel) {
        case 7: return launch_replay3_t<true, true, true>(rp, s, num_sms);
        case 6: return launch_replay3_t<true, true, false>(rp, s, num_sms);
        case 5: return launch_replay3_t<true, false, true>(rp, s, num_sms);
        case 4: return launch_replay3_t<true, false, false>(rp, s, num_sms);
        case 3: return launch_replay3_t<false, true, true>(rp, s, num_sms);
        case 2: return launch_replay3_t<false, true, false>(rp, s, num_sms);
        case 1: return launch_replay3_t<false, false, true>(rp, s, num_sms);
        default: return launch_replay3_t<false, false, false>(rp, s, num_sms);
    }
}

template <int D>
int launch_replay_ring(const ReplayPlan &rp, bool unit_gs, cudaStream_t s, int num_sms) {
    static std::atomic<uint64_t> attr_set_devices{0};  // the smem opt-in is per device
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    const int smem = ReplayRing<D>::smem(256);
    if (!(attr_set_devices.load() & bit)) {
        cudaFuncSetAttribute(replay_ring_kernel<true, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(replay_ring_kernel<false, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_set_devices.fetch_or(bit);
    }
    const unsigned grid = grid_for(rp.n_replay >> 3, 256, num_sms, 4);
    if (unit_gs)
        replay_ring_kernel<true, D><<<grid, 256, smem, s>>>(rp);
    else
        replay_ring_kernel<false, D><<<grid, 256, smem, s>>>(rp);
    return (int)cudaGetLastError();
}

int launch_replay(const ReplayArgs &a, void *stream, int num_sms) {
    if (a.n_replay == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ReplayPlan rp;
    bool unit_gs = false;
    if (replay_plan(a, &rp, &unit_gs)) {
        const char *e = getenv("GCK_REPLAY_IMPL");
        if (e && (e[0] == '5' || e[0] == '6')) {  // packed, more resident CTAs (fewer registers)
            const int mb = e[0] - '0';
            const unsigned grid = grid_for(a.n_replay >> 3, 256, num_sms, mb);
            if (mb == 5) {
                if (unit_gs) replay_kernel<true, true, true, 5><<<grid, 256, 0, s>>>(rp);
                else replay_kernel<false, true, true, 5><<<grid, 256, 0, s>>>(rp);
            } else {
                if (unit_gs) replay_kernel<true, true, true, 6><<<grid, 256, 0, s>>>(rp);
                else replay_kernel<false, true, true, 6><<<grid, 256, 0, s>>>(rp);
            }
            return (int)cudaGetLastError();
        }
        if (e && e[0] == 'x') {  // packed, heavy/light parts interleaved per 32-group unit
            const unsigned grid = grid_for(a.n_replay >> 3, 256, num_sms, 8);
            if (unit_gs) replay_kernel<true, true, true, 4, true><<<grid, 256, 0, s>>>(rp);
            else replay_kernel<false, true, true, 4, true><<<grid, 256, 0, s>>>(rp);
            return (int)cudaGetLastError();
        }
        if (e && e[0] == 'q') {  // packed, grid = 4 resident CTAs per SM exactly
            const unsigned grid = grid_for(a.n_replay >> 3, 256, num_sms, 4);
            if (unit_gs) replay_kernel<true, true, true><<<grid, 256, 0, s>>>(rp);
            else replay_kernel<false, true, true><<<grid, 256, 0, s>>>(rp);
            return (int)cudaGetLastError();
        }
        if (!e || e[0] == 'p' || e[0] == 'r') {  // default: packed pairs; 'r': scalar arithmetic
            const bool packed = !(e && e[0] == 'r');
            const unsigned grid = grid_for(a.n_replay >> 3, 256, num_sms, 8);
            const int sel = (unit_gs ? 4 : 0) | (all_fast(rp) ? 2 : 0) | (packed ? 1 : 0);
            switch (sel) {
                case 7: replay_kernel<true, true, true><<<grid, 256, 0, s>>>(rp); break;
                case 6: replay_kernel<true, true, false><<<grid, 256, 0, s>>>(rp); break;
                case 5: replay_kernel<true, false, true><<<grid, 256, 0, s>>>(rp); break;
                case 4: replay_kernel<true, false, false><<<grid, 256, 0, s>>>(rp); break;
                case 3: replay_kernel<false, true, true><<<grid, 256, 0, s>>>(rp); break;
                case 2: replay_kernel<false, true, false><<<grid, 256, 0, s>>>(rp); break;
                case 1: replay_kernel<false, false, true><<<grid, 256, 0, s>>>(rp); break;
                default: replay_kernel<false, false, false><<<grid, 256, 0, s>>>(rp); break;
            }
            return (int)cudaGetLastError();
        }
        if (e && e[0] == 'b') {  // TMA-pipelined (bulk copies, producer / consumer / store warps)
            const char *t = getenv("GCK_REPLAY_TMA");
            const int cfg = t ? atoi(t) : 0;
            switch (cfg) {
                case 1: return launch_replay_tma<2048, 16, 4, 3, 8>(rp, unit_gs, s, num_sms);
                case 2: return launch_replay_tma<4096, 8, 3, 2, 4>(rp, unit_gs, s, num_sms);
                case 3: return launch_replay_tma<2048, 8, 4, 3, 8>(rp, unit_gs, s, num_sms);
                default: return launch_replay_tma<4096, 16, 3, 2, 4>(rp, unit_gs, s, num_sms);
            }
        }
        if (e && e[0] == 'c') {  // the per-thread cp.async ring (state + D gradients ahead)
            const char *dcfg = getenv("GCK_REPLAY_D");
            const int D = dcfg ? atoi(dcfg) : 3;
            return D == 2 ? launch_replay_ring<2>(rp, unit_gs, s, num_sms)
                   : D == 4 ? launch_replay_ring<4>(rp, unit_gs, s, num_sms)
                            : launch_replay_ring<3>(rp, unit_gs, s, num_sms);
        }
        const bool pref_state = !(e && e[0] == 'u');  // 'u': unrolled, state loaded at group start
        return launch_replay3(rp, unit_gs, all_fast(rp), pref_state, s, num_sms);
    }
    const unsigned grid = grid_for((a.n_replay + 7) >> 3, 256, num_sms, 8);
    replay_generic_kernel<<<grid, 256, 0, s>>>(a);
    return (int)cudaGetLastError();
}

int launch_checksum(const ZcArgs &a, unsigned long long *d_out, void *stream, int num_sms) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(unsigned long long) * 2 * a.count, s);
    if (e != cudaSuccess) return (int)e;
    uint64_t maxv = 1;
    for (int k = 0; k < a.count; ++k) maxv = std::max<uint64_t>(maxv, a.bytes[k] >> 4);
    checksum_kernel<<<grid_for(maxv, 256, num_sms, 4), 256, 0, s>>>(a, d_out);
    return (int)cudaGetLastError();
}

int launch_flip_byte(void *dev_byte, void *stream) {
    flip_byte_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint8_t *>(dev_byte));
    return (int)cudaGetLastError();
}

int launch_cast_bf16(const float *src, uint16_t *dst, uint64_t n, void *stream, int num_sms) {
    if (n == 0) return 0;
    cast_bf16_kernel<<<grid_for(n, 256, num_sms, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
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

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

template <bool PACK, int kStages, int kOut, int kCW, int kTile, bool kUnitFast = false>
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
    // drain verification folded into the pack (a.ck): each consumer checksums the pre-update words
    // it loaded that the pack stores (state words of [lo, hi), gradient words of [0, ghi)); a vector
    // of 4 words at section index k0 adds sum to A and (k0+1) sum + (w1 + 2 w2 + 3 w3) to B
    const bool ck = PACK && a.ck != nullptr;
    uint64_t ca[4] = {0, 0, 0, 0}, cb[4] = {0, 0, 0, 0};
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
        if (ck) {
            const uint64_t base = tile * kTile;
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const uint64_t e0 = base + 4 * (uint64_t)(c + q * kThreads);  // boundaries are multiples of 8
                if (e0 < a.ghi) {
                    const uint64_t sum = (uint64_t)gq[q].x + gq[q].y;
                    ca[3] += sum;
                    cb[3] += (e0 / 2 + 1) * sum + gq[q].y;
                }
                if (e0 >= a.lo && e0 < a.hi) {
                    const uint64_t k1 = e0 - a.lo + 1;
                    const float4 *vs[3] = {&pq[q], &mq[q], &vq[q]};
#pragma unroll
                    for (int sec = 0; sec < 3; ++sec) {
                        const uint32_t w0 = __float_as_uint(vs[sec]->x), w1 = __float_as_uint(vs[sec]->y),
                                       w2 = __float_as_uint(vs[sec]->z), w3 = __float_as_uint(vs[sec]->w);
                        const uint64_t sum = (uint64_t)w0 + w1 + w2 + w3;
                        ca[sec] += sum;
                        cb[sec] += k1 * sum + ((uint64_t)w1 + 2 * (uint64_t)w2 + 3 * (uint64_t)w3);
                    }
                }
            }
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
                if (kUnitFast)  // gs == 1 and the record's ranges checked on the host: min/max guard
                    adamw_group_mm<4, true, true>(p, m, v, gb, r);
                else
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
        uint64_t *ta = ca, *tb = cb;  // the tail's packed bytes join this thread's folded checksum
        for (uint64_t e = n_tiles * kTile + (uint64_t)c; e < a.n; e += kThreads) {
            float p = a.p[e], m = a.m[e], v = a.v[e];
            const uint32_t g = a.g[e];
            if (PACK) {
                if (e >= a.lo && e < a.hi) {
                    a.sp[e - a.lo] = p;
                    a.sm[e - a.lo] = m;
                    a.sv[e - a.lo] = v;
                    const uint64_t w1 = e - a.lo + 1;
                    const uint32_t ws[3] = {__float_as_uint(p), __float_as_uint(m), __float_as_uint(v)};
#pragma unroll
                    for (int sec = 0; sec < 3; ++sec) {
                        ta[sec] += ws[sec];
                        tb[sec] += w1 * ws[sec];
                    }
                }
                if (e < a.ghi) {
                    a.sg[e] = (uint16_t)g;
                    const uint64_t half = (uint64_t)g << (16 * (e & 1));  // this element's share of word e/2
                    ta[3] += half;
                    tb[3] += (e / 2 + 1) * half;
                }
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
    if (ck) {
#pragma unroll
        for (int sec = 0; sec < 4; ++sec) {
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                ca[sec] += __shfl_xor_sync(0xFFFFFFFFu, ca[sec], d);
                cb[sec] += __shfl_xor_sync(0xFFFFFFFFu, cb[sec], d);
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int sec = 0; sec < 4; ++sec) {
                if (ca[sec] | cb[sec]) {
                    atomicAdd(a.ck + 2 * sec, (unsigned long long)ca[sec]);
                    atomicAdd(a.ck + 2 * sec + 1, (unsigned long long)cb[sec]);
                }
            }
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
template <bool kUnitGs, bool kAllFast>
__global__ void __launch_bounds__(256) replay_kernel(const ReplayPlan a) {
    __shared__ RecP srec[GCK_K_LIMIT];
    for (uint32_t q = threadIdx.x; q < a.nact; q += blockDim.x) srec[q].f = to_recf(a.rec[q]);
    __syncthreads();
    const uint64_t ngroups = a.n_replay >> 3;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t j = 0;
    for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
        const uint64_t e = gi << 3;
        while (e >= a.hi[j]) ++j;  // e only grows: amortised O(1)
        const uint32_t q0 = a.first[j];
        if (q0 >= a.nact) continue;  // every pending update of this part was skipped: already S(T)
        Vec8 p = ld8(a.p + e), m = ld8(a.m + e), v = ld8(a.v + e);
        uint4 gnext = *reinterpret_cast<const uint4 *>(a.glog[q0] + e);
        for (uint32_t q = q0; q < a.nact; ++q) {
            const uint4 gq = gnext;
            if (q + 1 < a.nact) gnext = *reinterpret_cast<const uint4 *>(a.glog[q + 1] + e);
            const uint32_t gb[8] = {gq.x & 0xFFFFu, gq.x >> 16, gq.y & 0xFFFFu, gq.y >> 16,
                                    gq.z & 0xFFFFu, gq.z >> 16, gq.w & 0xFFFFu, gq.w >> 16};
            adamw_group_mm<8, kUnitGs, kAllFast>(p.x, m.x, v.x, gb, srec[q].f);
        }
        st8(a.p + e, p);
        st8(a.m + e, m);
        st8(a.v + e, v);
    }
}

// a5 GPU replay, default when every stale part boundary is a multiple of 256 elements (plan_parts'
// default A = 1024): replay_kernel with warp-coalesced 16-B accesses — a warp owns 256 consecutive
// elements and lane l takes elements 4l..4l+3 and 128+4l..128+4l+3, so each LDG/STG.128 of the warp
// covers 512 contiguous bytes (replay_kernel's 8-consecutive-element threads touch every 32-B sector
// twice, half of it each time: 1.6x the L1 sector lookups, more long-scoreboard waits). 2-3% faster
// (GPT-2/K=8 645 vs 661 us, K=4 432 vs 447-466 us; ncu L1 load sectors 68M = the algorithmic bytes).
template <bool kUnitGs, bool kAllFast, int kBlk>
__global__ void __launch_bounds__(kBlk, 1024 / kBlk) replay_coalesced_kernel(const ReplayPlan a) {
    __shared__ RecP srec[GCK_K_LIMIT];
    for (uint32_t q = threadIdx.x; q < a.nact; q += blockDim.x) srec[q].f = to_recf(a.rec[q]);
    __syncthreads();
    const uint64_t nunits = a.n_replay >> 8;  // 256-element warp units
    const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t j = 0;
    for (uint64_t u = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nunits; u += wstride) {
        const uint64_t base = u << 8;
        while (base >= a.hi[j]) ++j;
        const uint32_t q0 = a.first[j];
        if (q0 >= a.nact) continue;
        const uint64_t e0 = base + 4 * lane, e1 = e0 + 128;
        float p[8], m[8], v[8];
        {
            const float4 a0 = *reinterpret_cast<const float4 *>(a.p + e0), a1 = *reinterpret_cast<const float4 *>(a.p + e1);
            const float4 b0 = *reinterpret_cast<const float4 *>(a.m + e0), b1 = *reinterpret_cast<const float4 *>(a.m + e1);
            const float4 c0 = *reinterpret_cast<const float4 *>(a.v + e0), c1 = *reinterpret_cast<const float4 *>(a.v + e1);
            p[0] = a0.x, p[1] = a0.y, p[2] = a0.z, p[3] = a0.w, p[4] = a1.x, p[5] = a1.y, p[6] = a1.z, p[7] = a1.w;
            m[0] = b0.x, m[1] = b0.y, m[2] = b0.z, m[3] = b0.w, m[4] = b1.x, m[5] = b1.y, m[6] = b1.z, m[7] = b1.w;
            v[0] = c0.x, v[1] = c0.y, v[2] = c0.z, v[3] = c0.w, v[4] = c1.x, v[5] = c1.y, v[6] = c1.z, v[7] = c1.w;
        }
        uint2 n0 = *reinterpret_cast<const uint2 *>(a.glog[q0] + e0), n1 = *reinterpret_cast<const uint2 *>(a.glog[q0] + e1);
        for (uint32_t q = q0; q < a.nact; ++q) {
            const uint2 g0 = n0, g1 = n1;
            if (q + 1 < a.nact) {
                n0 = *reinterpret_cast<const uint2 *>(a.glog[q + 1] + e0);
                n1 = *reinterpret_cast<const uint2 *>(a.glog[q + 1] + e1);
            }
            const uint32_t gb[8] = {g0.x & 0xFFFFu, g0.x >> 16, g0.y & 0xFFFFu, g0.y >> 16,
                                    g1.x & 0xFFFFu, g1.x >> 16, g1.y & 0xFFFFu, g1.y >> 16};
            adamw_group_mm<8, kUnitGs, kAllFast>(p, m, v, gb, srec[q].f);
        }
        *reinterpret_cast<float4 *>(a.p + e0) = make_float4(p[0], p[1], p[2], p[3]);
        *reinterpret_cast<float4 *>(a.p + e1) = make_float4(p[4], p[5], p[6], p[7]);
        *reinterpret_cast<float4 *>(a.m + e0) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4 *>(a.m + e1) = make_float4(m[4], m[5], m[6], m[7]);
        *reinterpret_cast<float4 *>(a.v + e0) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4 *>(a.v + e1) = make_float4(v[4], v[5], v[6], v[7]);
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
    const gck_step_record &r = a.rec;  // host mirror of to_recf's range test + unit grad_scale
    const bool unit_fast = r.gs == 1.0f && r.bc1 >= 9.5367431640625e-07f && r.bc1 <= 1.0f &&
                           r.bc2 >= 9.5367431640625e-07f && r.bc2 <= 1.0f && r.eps >= 0.0f && r.eps <= 1.0f &&
                           !(getenv("GCK_FUSED_GUARD") && getenv("GCK_FUSED_GUARD")[0] == 'g');
    if (unit_fast && S == 3 && O == 3 && CW == 16) {
        static std::atomic<uint64_t> attr2{0};
        if (!(attr2.load() & bit)) {
            cudaFuncSetAttribute(fused_adamw_pack_tmast_kernel<true, S, O, CW, TL, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, tmast_smem(S, O, TL));
            cudaFuncSetAttribute(fused_adamw_pack_tmast_kernel<false, S, O, CW, TL, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, tmast_smem(S, O, TL));
            attr2.fetch_or(bit);
        }
        if (pack)
            fused_adamw_pack_tmast_kernel<true, S, O, CW, TL, true><<<grid, block, tmast_smem(S, O, TL), s>>>(a);
        else
            fused_adamw_pack_tmast_kernel<false, S, O, CW, TL, true><<<grid, block, tmast_smem(S, O, TL), s>>>(a);
        return (int)cudaGetLastError();
    }
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

int launch_fused(const FusedArgs &a, bool pack, void *stream, int num_sms, bool *ck_folded) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (ck_folded) *ck_folded = false;
    const int impl = fused_impl_default();
    const bool aligned = ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                           reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.g)) & 15u) == 0;
    const bool out_aligned = (reinterpret_cast<uintptr_t>(a.out) & 15u) == 0;
    // default for n >= 2^18: the bulk-store variant (3 input + 3 output stages); GCK_FUSED_IMPL=t
    // selects the STG-store TMA kernel, s the plain grid-stride kernel
    if (aligned && out_aligned && (impl == 3 ? a.n >= 2048 : (impl == 0 && a.n >= kTmaMinElems))) {
        if (ck_folded) *ck_folded = pack && a.ck != nullptr;
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
    const char *e = getenv("GCK_REPLAY_IMPL");
    return (al & 15u) == 0 && !(e && e[0] == 's');
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

int launch_replay(const ReplayArgs &a, void *stream, int num_sms) {
    if (a.n_replay == 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ReplayPlan rp;
    bool unit_gs = false;
    if (replay_plan(a, &rp, &unit_gs)) {
        // 64 CTAs per SM of 256 threads (~5 grid-stride iterations per thread at GPT-2 size; the
        // coalesced kernel runs the same threads as 128-thread CTAs, below): the CTA scheduler then
        // keeps starting fresh CTAs on every SM while others are still on earlier parts, which mixes
        // the FP-heavy first parts with the HBM-heavy last parts on each SM (r02_replay11.jsonl: 8 per SM
        // 644 us, 16: 618, 64: 611 at GPT-2/K=8; K=4 444 -> 408 us; one wave (4): 695 us)
        const char *w = getenv("GCK_REPLAY_CTAS_PER_SM");  // experiment knob
        const unsigned grid = grid_for(a.n_replay >> 3, 256, num_sms, w ? (unsigned)atoi(w) : 64);
        bool b256 = (a.n_replay & 255u) == 0;
        for (uint32_t i = 0; i + 1 < a.K; ++i) b256 = b256 && ((a.hi[i] & 255u) == 0);
        const char *ce = getenv("GCK_REPLAY_COALESCED");  // "0": the 8-consecutive-element form
        if (b256 && !(ce && ce[0] == '0')) {
            // 128-thread CTAs, twice as many (the same threads in flight): the finer-grained CTAs let
            // the scheduler mix FP-heavy and HBM-heavy parts on an SM more evenly (GPT-2/K=8 599 vs 611 us,
            // K=4 and 7B/K=8 unchanged; r02_replay_blk*.jsonl)
            const unsigned g2 = grid * 2;
            switch ((unit_gs ? 2 : 0) | (all_fast(rp) ? 1 : 0)) {
                case 3: replay_coalesced_kernel<true, true, 128><<<g2, 128, 0, s>>>(rp); break;
                case 2: replay_coalesced_kernel<true, false, 128><<<g2, 128, 0, s>>>(rp); break;
                case 1: replay_coalesced_kernel<false, true, 128><<<g2, 128, 0, s>>>(rp); break;
                default: replay_coalesced_kernel<false, false, 128><<<g2, 128, 0, s>>>(rp); break;
            }
            return (int)cudaGetLastError();
        }
        switch ((unit_gs ? 2 : 0) | (all_fast(rp) ? 1 : 0)) {
            case 3: replay_kernel<true, true><<<grid, 256, 0, s>>>(rp); break;
            case 2: replay_kernel<true, false><<<grid, 256, 0, s>>>(rp); break;
            case 1: replay_kernel<false, true><<<grid, 256, 0, s>>>(rp); break;
            default: replay_kernel<false, false><<<grid, 256, 0, s>>>(rp); break;
        }
        return (int)cudaGetLastError();
    }
    const unsigned grid = grid_for((a.n_replay + 7) >> 3, 256, num_sms, 64);
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

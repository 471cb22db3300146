// Host replay engine (a5): the CPU reconstruction phase of GoCkpt, §4.3.1
// ("we update parameters on the CPU using the AdamW optimization strategy ... we also use
// a multi-threading mechanism to update the parameters in parallel").
//
// Every stale part j < K is brought from S(t0+j-1) to S(t0+K-1) by applying updates
// t0+j .. t0+K-1 in ascending order with the recorded gradients and StepRecords. The
// per-element op sequence is the normative update, identical to the sm_100a
// kernels, so the result is bit-identical to the GPU's synchronous snapshot.
//
// Build flags that the bit-exactness depends on (see build.py): -ffp-contract=off (no FMA
// contraction), no -ffast-math, -fno-math-errno (lets GCC vectorise sqrtf; IEEE sqrt is
// unchanged). Each worker clears MXCSR.FTZ/DAZ (denormals are kept, reading R13).
//
// Traffic: the batch order streams each stale element once (load p, m, v; K-j updates
// in L1; store), i.e. 24 B + 2 B per pending step, the minimum for a batch replay.
#include <cpuid.h>
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>
#include <unistd.h>
#include <xmmintrin.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.h"

namespace gck {
namespace {

constexpr int kBlock = 1024;            // elements kept hot in L1 across the K-j updates (12 KiB)
constexpr uint64_t kTask = 1ull << 16;  // elements per scheduling task

struct Rec {
    float b1, c1, b2, c2, bc1, bc2, lr, eps, wd, gs;
};

// One update over cnt contiguous elements. The loop is vectorised (AVX-512 / AVX2 clones);
// vdivps / vsqrtps are correctly rounded, and -ffp-contract=off keeps every * and + separate.
__attribute__((target_clones("avx512f", "avx2", "default"))) void update_block(
    float *__restrict p, float *__restrict m, float *__restrict v, const uint16_t *__restrict g, int cnt,
    const Rec &r) {
    for (int e = 0; e < cnt; ++e) {
        const uint32_t bits = (uint32_t)g[e] << 16;
        float gf;
        std::memcpy(&gf, &bits, 4);
        gf = gf * r.gs;
        const float mm = (r.b1 * m[e]) + (r.c1 * gf);
        const float vv = (r.b2 * v[e]) + (r.c2 * (gf * gf));
        const float mh = mm / r.bc1;
        const float vh = vv / r.bc2;
        const float u = mh / (__builtin_sqrtf(vh) + r.eps);
        p[e] = p[e] - (r.lr * (u + (r.wd * p[e])));
        m[e] = mm;
        v[e] = vv;
    }
}

// Partial checksum of cnt 32-bit words with local indices 0..cnt-1 (see checksum_host):
// A = sum w_k, B = sum (k+1) w_k, mod 2^64. Computed without multiplies in the loop: 8 interleaved
// Fletcher lanes (lane l takes words l, l+8, ...: a_l += w; b_l += a_l, so after M words
// b_l = sum_m (M - m) w_{l+8m}), combined exactly at the end:
// B = sum_l [(l+1) a_l + 8 (M a_l - b_l)]  (all mod 2^64), plus the scalar tail.
__attribute__((target_clones("avx512f", "avx2", "default"))) void sum_words(const uint32_t *__restrict w,
                                                                         uint32_t cnt, uint64_t *a, uint64_t *b) {
    constexpr int L = 8;
    uint64_t la[L] = {0}, lb[L] = {0};
    const uint32_t M = cnt / L;
    for (uint32_t mm = 0; mm < M; ++mm) {
        const uint32_t *q = w + (uint64_t)mm * L;
        for (int l = 0; l < L; ++l) {
            la[l] += q[l];
            lb[l] += la[l];
        }
    }
    uint64_t A = 0, B = 0;
    for (int l = 0; l < L; ++l) {
        A += la[l];
        B += (uint64_t)(l + 1) * la[l] + (uint64_t)L * ((uint64_t)M * la[l] - lb[l]);
    }
    for (uint32_t k = M * L; k < cnt; ++k) {
        A += w[k];
        B += (uint64_t)(k + 1) * w[k];
    }
    *a = A;
    *b = B;
}

struct Task {
    uint32_t j;  // 0-based part index
    uint64_t a, b;
};

void clear_ftz_daz() {
    // MXCSR bits: 15 = FTZ, 6 = DAZ; rounding control 13-14 = 00 (nearest)
    unsigned csr = _mm_getcsr();
    csr &= ~((1u << 15) | (1u << 6) | (3u << 13));
    _mm_setcsr(csr);
}

bool cpu_has_clflushopt() {
    unsigned a = 0, b = 0, c = 0, d = 0;
    return __get_cpuid_count(7, 0, &a, &b, &c, &d) && (b & (1u << 23));
}

__attribute__((target("clflushopt"))) void flush_opt(const char *a, const char *e) {
    for (; a < e; a += 64) _mm_clflushopt(const_cast<char *>(a));
}

void flush_plain(const char *a, const char *e) {
    for (; a < e; a += 64) _mm_clflush(a);
}

}  // namespace

uint64_t evict_budget() {
    static const uint64_t budget = [] {
        if (const char *e = getenv("GCK_EVICT_BYTES")) return (uint64_t)strtoull(e, nullptr, 10);
        // the private caches that can hold arena lines are those of the cores this process may run on
        // (its affinity mask: on a multi-GPU host each rank's replay threads are bound to a subset)
        const long l2 = sysconf(_SC_LEVEL2_CACHE_SIZE), l3 = sysconf(_SC_LEVEL3_CACHE_SIZE);
        const long cpus = default_threads();
        uint64_t cached = (l2 > 0 && cpus > 0 ? (uint64_t)l2 * (uint64_t)cpus : 0) + (l3 > 0 ? (uint64_t)l3 : 0);
        if (cached == 0) cached = 128ull << 20;  // sysconf without cache data: a generous guess
        return std::max<uint64_t>(2 * cached, 16ull << 20);
    }();
    return budget;
}

void evict_lines(const void *p, uint64_t bytes) {
    static const bool opt = cpu_has_clflushopt();
    if (!bytes) return;
    const char *a = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(63));
    const char *e = static_cast<const char *>(p) + bytes;
    if (opt)
        flush_opt(a, e);
    else
        flush_plain(a, e);
}

void evict_fence() { _mm_sfence(); }

int default_threads() {
    cpu_set_t set;
    CPU_ZERO(&set);
    if (sched_getaffinity(0, sizeof(set), &set) == 0) {
        const int c = CPU_COUNT(&set);
        if (c > 0) return c;
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? (int)h : 1;
}

void checksum_host(const void *p, uint64_t bytes, uint64_t *A, uint64_t *B, int threads, const cpu_set_t *cpus) {
    const uint8_t *src = static_cast<const uint8_t *>(p);
    const uint64_t nw = bytes >> 2;
    constexpr uint64_t kChunk = 1ull << 20;  // words per task (4 MiB: enough tasks for every thread)
    const uint64_t ntask = (nw + kChunk - 1) / kChunk;
    std::vector<uint64_t> pa(ntask, 0), pb(ntask, 0);
    std::atomic<uint64_t> next{0};
    // the chunks summed last may still be cached when the next drain DMA-writes them: evict them
    const uint64_t tail = evict_budget() / (kChunk * 4);
    const uint64_t first_evict = ntask > tail ? ntask - tail : 0;
    auto worker = [&]() {
        if (cpus) pthread_setaffinity_np(pthread_self(), sizeof(cpu_set_t), cpus);
        bool evicted = false;
        for (;;) {
            const uint64_t t = next.fetch_add(1, std::memory_order_relaxed);
            if (t >= ntask) break;
            const uint64_t w0 = t * kChunk, cnt = std::min(kChunk, nw - w0);
            uint64_t a = 0, b = 0;
            sum_words(reinterpret_cast<const uint32_t *>(src) + w0, (uint32_t)cnt, &a, &b);
            pa[t] = a;
            pb[t] = b + w0 * a;  // global weights (w0 + k + 1) = local (k + 1) + w0
            if (t >= first_evict) {
                evict_lines(src + 4 * w0, 4 * cnt);
                evicted = true;
            }
        }
        if (evicted) evict_fence();
    };
    if (threads <= 0) threads = cpus ? std::max(1, CPU_COUNT(cpus)) : default_threads();
    threads = (int)std::min<uint64_t>((uint64_t)threads, std::max<uint64_t>(1, ntask));
    if (threads <= 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        for (int k = 0; k < threads; ++k) pool.emplace_back(worker);
        for (auto &th : pool) th.join();
    }
    uint64_t a = 0, b = 0;
    for (uint64_t t = 0; t < ntask; ++t) {
        a += pa[t];
        b += pb[t];
    }
    if (bytes & 3) {  // partial last word, zero-padded
        uint32_t w = 0;
        for (uint64_t k = 0; k < (bytes & 3); ++k) w |= (uint32_t)src[4 * nw + k] << (8 * k);
        a += w;
        b += (nw + 1) * (uint64_t)w;
    }
    *A = a;
    *B = b;
}

gck_status replay_host_impl(const gck_step_record *recs, uint32_t K, const uint64_t *lo, const uint64_t *hi,
                            float *p, float *m, float *v, const uint16_t *const *glog, int threads,
                            int *threads_used, const cpu_set_t *cpus, ReplayChecksums *sums) {
    if (K <= 1) {
        if (threads_used) *threads_used = 0;
        return GCK_OK;
    }
    std::vector<Rec> rr(K);
    for (uint32_t i = 0; i < K; ++i)
        rr[i] = Rec{recs[i].b1, recs[i].c1, recs[i].b2, recs[i].c2, recs[i].bc1, recs[i].bc2,
                    recs[i].lr, recs[i].eps, recs[i].wd, recs[i].gs};
    // tasks, heaviest first (part j carries K-1-j pending updates)
    std::vector<Task> tasks;
    for (uint32_t j = 0; j + 1 < K; ++j)
        for (uint64_t a = lo[j]; a < hi[j]; a += kTask) tasks.push_back(Task{j, a, std::min(hi[j], a + kTask)});
    std::stable_sort(tasks.begin(), tasks.end(), [](const Task &x, const Task &y) { return x.j < y.j; });
    if (threads <= 0) threads = cpus ? std::max(1, CPU_COUNT(cpus)) : default_threads();
    threads = (int)std::min<uint64_t>((uint64_t)threads, std::max<uint64_t>(1, tasks.size()));
    if (threads_used) *threads_used = threads;
    // the tasks processed last may still be cached when the next session's drains DMA-write the
    // same lines (state and gradient log): their blocks are evicted right after their updates
    uint64_t first_evict = tasks.size();
    for (uint64_t acc = 0, budget = evict_budget(); first_evict > 0;) {
        const Task &tk = tasks[first_evict - 1];
        acc += (tk.b - tk.a) * (12 + 2 * (uint64_t)(K - 1 - tk.j));
        if (acc > budget) break;
        --first_evict;
    }
    std::atomic<uint64_t> next{0};
    std::mutex sums_mu;
    auto worker = [&]() {
        if (cpus) pthread_setaffinity_np(pthread_self(), sizeof(cpu_set_t), cpus);  // NUMA-local
        const unsigned saved_csr = _mm_getcsr();
        clear_ftz_daz();
        bool evicted = false;
        for (;;) {
            const uint64_t t = next.fetch_add(1, std::memory_order_relaxed);
            if (t >= tasks.size()) break;
            const Task &tk = tasks[t];
            const bool evict = t >= first_evict;
            evicted = evicted || evict;
            uint64_t sa[3] = {0, 0, 0}, sb[3] = {0, 0, 0}, ga[GCK_K_LIMIT] = {}, gb[GCK_K_LIMIT] = {};
            for (uint64_t b0 = tk.a; b0 < tk.b; b0 += kBlock) {
                const int cnt = (int)std::min<uint64_t>(kBlock, tk.b - b0);
                if (sums && b0 + kBlock < tk.b) {
                    // the checksum pass below is the block's first touch and has little compute to hide
                    // DRAM latency behind: prefetch the next block's state and gradient lines now, so
                    // their misses overlap this block's updates (the replay alone needs no prefetch:
                    // its first touch is inside the update arithmetic)
                    const uint64_t b1 = b0 + kBlock, c1 = std::min<uint64_t>(kBlock, tk.b - b1);
                    for (uint64_t o = 0; o < c1 * 4; o += 64) {
                        _mm_prefetch(reinterpret_cast<const char *>(p + b1) + o, _MM_HINT_T0);
                        _mm_prefetch(reinterpret_cast<const char *>(m + b1) + o, _MM_HINT_T0);
                        _mm_prefetch(reinterpret_cast<const char *>(v + b1) + o, _MM_HINT_T0);
                    }
                    for (uint32_t i = tk.j; i + 1 < K; ++i)
                        for (uint64_t o = 0; o < c1 * 2; o += 64)
                            _mm_prefetch(reinterpret_cast<const char *>(glog[i] + b1) + o, _MM_HINT_T0);
                }
                if (sums) {  // the block's landed bytes, before the first update overwrites them (in L1)
                    const float *sec[3] = {p + b0, m + b0, v + b0};
                    const uint64_t w0 = b0 - lo[tk.j];  // word index inside the part's sections
                    for (int k = 0; k < 3; ++k) {
                        uint64_t a = 0, b = 0;
                        sum_words(reinterpret_cast<const uint32_t *>(sec[k]), (uint32_t)cnt, &a, &b);
                        sa[k] += a;
                        sb[k] += b + w0 * a;
                    }
                }
                for (uint32_t i = tk.j; i + 1 < K; ++i) {  // updates t0+j+1 .. t0+K-1 (1-based parts)
                    if (sums) {  // slice i's words [b0/2, (b0+cnt)/2), right before the update reads them
                        uint64_t a = 0, b = 0;
                        sum_words(reinterpret_cast<const uint32_t *>(glog[i] + b0), (uint32_t)cnt / 2, &a, &b);
                        ga[i] += a;
                        gb[i] += b + (b0 / 2) * a;
                    }
                    if (recs[i].skip) continue;
                    update_block(p + b0, m + b0, v + b0, glog[i] + b0, cnt, rr[i]);
                }
                if (evict) {
                    evict_lines(p + b0, 4ull * cnt);
                    evict_lines(m + b0, 4ull * cnt);
                    evict_lines(v + b0, 4ull * cnt);
                    for (uint32_t i = tk.j; i + 1 < K; ++i) evict_lines(glog[i] + b0, 2ull * cnt);
                }
            }
            if (sums) {
                std::lock_guard<std::mutex> lk(sums_mu);
                for (int k = 0; k < 3; ++k) {
                    sums->a[tk.j][k] += sa[k];
                    sums->b[tk.j][k] += sb[k];
                }
                for (uint32_t i = tk.j; i + 1 < K; ++i) {
                    sums->a[i][3] += ga[i];
                    sums->b[i][3] += gb[i];
                }
            }
        }
        if (evicted) evict_fence();
        _mm_setcsr(saved_csr);
    };
    if (threads == 1 && !cpus) {
        worker();
    } else {
        std::vector<std::thread> pool;
        pool.reserve(threads);
        for (int k = 0; k < threads; ++k) pool.emplace_back(worker);
        for (auto &th : pool) th.join();
    }
    return GCK_OK;
}

}  // namespace gck

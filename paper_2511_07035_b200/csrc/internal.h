// Internal declarations shared by the runtime (gockpt_runtime.cpp), the host
// replay (replay_host.cpp) and the sm_100a kernels (kernels.cu). Not part of the ABI.
#pragma once

#include <sched.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "gockpt.h"

namespace gck {

// Arguments of one fused AdamW(+pack) launch (a2).
struct FusedArgs {
    float *p, *m, *v;            // live state (device)
    const uint16_t *g;           // bf16 gradient (device)
    uint16_t *out;               // bf16 working copy (device, nullable)
    uint64_t n;
    gck_step_record rec;
    // pack (session steps only): pre-update [lo, hi) -> slot state, g[0:ghi) -> slot grad
    uint64_t lo, hi, ghi;
    float *sp, *sm, *sv;
    uint16_t *sg;
    // drain verification folded into the pack (nullable): (A, B) of sections master, m, v, gradient
    // at ck[2s], ck[2s+1], accumulated (zeroed by the caller) over the bytes the pack stores
    unsigned long long *ck;
};

// Arguments of one replay launch (a5, GPU).
struct ReplayArgs {
    float *p, *m, *v;
    uint64_t n_replay;                        // = hi_{K-1}: elements of parts 1..K-1
    uint32_t K;
    uint64_t lo[GCK_K_LIMIT], hi[GCK_K_LIMIT];
    const uint16_t *glog[GCK_K_LIMIT];
    gck_step_record rec[GCK_K_LIMIT];
};

// The replay kernel's compacted plan (built from ReplayArgs by launch_replay): the K-1 stale part
// ends and, in ascending order, only the non-skipped StepRecords with their gradient slices;
// part j (0-based) needs compacted records first[j] .. nact-1.
struct ReplayPlan {
    float *p, *m, *v;
    uint64_t n_replay;
    uint32_t nact, _pad;
    uint64_t hi[GCK_K_LIMIT];
    uint32_t first[GCK_K_LIMIT];
    const uint16_t *glog[GCK_K_LIMIT];
    gck_step_record rec[GCK_K_LIMIT];
};

// Up to 4 (src, dst, bytes) sections drained by the zero-copy kernel (a3 variant).
struct ZcArgs {
    const void *src[4];
    void *dst[4];
    uint64_t bytes[4];
    int count;
};

// Launchers (kernels.cu). Return the cudaError_t as int (0 = success).
// *ck_folded (nullable) = true when the launched kernel accumulated a.ck (the bulk-store kernel's
// pack warp); false when the caller still has to checksum the slot with launch_checksum.
int launch_fused(const FusedArgs &a, bool pack, void *stream, int num_sms, bool *ck_folded = nullptr);
int launch_replay(const ReplayArgs &a, void *stream, int num_sms);
int launch_zerocopy_drain(const ZcArgs &a, int ctas, void *stream);
int launch_generate(int kind, int mode, uint64_t seed, uint64_t step, uint64_t offset, uint64_t n,
                    uint32_t zero_per_256, void *out, void *stream, int num_sms);

int launch_cast_bf16(const float *src, uint16_t *dst, uint64_t n, void *stream, int num_sms);
// Drain verification: d_out[2s], d_out[2s+1] = (A, B) checksums of section s (checksum_host's
// definition), zeroed first; async on stream.
int launch_checksum(const ZcArgs &a, unsigned long long *d_out, void *stream, int num_sms);

// Persistence (persist.cpp).
// The replay log a version-2 (replay-on-restore) file carries: the session plan, its K
// StepRecords and the host gradient slices glog[i] (hi[i] elements, i < K-1).
struct ReplayLog {
    uint32_t K = 0;
    uint64_t t0 = 0;
    uint64_t lo[GCK_K_LIMIT]{}, hi[GCK_K_LIMIT]{};
    gck_step_record rec[GCK_K_LIMIT]{};
    const uint16_t *glog[GCK_K_LIMIT]{};
};
// A version-2 load that defers the replay to the caller (the GPU restore) receives the log
// here; the slices land in `buf` (buf_elems capacity, slices 128-element aligned) if it is
// large enough, else in `storage`.
struct LoadedLog {
    bool present = false;
    gck_log_header lh{};
    uint16_t *glog[GCK_K_LIMIT]{};
    uint16_t *buf = nullptr;
    uint64_t buf_elems = 0;
    std::vector<uint16_t> storage;
};
// Checks a plan (contiguous, ascending, non-empty parts covering [0, n)); "" if valid.
std::string plan_error(uint32_t K, const uint64_t *lo, const uint64_t *hi, uint64_t n);

gck_status write_checkpoint_impl(const char *path, const gck_file_header *hdr, const float *const sec[3], int threads,
                                 const char *meta_json, gck_persist_stats *stats, std::string *err,
                                 const ReplayLog *log = nullptr);
gck_status read_header_impl(const char *path, gck_file_header *out, std::string *err);
gck_status read_log_header_impl(const char *path, gck_log_header *out, std::string *err);
// defer == nullptr: a version-2 file is replayed on the host (threads) after the read.
gck_status load_checkpoint_impl(const char *path, float *const dst[3], uint64_t n, int threads, gck_file_header *hdr_out,
                                gck_persist_stats *stats, std::string *err, LoadedLog *defer = nullptr);

gck_status load_range_impl(const char *path, uint64_t offset, uint64_t count, float *const dst[3], int threads,
                           gck_file_header *hdr_out, std::string *err);

// Drain verification folded into the batch replay: the checksums (checksum_host's definition) of the
// bytes the replay reads, taken before it overwrites them — session step s = part s (0-based) state
// sections [lo_s, hi_s) of master / m / v (sections 0..2) and gradient slice s (section 3) — so the
// verification costs no extra pass over host DRAM. Sums are mod 2^64 and order-independent.
struct ReplayChecksums {
    uint64_t a[GCK_K_LIMIT][4], b[GCK_K_LIMIT][4];
};

// Host replay (replay_host.cpp). sums: optional, see ReplayChecksums (every stale part's state and
// every gradient slice is read exactly once by the batch replay, skipped records included).
gck_status replay_host_impl(const gck_step_record *recs, uint32_t K, const uint64_t *lo, const uint64_t *hi,
                            float *p, float *m, float *v, const uint16_t *const *glog, int threads,
                            int *threads_used, const cpu_set_t *cpus = nullptr, ReplayChecksums *sums = nullptr);
int default_threads();
// Drain verification (replay_host.cpp): A = sum w_i, B = sum (i+1) w_i (mod 2^64) over the
// little-endian 32-bit words of [p, p+bytes), a partial last word zero-padded.
void checksum_host(const void *p, uint64_t bytes, uint64_t *A, uint64_t *B, int threads, const cpu_set_t *cpus);

// Keeping DMA destinations out of the CPU caches (replay_host.cpp). The next session's drains
// DMA-write into the pinned arena; a line a host pass (replay, verification, persist) left in a
// core's cache turns each such write into a snoop + invalidate (+ write-back): measured on the
// B200 box, 1 MiB D2H copies into lines the replay threads had touched took 100-230 us instead of
// 22 us (profiles/r02_small_drain.txt). The host passes therefore write back and drop the lines
// of the tail of their work that can still be cached: evict_budget() bytes (2 x (all L2s + L3);
// GCK_EVICT_BYTES overrides, 0 = off), evicted with evict_lines() (clflushopt, else clflush;
// weakly ordered: evict_fence() once at the end of each thread's pass).
uint64_t evict_budget();
void evict_lines(const void *p, uint64_t bytes);
void evict_fence();

}  // namespace gck

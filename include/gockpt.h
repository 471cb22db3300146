/*
 * gockpt.h — C ABI of the B200-native GoCkpt hot path: the multi-step overlapped
 * checkpoint of GoCkpt (arXiv 2511.07035).
 *
 * Citations: "P:n" = line n of the paper's text, with its section.
 *
 * What one session computes (§4.2.1, §4.3.1): a checkpoint begun
 * after training step t0 is split into K contiguous parts P_1..P_K of the
 * fp32 optimizer shard (master params, Adam m, Adam v; §2.2). Session
 * step i = training step t0+i (i = 1..K) captures part i at version S(t0+i-1)
 * (the state before update t0+i) and, for i < K, the bf16 gradient G(t0+i)
 * restricted to parts 1..i, i.e. the prefix [0, hi_i) ("the gradients
 * corresponding to the existing checkpoints ... G_A^1 and G_AB^2"). A
 * gradient-assisted replay applies updates t0+j .. t0+K-1 to each stale part
 * j < K ("version 1 of part A ... gradients of part A computed in Steps
 * N+1 and N+2 are used to update checkpoint version 3"), so the assembled host
 * checkpoint equals the synchronous snapshot S(T), T = t0+K-1, bit for bit.
 *
 * The library IS the optimizer step: gck_submit launches the fused AdamW
 * kernel whether or not a session is active, so the update's operation order
 * is identical inside and outside sessions and identical to the host and GPU
 * replays (normative update: DESIGN.md "Normative update").
 *
 * Conventions
 *  - Every function returns gck_status; nothing throws or aborts across the
 *    ABI. gck_last_error(ctx) gives a text for the last failure on ctx
 *    (thread-local text for the stateless helpers: gck_last_error(NULL)).
 *  - "device" pointers are CUDA device (or managed) addresses on cfg.device;
 *    "host" pointers are ordinary process memory. Streams are passed as
 *    void* holding a cudaStream_t (NULL = the legacy default stream).
 *  - Arrays are flat and contiguous. fp32 arrays and the bf16 gradient /
 *    param arrays must be 16-byte aligned (the PyTorch caching allocator
 *    gives 512 B); a violation returns GCK_E_INVALID.
 *  - One context per (process, CUDA device, optimizer shard). A context is
 *    driven by one host thread at a time (the library's own internal
 *    threads never touch caller memory).
 */
#ifndef GOCKPT_H_
#define GOCKPT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GCK_ABI_VERSION 2u /* 2: gck_config.plan, plan arguments of ring sizing and K selection */
#define GCK_K_LIMIT 64u /* largest K a session may use */

typedef enum {
    GCK_OK = 0,
    GCK_E_INVALID = 1,    /* bad argument: K = 0 or K > ceil(n/A), NULL or misaligned pointer, n = 0 */
    GCK_E_PROTOCOL = 2,   /* call out of order: begin while a session/checkpoint is live,
                             finalize before part K, plain submit inside a session */
    GCK_E_STALE = 3,      /* submit's part/step does not match the session (part != step - t0,
                             or not the next part) */
    GCK_E_NOMEM = 4,      /* host or device allocation failed */
    GCK_E_CUDA = 5,       /* a CUDA call failed; the context is poisoned */
    GCK_E_INCOMPLETE = 6, /* a session slice never arrived; the checkpoint is discarded */
    GCK_E_ABORTED = 7,    /* the checkpoint path failed; training continues, the session is void */
    GCK_E_BUSY = 8,       /* gck_finalize_poll: the checkpoint is not consistent yet */
    GCK_E_NODEVICE = 9,   /* no CUDA device (the library never falls back to the CPU) */
    GCK_E_IO = 10,        /* persistence: a file operation failed (errno text in gck_last_error) */
    GCK_E_CORRUPT = 11    /* persistence: bad magic/version, header/table/data CRC mismatch, truncation */
} gck_status;

typedef struct gck_ctx gck_ctx;

/* AdamW hyperparameters, binary64; every binary32 scalar the update uses is
 * derived from these once per step (reading R7). */
typedef struct {
    double beta1, beta2, eps, weight_decay;
} gck_hparams;

enum { GCK_COPY_ENGINE = 0, GCK_COPY_ZEROCOPY = 1 };
enum { GCK_REPLAY_HOST = 0, GCK_REPLAY_GPU = 1, GCK_REPLAY_DEFERRED = 2, GCK_REPLAY_STREAM = 3 };
enum { GCK_STAGE_RING = 0, GCK_STAGE_DIRECT = 1, GCK_STAGE_BLOCKING = 2 };
/* Partition plans (a1). EQUAL: K parts of equal size over A-element units, remainder to the earliest
 * parts (R11). BALANCED (ours, R17; the paper leaves the part sizes
 * open): the contiguous unit-aligned parts that minimise the largest per-step transfer
 * V_max = max_i 12|P_i| + 2 hi_i [i<K] — early parts larger, later ones smaller — kept only when it
 * beats EQUAL; V_max 2.42n vs 3.25n at K = 8. The checkpoint S(T) is the same under either plan. */
enum { GCK_PLAN_EQUAL = 0, GCK_PLAN_BALANCED = 1 };

typedef struct {
    uint32_t abi_version;   /* must be GCK_ABI_VERSION */
    int32_t device;         /* CUDA device ordinal the tensors live on */
    uint64_t n;             /* elements in this rank's optimizer shard (ZeRO-1, §4.5) */
    uint32_t k_min, k_max;  /* session K range; sizes the HBM ring and pinned arena (1..GCK_K_LIMIT) */
    uint32_t part_align;    /* A: partition boundaries are multiples of A elements (0 -> 1024; must be
                               a multiple of 8) */
    uint32_t ring_slots;    /* R: HBM staging slots, 1 or 2 (0 -> 2); R=2 double-buffers so one
                               slot drains while the next step packs (§4.4.1) */
    int32_t copy_mode;      /* GCK_COPY_ENGINE (cudaMemcpyAsync on a side stream) or GCK_COPY_ZEROCOPY
                               (SM stores into mapped pinned memory) */
    uint64_t chunk_bytes;   /* copy-engine chunk size (0 = one copy per section); P:362 uses 4 MiB */
    uint32_t zc_ctas;       /* CTAs of the zero-copy drain kernel (0 -> 32) */
    int32_t replay_mode;    /* GCK_REPLAY_HOST: the host thread pool replays in place;
                               GCK_REPLAY_GPU: the stale parts + gradient log go back up to HBM, the
                               replay kernel runs there, the consistent parts come back (no host
                               arithmetic; library-owned device scratch allocated on first use);
                               GCK_REPLAY_DEFERRED (replay-on-restore): finalize
                               does no replay — the handle holds the captured parts (replay_pending = 1),
                               gck_persist_begin writes them with the gradient log and StepRecords
                               (file version 2), and the replay runs at load time: on the GPU inside
                               gck_restore, on the host inside gck_load_checkpoint(_range);
                               GCK_REPLAY_STREAM (streaming host replay):
                               a library thread started at begin applies update t0+i to the prefix
                               [0, hi_i) as soon as slice i has drained (parts 1..i are then all at
                               S(t0+i)), so the gradient log is a ring of stream_buffers slices of n
                               elements (pinned arena 12n + 2n*B bytes instead of 12n + n(K-1));
                               gck_submit blocks (host) before reusing a slice buffer whose update has
                               not been applied yet. Same per-element op order as the batch replay.
                               Always eager; gck_get_staged / gck_replay_gpu are PROTOCOL errors */
    int32_t replay_threads; /* host replay threads (0 -> all cores of the affinity mask) */
    int32_t timing;         /* 1: record CUDA events for stall / kernel / D2H times (gck_stats) */
    int32_t eager_replay;   /* 1: replay starts on a library thread as soon as the gradient log is
                               complete (overlaps training); 0: replay runs inside gck_finalize
                               (lets tests read the staged bytes first) */
    int32_t staging;        /* GCK_STAGE_RING: the fused kernel packs part i + G[0:hi_i] into an HBM
                               ring slot (no transfer deadline on the compute stream but slot reuse).
                               GCK_STAGE_DIRECT (GoCkpt-O literal; NEXT-2): no ring — part
                               i is copied from the live arrays while step t0+i's F/B runs (the update
                               waits for it) and G(t0+i)[0:hi_i] from the caller's gradient buffer,
                               which the caller must not overwrite before gck_grad_fence.
                               GCK_STAGE_BLOCKING: the paper-faithful GoCkpt — as DIRECT,
                               but each update also waits until its gradient slice is on the host
                               (NEXT-3 comparison scheme). */
    int32_t numa_node;      /* host placement of the pinned arena and of the replay/persist threads:
                               >= 0 binds them to that NUMA node; -1 = the GPU's own node (from its PCI
                               address; no binding if the platform reports none); -2 = no binding.
                               P:401: "28 cores per process, same NUMA domain". */
    uint32_t stream_buffers; /* GCK_REPLAY_STREAM: gradient slice buffers B (0 -> min(4, k_max - 1)); ignored
                                otherwise */
    int32_t verify_drain;   /* 1: verify every drained slice (a3) — the device checksums the staged bytes (ring
                               staging with the bulk-store fused kernel: folded into the pack, from the words
                               the kernel stores; otherwise a checksum kernel reads each section on the D2H
                               stream right before its copy), the host
                               recomputes the checksum of the landed bytes before the replay uses them
                               (A = sum w_i, B = sum (i+1) w_i mod 2^64 over 32-bit words); a mismatch
                               voids the session with GCK_E_CORRUPT. 0: no verification */
    int32_t plan;           /* GCK_PLAN_EQUAL (0) or GCK_PLAN_BALANCED: the partition plan of every session;
                               also sizes the ring and the gradient log */
} gck_config;

/* Caller-owned device tensors (PyTorch owns them; they must outlive the context). */
typedef struct {
    float *master;          /* fp32[n] master params (device) */
    float *exp_avg;         /* fp32[n] Adam m (device) */
    float *exp_avg_sq;      /* fp32[n] Adam v (device) */
    uint16_t *param_bf16;   /* bf16[n] working params written as RNE(master') (device; NULL = skip) */
    void *ring;             /* optional caller-owned HBM staging ring (device, 256-B aligned; NULL = the
                               library allocates it); ring staging only */
    uint64_t ring_bytes;    /* its capacity; must be >= gck_ring_bytes_required(...) */
} gck_tensors;

/* One training step's update (§2.1: update N consumes G^N). */
typedef struct {
    uint64_t step;              /* training-step index s of this update */
    uint64_t adam_t;            /* bias-correction count t(s) >= 1 (non-skipped updates up to s) */
    double lr;                  /* learning rate of this step (schedule applied by the caller) */
    double grad_scale;          /* multiplies the gradient (loss-scale unscale x clip coefficient; 1.0) */
    int32_t skip;               /* 1: update skipped (overflow); state unchanged */
    const uint16_t *grad_bf16;  /* bf16[n] gradient shard G(s) (device). In ring mode it only has to
                                   stay valid until the stream passes this step's kernel. */
} gck_step_args;

/* The binary32 scalars one update consumes (a0). Shared by the GPU update, the
 * host replay and the GPU replay, which is what makes them bit-identical. */
typedef struct {
    float b1, c1, b2, c2, bc1, bc2, lr, eps, wd, gs;  /* c = f32(1-beta), bc = f32(1-beta^t) */
    int32_t skip;
    uint32_t _pad;
    uint64_t t;
} gck_step_record;

/* A consistent checkpoint S(step) of this shard, in library-owned pinned host
 * memory, valid until gck_release ("the CPU retains the full checkpoint"). */
typedef struct {
    uint64_t step;              /* = T = t0 + K - 1 */
    uint64_t n;
    const float *master, *exp_avg, *exp_avg_sq;
    uint32_t K;                 /* the session's K */
    uint32_t replay_pending;    /* 1 (GCK_REPLAY_DEFERRED only): master/m/v still hold part i at
                                   S(t0+i-1); S(T) is materialised when the persisted file is loaded */
} gck_checkpoint;

/* The staged (pre-replay) host bytes of the current session, for verification:
 * part i's ranges of master/m/v hold S(t0+i-1); glog[i-1] holds G(t0+i)[0:hi_i]. */
typedef struct {
    uint64_t t0, n;
    uint32_t K, _pad;
    uint64_t lo[GCK_K_LIMIT], hi[GCK_K_LIMIT];      /* part i = [lo[i-1], hi[i-1]) */
    const float *master, *exp_avg, *exp_avg_sq;      /* host, n each */
    const uint16_t *glog[GCK_K_LIMIT];               /* host; glog[i-1] has hi[i-1] elements, i < K */
} gck_staged;

typedef struct {
    uint64_t sessions, steps, session_steps;
    uint64_t d2h_bytes;            /* bytes drained to host, all sessions */
    double stall_ms_total;         /* slot-reuse waits on the compute stream (a4), all sessions */
    double stall_ms_max;           /* largest single wait */
    double kernel_ms_total;        /* fused kernel time, timed steps */
    uint64_t kernel_launches_timed;
    double d2h_ms_total;           /* D2H stream busy time */
    double last_session_stall_ms, last_session_d2h_ms;
    double last_replay_ms;         /* host replay compute time of the last session */
    double last_worker_ms;         /* replay worker wall time: wait for the gradient log + replay + last drain */
    double last_finalize_wait_ms;  /* time gck_finalize blocked */
    uint64_t last_session_d2h_bytes;
    uint64_t gpu_launches;         /* kernels this context launched */
    int32_t replay_threads;
    int32_t numa_node;             /* node the arena and threads are bound to (-1: unbound) */
    uint32_t last_session_k;       /* K of the last begun session (K = 0 at begin: chosen automatically) */
    uint32_t _pad2;
    double auto_step_ms;           /* step time the last automatic K used (0: not measured) */
    double auto_link_gbs;          /* link rate the last automatic K used */
    double last_stream_wait_ms;    /* GCK_REPLAY_STREAM: host time gck_submit blocked on slice-buffer reuse */
    double last_verify_ms;         /* batch replay: host time of the last session's completeness check and
                                      drain verification (cfg.verify_drain) before the replay */
} gck_stats;

/* One session step of the last finalized session (gck_get_session_steps): the per-step log behind
 * the stall metric (a4) and the drain rate (a3). Times need cfg.timing (else 0). */
typedef struct {
    uint32_t part;        /* session step i (1..K) */
    uint32_t slot;        /* ring slot it packed into ((i-1) mod R); UINT32_MAX for direct staging */
    float wait_ms;        /* the slot-reuse (direct: state-copy) wait on the compute stream before the update */
    float kernel_ms;      /* the fused AdamW + pack kernel */
    float d2h_ms;         /* this step's D2H copies on the drain stream (copy-engine busy time) */
    uint32_t _pad;
    uint64_t d2h_bytes;   /* bytes this step drained: 12 |P_i| + 2 hi_i (i < K) */
} gck_session_step;

/* ---- context lifecycle -------------------------------------------------- */

/* HBM bytes the ring needs for (n, K in [k_min, k_max], A, R slots, plan): R x the largest
 * 256-B-aligned [master_i | m_i | v_i | G[0:hi_i]] slot. Host-only. 0 on invalid input. */
uint64_t gck_ring_bytes_required(uint64_t n, uint32_t k_min, uint32_t k_max, uint32_t part_align, uint32_t ring_slots,
                                 int32_t plan);

/* Validate, create the D2H stream + events, allocate the HBM staging ring
 * (R slots sized for K in [k_min, k_max]) and the pinned host arena
 * (12n checkpoint bytes + the gradient log; §4.4.2 "pre-register the
 * CPU memory used as Pinned Memory"). Errors: INVALID, NOMEM, CUDA, NODEVICE. */
gck_status gck_create(const gck_config *cfg, const gck_hparams *hp, const gck_tensors *t, gck_ctx **out);

/* Waits for outstanding work, frees everything the library owns. NULL is a no-op. */
gck_status gck_destroy(gck_ctx *ctx);

/* ---- the session (BJ: begin_checkpoint(step, K), submit, finalize) ------ */

/* Plan a session after step t0 with K parts (a1): parts balanced over
 * A-element units, remainder to the earliest parts. K = 0 picks K automatically (NEXT-4): the
 * smallest K in [k_min, k_max] whose largest per-step D2H fits in one step, from the step time
 * measured between recent submits (cfg.timing) and the link rate of previous drains
 * (gck_stats.last_session_k reports the choice). Host-only, no GPU work (direct staging also
 * enqueues part 1's copy).
 * Errors: INVALID (K outside [k_min, k_max] or > ceil(n/A)), PROTOCOL (a
 * session or an unreleased checkpoint is live). */
gck_status gck_begin_checkpoint(gck_ctx *ctx, uint64_t t0, uint32_t K);

/* Enqueue one optimizer step on `stream` (async; returns before the GPU runs).
 * part = 0: a plain step (no session active). part = i in 1..K: session step
 * i, requires args->step == t0 + i. Inside a session the compute stream first
 * waits for the slot it is about to reuse to have drained (the only stall
 * point, a4; "transmitted by blocking"), then runs the fused kernel that
 * packs part i (pre-update) and G[0:hi_i] into the slot and applies the
 * update (a2), then the D2H stream drains the slot into pinned memory (a3).
 * Errors: INVALID, PROTOCOL, STALE, CUDA (kernel launch failure poisons ctx),
 * ABORTED (the checkpoint path failed — now or earlier in this session; the update still ran
 * as a plain step, the session is void: gck_finalize reports ABORTED, gck_begin_checkpoint
 * starts a new one). Test hooks (environment, read at gck_begin_checkpoint; i = session step):
 * GCK_FAULT_DRAIN=<i> fails the drain enqueue of step i (ABORTED here); GCK_FAULT_DROP_SLICE=<i>
 * silently skips step i's drain (gck_finalize then reports INCOMPLETE); GCK_FAULT_FLIP=<i> flips
 * one landed byte of step i's state part on the host before verification (gck_finalize reports
 * CORRUPT with cfg.verify_drain, else the checkpoint differs from S(T)). */
gck_status gck_submit(gck_ctx *ctx, uint32_t part, const gck_step_args *args, void *stream);

/* Direct staging: make `stream` wait until the gradient slice of the latest session step has
 * been copied out of the caller's gradient buffer. Call before the next backward overwrites
 * that buffer ("do not overwrite the original gradient space ... until the next
 * backpropagation"). No-op in ring mode or outside sessions. */
gck_status gck_grad_fence(gck_ctx *ctx, void *stream);

/* Wait until every slot of the session has drained. Does not replay. */
gck_status gck_wait_drained(gck_ctx *ctx);

/* Pointers to the staged pre-replay bytes (after gck_wait_drained, before
 * gck_finalize). Errors: PROTOCOL if not drained or already replayed. */
gck_status gck_get_staged(gck_ctx *ctx, gck_staged *out);

/* Block until the checkpoint is consistent (drains complete, replay done, a5/a6)
 * and describe it. Before the replay uses any slice, every session step must have drained its
 * state part and gradient slice, else INCOMPLETE (a missing slice is never replayed
 * around); with cfg.verify_drain every landed section must match the checksum of the staged
 * bytes, else CORRUPT. Both void the session (state as after ABORTED: gck_release, then a new
 * gck_begin_checkpoint; training is unaffected).
 * Errors: PROTOCOL (part K not yet submitted), ABORTED, INCOMPLETE, CORRUPT. */
gck_status gck_finalize(gck_ctx *ctx, gck_checkpoint *out);

/* Non-blocking finalize: GCK_E_BUSY while drains/replay are still running. */
gck_status gck_finalize_poll(gck_ctx *ctx, gck_checkpoint *out);

/* Return the checkpoint memory to the library; the next session may begin. Also the way out of a
 * voided session (ABORTED / INCOMPLETE / CORRUPT): release then waits for the library's threads and its
 * D2H stream, so no copy of the voided session can still land in the pinned arena afterwards. */
gck_status gck_release(gck_ctx *ctx);

/* ---- references and variants -------------------------------------------- */

/* Synchronous snapshot (the reference GoCkpt must equal): D2H copy of
 * the live master/m/v, ordered after all work queued on `stream`; blocks until
 * done. h_* are host arrays of n floats. */
gck_status gck_sync_snapshot(gck_ctx *ctx, void *stream, float *h_master, float *h_m, float *h_v);

/* GPU replay of the staged session (variant of a5): uploads the staged host
 * bytes into the caller's device arrays d_* (n floats each) and a gradient
 * scratch d_glog (>= n*(K-1) bf16 elements; slices are 256-B aligned inside it), then runs the replay
 * kernel on `stream`. Same per-element op sequence as the host replay. Call
 * after gck_wait_drained and before gck_finalize. Blocks until done. */
gck_status gck_replay_gpu(gck_ctx *ctx, void *stream, float *d_master, float *d_m, float *d_v, uint16_t *d_glog);

gck_status gck_get_stats(const gck_ctx *ctx, gck_stats *out);

/* Per-step log of the last finalized session: writes min(K, cap) entries, *count = K (0 before the
 * first finalized session). Host-only. Errors: INVALID (NULL ctx/count, or out NULL with cap > 0). */
gck_status gck_get_session_steps(const gck_ctx *ctx, gck_session_step *out, uint32_t cap, uint32_t *count);
const char *gck_last_error(const gck_ctx *ctx);

/* ---- stateless building blocks (used by the context; exported for tests) */

/* a0: binary32 scalars of update t from binary64 hyperparameters; beta^t is a
 * left-to-right binary64 running product (reading R7). Host-only. */
gck_status gck_make_step_record(const gck_hparams *hp, uint64_t adam_t, double lr, double grad_scale,
                                int32_t skip, gck_step_record *out);

/* a1: the K part ranges of [0, n) with alignment A under the EQUAL plan; lo_hi[2i], lo_hi[2i+1] =
 * lo_{i+1}, hi_{i+1}. Host-only. Errors: INVALID. */
gck_status gck_plan_parts(uint64_t n, uint32_t K, uint32_t A, uint64_t *lo_hi);
/* a1 under either plan (GCK_PLAN_EQUAL / GCK_PLAN_BALANCED, R17); same layout. Host-only.
 * Errors: INVALID (n = 0, A = 0, K = 0, K > ceil(n/A), K > GCK_K_LIMIT, bad plan). */
gck_status gck_plan_parts_mode(uint64_t n, uint32_t K, uint32_t A, int32_t plan, uint64_t *lo_hi);

/* a5, host: replay a staged session in place. master/m/v: host arrays of n
 * floats holding part j at S(t0+j-1); glog[i-1]: host bf16 array of >= hi_i
 * elements (i = 1..K-1); recs[i-1]: StepRecord of update t0+i. Runs on
 * `threads` threads (0 = all cores). Host-only; usable without a GPU. Side effect on the CPU
 * caches only: the lines of the last ~2 x (L2s + L3) bytes it touched are written back and evicted
 * (clflushopt), so a following DMA into the same pinned memory does not snoop other cores' caches
 * (GCK_EVICT_BYTES=<bytes> overrides the amount, 0 = off; gck_checksum and the persist writers
 * do the same). */
gck_status gck_replay_host(const gck_step_record *recs, uint32_t K, const uint64_t *lo_hi, uint64_t n,
                           float *master, float *m, float *v, const uint16_t *const *glog, int32_t threads);

/* a5, GPU: the same replay on device arrays (d_glog[i-1] device pointers). Async on stream. */
gck_status gck_replay_device(const gck_step_record *recs, uint32_t K, const uint64_t *lo_hi, uint64_t n,
                             float *d_master, float *d_m, float *d_v, const uint16_t *const *d_glog,
                             void *stream);

/* a2 without a session: one fused AdamW step on device arrays. Async on stream. */
gck_status gck_adamw_step(const gck_step_record *rec, uint64_t n, float *d_master, float *d_m, float *d_v,
                          const uint16_t *d_grad, uint16_t *d_param_bf16, void *stream);

/* a3 without a session: copy `bytes` from device memory to pinned host memory on `stream` by
 * the drain's own mechanisms — GCK_COPY_ENGINE (cudaMemcpyAsync, in chunk_bytes pieces if
 * nonzero) or GCK_COPY_ZEROCOPY (zc_ctas CTAs of 16-B stores; dst must be mapped pinned memory,
 * both 16-B aligned). Async. Used by the host-link bandwidth sweep (BASELINE config 5). */
gck_status gck_d2h_copy(void *dst_host, const void *src_dev, uint64_t bytes, int32_t mode, uint64_t chunk_bytes,
                        uint32_t zc_ctas, void *stream);

/* a3 drain verification, host side (the definition cfg.verify_drain uses on both sides): over the
 * little-endian 32-bit words w_0..w_{W-1} of [host, host+bytes) (a partial last word zero-padded),
 * out_ab[0] = A = sum w_i, out_ab[1] = B = sum (i+1) w_i, both mod 2^64. Host-only; `threads`
 * threads (0 = all cores of the affinity mask). Errors: INVALID (NULL pointers). */
gck_status gck_checksum(const void *host, uint64_t bytes, int32_t threads, uint64_t *out_ab);

/* ---- NEXT-1: persistence and restore (§4.3.2, §4.4.1, §4.4.3) -------- */

#define GCK_FILE_MAGIC "GOCKPT\0\1"
#define GCK_FILE_VERSION 1u

/* On-disk header of one rank's checkpoint file (little-endian, the first 4096 bytes). The CRC
 * table (3 x nblocks uint32 CRC-32/zlib of each block_bytes block of master, exp_avg,
 * exp_avg_sq) starts at table_offset; sections start at section_offset[], 4096-aligned. */
typedef struct {
    char magic[8];               /* GCK_FILE_MAGIC */
    uint32_t version, header_bytes;
    uint64_t step;               /* T: the checkpoint is the state after update T */
    uint64_t adam_t;             /* bias-correction count of S(T) (resume with adam_t + 1) */
    uint64_t n;
    uint32_t rank, world;        /* ZeRO-1 shard identity */
    double beta1, beta2, eps, weight_decay;
    uint64_t block_bytes, nblocks, table_offset;
    uint64_t section_offset[3], section_bytes[3];
    uint32_t table_crc;          /* CRC-32 of the table's 3*nblocks entries */
    uint32_t header_crc;         /* CRC-32 of every header byte before this field */
} gck_file_header;

typedef struct {
    uint64_t bytes;              /* file bytes */
    double seconds;              /* wall time of the call (write: through fsync, rename, metadata, LATEST) */
    double data_seconds;         /* write: until the data + header were written (before fsync) */
    double gbs;                  /* 3 x 4n bytes / seconds / 1e9 */
    int32_t threads, _pad;
} gck_persist_stats;

/* Write a checkpoint file with `threads` writer threads (0 = min(16, cores)): data to
 * `<path>.tmp` (disjoint 64 MiB blocks, CRC per block), then CRC table + header, fsync, rename
 * to `path`, then `<path>.meta.json` (step, adam_t, n, rank, world, bytes, user JSON
 * `meta_json` or null) and `<dir>/LATEST.rank<r>` (atomic rename) — "saving this metadata
 * marks the completion of the latest checkpoint". hdr supplies step, adam_t, n, rank,
 * world and the hyperparameters; the layout fields are filled in. Host-only, blocking.
 * Errors: INVALID, IO, ABORTED (fault injection GCK_FAULT_PERSIST=<blocks>). */
gck_status gck_write_checkpoint(const char *path, const gck_file_header *hdr, const float *master, const float *m,
                                const float *v, int32_t threads, const char *meta_json, gck_persist_stats *stats);

/* Read and validate (magic, version 1 or 2, header CRC) a checkpoint file's header. Host-only. */
gck_status gck_read_header(const char *path, gck_file_header *out);

/* Read a checkpoint file into host arrays of n floats each, verifying every block CRC
 * ("first read from the SSD into CPU memory"). A version-2 file is replayed on the host
 * (`threads` threads) after the read, so the arrays receive S(T) either way. Host-only, blocking.
 * Errors: INVALID (n mismatch), IO, CORRUPT. */
gck_status gck_load_checkpoint(const char *path, uint64_t n, float *master, float *m, float *v, int32_t threads,
                               gck_file_header *out, gck_persist_stats *stats);

/* Read elements [offset, offset + count) of a checkpoint file's master / m / v into host arrays of
 * count floats; every 64 MiB block the range touches is read whole and CRC-verified. For loading
 * into a different ZeRO-1 degree: a new rank's range spans parts of old ranks' files.
 * A version-2 file also reads the gradient slices over the range and replays it (S(T)). Host-only. Errors: INVALID (range outside n), IO, CORRUPT. */
gck_status gck_load_checkpoint_range(const char *path, uint64_t offset, uint64_t count, float *master, float *m,
                                     float *v, int32_t threads, gck_file_header *out);

/* ---- NEXT-2: replay-on-restore (file version 2) ------------------------------------------
 * A version-2 file is a version-1 file whose three sections hold the session's CAPTURED parts
 * (part i = [lo_i, hi_i) at S(t0+i-1), §4.2.1) instead of S(T), followed by the replay
 * log: at offset L (= the end of a version-1 file of the same n, i.e. section_offset[2] +
 * section_bytes[2] rounded up to 4096) one gck_log_header (padded to 8192 bytes), at
 * glog_table_offset the per-block CRC-32 table of the gradient slices (glog_nblocks entries,
 * slices in order, each slice split into block_bytes blocks), and each slice i < K
 * (G(t0+i)[0:hi_i], bf16 bits, "G_A^1 and G_AB^2") at glog_offset[i-1], 4096-aligned.
 * Loading applies updates t0+j .. T to every part j < K in ascending order with rec[] — the
 * same per-element op sequence as the session replay (§4.3.1) — so the loaded state
 * is S(T) bit for bit. header.step = T and header.adam_t = t(T), as in version 1. */
#define GCK_FILE_VERSION_LOG 2u
#define GCK_LOG_MAGIC "GCKRLOG\0"
#define GCK_LOG_HEADER_BYTES 8192u

typedef struct {
    char magic[8];                          /* GCK_LOG_MAGIC */
    uint32_t K, _pad;                       /* session K, 1..GCK_K_LIMIT */
    uint64_t t0;                            /* the session began after update t0; T = t0 + K - 1 */
    uint64_t lo[GCK_K_LIMIT], hi[GCK_K_LIMIT];  /* part i = [lo[i-1], hi[i-1]); zero beyond K */
    gck_step_record rec[GCK_K_LIMIT];       /* rec[i-1] = StepRecord of update t0+i, i = 1..K */
    uint64_t glog_offset[GCK_K_LIMIT];      /* file offset of slice i (i < K; hi[i-1] bf16); else 0 */
    uint64_t glog_table_offset, glog_nblocks;
    uint32_t glog_table_crc;                /* CRC-32 of the glog_nblocks table entries */
    uint32_t log_crc;                       /* CRC-32 of every byte of this struct before this field */
} gck_log_header;

/* Write a version-2 (replay-on-restore) file: master/m/v are the captured host arrays (n floats
 * each; part i at S(t0+i-1)), lo_hi the K parts as 2K uint64 (the a1 plan: contiguous,
 * ascending, covering [0, n)), recs the K StepRecords of updates t0+1 .. t0+K, glog[i] (i < K-1)
 * the host gradient slice of update t0+i+1 with hi_{i+1} elements. Same atomic publication as
 * gck_write_checkpoint. Host-only, blocking. Errors: INVALID (K, plan or pointers), IO, ABORTED. */
gck_status gck_write_checkpoint_log(const char *path, const gck_file_header *hdr, const float *master,
                                    const float *m, const float *v, uint32_t K, uint64_t t0,
                                    const uint64_t *lo_hi, const gck_step_record *recs,
                                    const uint16_t *const *glog, int32_t threads, const char *meta_json,
                                    gck_persist_stats *stats);

/* Read and validate (magic, log CRC, plan) the replay log header of a version-2 file.
 * Errors: INVALID (a version-1 file), IO, CORRUPT. Host-only. */
gck_status gck_read_log_header(const char *path, gck_log_header *out);

/* Persist the finalized checkpoint (state READY) in the background on a library thread;
 * gck_release (and gck_destroy) wait for it, so the next session cannot begin before the
 * previous checkpoint is durable ("GoCkpt will wait for the last checkpoint").
 * With GCK_REPLAY_DEFERRED the file is version 2 (captured parts + gradient log + records). */
gck_status gck_persist_begin(gck_ctx *ctx, const char *path, uint32_t rank, uint32_t world, const char *meta_json);

/* Wait for the background persist; returns its status and stats. */
gck_status gck_persist_wait(gck_ctx *ctx, gck_persist_stats *out);

/* Restore (no session live): load `path` into the pinned arena, upload master/m/v into the
 * context's device tensors on `stream`, re-derive the bf16 working copy RNE(master), and
 * synchronize ("then transferred to GPU memory ... resumed at the step after").
 * A version-2 file's gradient slices go up to temporary device memory and the replay kernel
 * brings the stale parts to S(T) in place on the device tensors before the bf16 cast
 * (replay-on-restore: HBM-speed reconstruction, no host arithmetic). A version-2 file's K may
 * exceed the context's k_max. Before it touches the arena it joins the library's threads and waits
 * for its D2H stream. Errors: PROTOCOL, INVALID (n mismatch), IO, CORRUPT, NOMEM, CUDA. */
gck_status gck_restore(gck_ctx *ctx, const char *path, void *stream, gck_file_header *out);

/* ---- NEXT-4: analytic model (§3.1; §4.2.3) and K selection ------ */

/* P = T_ckpt/(N T_step) + p N T_step/2 + p T_load; times in seconds, p in 1/s. */
double gck_model_waste_fraction(double t_ckpt, double interval_steps, double t_step, double p_fail, double t_load);
/* N* = sqrt(2 T_ckpt / (p T_step^2)). */
double gck_model_optimal_interval(double t_ckpt, double t_step, double p_fail);
/* P* = sqrt(2 p T_ckpt) + p T_load; GPU-utilization overhead is P* / (P* + 1). */
double gck_model_optimal_waste(double t_ckpt, double p_fail, double t_load);
/* Stall of one checkpoint: Async-O (N-1) T_step; GoCkpt share*N(N-1)/2 T_step (P:320,
 * share = 1/7 in the paper's formula, 1/6 for a 12-B state + 2-B gradient, R4). */
double gck_model_stall_async_o(uint32_t N, double t_step);
double gck_model_stall_gockpt(uint32_t N, double t_step, double grad_share);
/* Smallest K in [1, k_max] whose largest per-step D2H V_max(K) (a1 plan `plan` with alignment A)
 * takes at most budget x t_step at link_gbs GB/s (SURVEY §8(d) K_min). *k_out = 0 and
 * GCK_E_INVALID if none does. v_max_bytes (nullable) receives V_max of the chosen K. */
gck_status gck_recommend_k(uint64_t n, uint32_t part_align, int32_t plan, double link_gbs, double t_step_s,
                           double budget, uint32_t k_max, uint32_t *k_out, double *v_max_bytes);

/* ---- harness-only (NOT the method): seeded synthetic inputs ------------- */

/* Fill d_out with the counter-hash generator of gockpt_inputs.py (DESIGN.md
 * "Input recipe"): kind 1 = master (mode 0 flat / 1 model), 2 = exp_avg,
 * 3 = exp_avg_sq, 4 = bf16 gradient of `step` (mode 0 uniform / 1 llm,
 * zero_per_256). Element k gets global index offset + k. Async on stream. */
gck_status gck_h_generate(int32_t kind, int32_t mode, uint64_t seed, uint64_t step, uint64_t offset,
                          uint64_t n, uint32_t zero_per_256, void *d_out, void *stream);

/* Query: number of CUDA devices visible (0 on a CPU-only host). */
int32_t gck_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* GOCKPT_H_ */

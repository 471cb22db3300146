#!/usr/bin/env python
"""bench.py — GoCkpt hot path on B200: training throughput with the multi-step
overlapped checkpoint on, per-step checkpoint stall, D2H GB/s vs the host link.

One bench step = one checkpoint interval of `--interval` training steps
(default 50, the paper's "checkpoint every 50 steps") on the GPT-2 small
config (BASELINE.json configs[1]: 124,439,808-element fp32 AdamW shard, K=8):
  training step s:   F/B stand-in (GPT-2 small GEMM chain, CUDA graph, cuBLAS)
                     -> bf16 gradient (harness generator kernel)
                     [-> NCCL reduce-scatter into the ZeRO-1 shard when N > 1]
                     -> gck_submit: fused AdamW (+ pack of part i in the first K
                        steps of the interval) -> D2H drain on the side stream
                     [-> NCCL all-gather of the bf16 params when N > 1]
  after step K:      host replay runs on library threads while training goes on
  interval end:      gck_finalize (the consistent checkpoint S(t0+K-1)) + release.
All §8(a) rows (a0-a6) run inside every bench step.

Reported: value = tokens/s (all ranks) with checkpointing; the checkpoint-free
throughput of the same run; per-step stall (event-timed slot waits and step-time
delta); D2H GB/s vs the measured link peak; the fused kernel's HBM roofline;
the oracle timed on host cores (cpu_baseline); an end-to-end pass with the
gradient arriving from pinned host memory (e2e).

`--impl reference` times the CPU oracle (the tier's reference arm) instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "per-step checkpoint stall ms & train throughput w/ ckpt; D2H GB/s vs link peak"
WORKLOADS = {  # BASELINE.json configs
    "gpt2-small": "GPT-2 small 124M mixed-precision AdamW state, K=8 partitions, 1 B200",
    "llama2-7b": "Llama-2 7B ZeRO-1 optimizer shards across 8\u00d7B200, K=8, checkpoint every 100 steps",
    "llama2-13b": "Llama-2 13B ZeRO-1 across 2/4/8 B200, K sweep 2\u201316 (stall vs consistency-replay cost)",
}
DEFAULT_TOKENS = {"gpt2-small": 16 * 1024, "llama2-7b": 2 * 4096, "llama2-13b": 2048}
HP = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
LR = 3e-4
T_WARM = 100  # updates already done before the bench starts (bias-correction count offset)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5, help="timed checkpoint intervals")
    ap.add_argument("--warmup", type=int, default=3, help="untimed checkpoint intervals (>= 3)")
    ap.add_argument("--impl", default="gockpt", choices=["gockpt", "reference"])
    ap.add_argument("--interval", type=int, default=50)
    ap.add_argument("--K", type=int, default=8,
                    help="partitions per session; 0 = automatic (NEXT-4: chosen by the library from the measured "
                         "step time and link during warm-up, then held for the timed region)")
    ap.add_argument("--model", default="gpt2-small", choices=list(WORKLOADS))
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="nccl (default; the harness's gradient reduce-scatter / param all-gather run on it). "
                         "gloo = plumbing smoke test with several ranks sharing one GPU: no harness collectives")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="ZeRO-1 data-parallel degree the shard is cut for (0 = the launched world size); "
                         "e.g. 8 on one GPU = one rank of an 8-GPU job")
    ap.add_argument("--n", type=int, default=0, help="override the optimizer-shard elements per rank")
    ap.add_argument("--tokens", type=int, default=0, help="tokens per step per rank (0 = model default)")
    ap.add_argument("--copy-mode", default="ce", choices=["ce", "zerocopy"])
    ap.add_argument("--ring-slots", type=int, default=2)
    ap.add_argument("--staging", default="ring", choices=["ring", "direct", "blocking"],
                    help="ring: fused kernel packs into an HBM ring; direct: GoCkpt-O literal (no ring); "
                         "blocking: paper-faithful GoCkpt (the update waits for its gradient slice)")
    ap.add_argument("--scheme", default="gockpt", choices=["gockpt", "sync", "async-o"],
                    help="NEXT-3 baselines in the same harness: sync = blocking D2H snapshot of the full "
                         "state (DeepSpeed/Async snapshot phase); async-o = the snapshot overlaps the next "
                         "step's F/B and its update waits for it (P:312-318)")
    ap.add_argument("--replay-mode", default="host", choices=["host", "gpu", "deferred", "stream"],
                    help="consistency replay on the host pool (default) or in the GPU replay kernel; deferred "
                         "= replay-on-restore (finalize leaves the captured parts + gradient log for the "
                         "persisted file; S(T) is materialised at load); stream = streaming host replay (each slice's "
                         "update applied as it drains; gradient log = --stream-buffers recycled slices)")
    ap.add_argument("--stream-buffers", type=int, default=0, help="streaming replay slice buffers (0 = 4)")
    ap.add_argument("--replay-threads", type=int, default=0,
                    help="host replay / persist threads (0 = the host's cores divided by the local ranks)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 24,
                    help="elements of the oracle sample (cpu_baseline leg, ~15 s; --impl reference uses 1/16)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            mp = json.load(fh)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of fused_adamw_pack from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "fused_adamw_pack_ncu.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return None


# ----------------------------------------------------------------------------- oracle (CPU) timing
def oracle_interval_seconds(n_sample: int, K: int, interval: int, seed: int = 42) -> tuple[float, int]:
    """Time the oracle on the CPU work of one checkpoint interval over n_sample elements:
    `interval` AdamW updates (O1 trajectory) with a K-part session (capture + O2 replay)."""
    import numpy as np

    import gockpt_inputs as gi
    import oracle

    p, m, v = gi.warm_state(seed, n_sample)
    grads = [gi.grad_bits(seed, T_WARM + s, n_sample) for s in range(1, interval + 1)]
    recs = [oracle.make_step_record(t=T_WARM + s, lr=LR, **HP) for s in range(1, interval + 1)]
    t_start = time.perf_counter()
    parts = oracle.make_parts(n_sample, K, 1024)
    cap, glog, live = oracle.capture_session(p, m, v, grads[:K], recs[:K], parts)   # session steps 1..K
    ck = oracle.replay(cap, glog, recs[:K], parts)
    p, m, v = live
    for s in range(K, interval):                                                     # the rest of the interval
        p, m, v, _ = oracle.adamw_update(p, m, v, grads[s], recs[s])
    dt = time.perf_counter() - t_start
    assert ck[0].dtype == np.float32
    return dt, 1


def resolve(args):
    """Per-rank shard size and tokens from --model / --shard-of (ZeRO-1)."""
    from paper_2511_07035_b200.harness import MODELS, zero1_shard
    world, rank, _ = dist_env()
    W = args.shard_of or world
    N = MODELS[args.model][0]
    if not args.n:
        args.n = N if W == 1 else zero1_shard(N, W, min(rank, W - 1), 512)[1]
    if not args.tokens:
        args.tokens = DEFAULT_TOKENS[args.model]
    args.W = W
    args.workload = WORKLOADS[args.model]
    return args


def run_reference(args):
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return
    n_s = min(args.cpu_sample // 16, args.n)
    for _ in range(args.warmup):
        oracle_interval_seconds(min(n_s, 1 << 16), args.K, args.interval)
    times = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        dt, _ = oracle_interval_seconds(n_s, args.K, args.interval)
        times.append(dt * args.n / n_s)   # extrapolated to the full per-rank shard
    wall = time.perf_counter() - t0
    per_interval = statistics.mean(times)
    value = args.interval * args.tokens / per_interval
    cores = 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_interval * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.workload, "n_per_rank": args.n, "K": args.K, "interval": args.interval,
                   "tokens_per_step": args.tokens, "zero1_degree": args.W},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n_s} of {args.n} elements per interval, time x{args.n / n_s:.1f}; "
                                   f"the oracle's AdamW + capture + replay only (no F/B)",
                         "wall_s": wall},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- the GPU arm
def main():
    args = resolve(parse())
    if args.impl == "reference":
        return run_reference(args)
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_07035_b200 as G
    from paper_2511_07035_b200 import build as gbuild
    from paper_2511_07035_b200.harness import ClockSampler, TransformerGemmStandIn, max_over_ranks, all_ranks_ok

    world, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    local = local % torch.cuda.device_count()   # gloo smoke runs may put several ranks on one GPU
    torch.cuda.set_device(local)
    coll = world > 1 and args.dist_backend == "nccl"   # the harness's NCCL reduce-scatter / all-gather
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    gbuild.build()
    dev = torch.device("cuda", local)
    n, K, I, T = args.n, args.K, args.interval, args.tokens
    if not args.replay_threads:   # share the host's cores between the ranks of this node
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        args.replay_threads = max(1, len(os.sched_getaffinity(0)) // max(1, local_world))
    stream = torch.cuda.current_stream()

    # ---- state (synthetic warm S(t0), generated on device by the harness generator)
    master = torch.empty(n, dtype=torch.float32, device=dev)
    exp_avg = torch.empty_like(master)
    exp_avg_sq = torch.empty_like(master)
    param = torch.empty(n, dtype=torch.int16, device=dev)
    seed = 42 + rank
    G.h_generate(G.GEN_MASTER, master, seed, 0, rank * n, 1)
    G.h_generate(G.GEN_EXP_AVG, exp_avg, seed, 0, rank * n)
    G.h_generate(G.GEN_EXP_AVG_SQ, exp_avg_sq, seed, 0, rank * n)
    grad = torch.empty(n, dtype=torch.int16, device=dev)
    if coll:
        full_grad = torch.empty(n * world, dtype=torch.bfloat16, device=dev)
        full_param = torch.empty(n * world, dtype=torch.bfloat16, device=dev)
    fb = TransformerGemmStandIn(args.model, tokens=T, device=dev)
    fb.capture()
    auto_k = K == 0
    ctx = G.GoCkpt(master, exp_avg, exp_avg_sq, param, **HP, k_min=1 if auto_k else K, k_max=32 if auto_k else K,
                   part_align=1024,
                   ring_slots=args.ring_slots, copy_mode=args.copy_mode, replay_threads=args.replay_threads,
                   timing=True, eager_replay=True, staging=args.staging, replay_mode=args.replay_mode,
                   stream_buffers=args.stream_buffers)
    baseline = args.scheme != "gockpt"
    if baseline:
        snap_host = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(3)]
        side = torch.cuda.Stream()
    state = {"step": 0, "gen": 0, "K": K if not auto_k else 32, "auto": auto_k}

    # ---- host-link peak: best-of-5 1 GiB D2H into pinned memory, measured in this run
    link = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    link_h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        link_h.copy_(link, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    link_peak = (1 << 30) / best / 1e6
    del link, link_h

    result_host = []
    e2e_io = {}
    plain_bytes = 28 * n
    kern = {"plain_ms": [], "plain_bytes": 0, "sess_ms0": 0.0, "sess_n0": 0, "sess_bytes": 0}

    def train_step(part, h_grad=None, time_kernel=False, step_events=None, snapshot=False):
        state["step"] += 1
        s = state["step"]
        if step_events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            step_events.append(ev)
        pre_wait = baseline_snapshot() if snapshot else None   # NEXT-3 baselines: S(t0) = the state now
        g_in = grad
        if h_grad is not None:
            # e2e: the reduced gradient shard arrives from pinned host memory. Like a data loader it is
            # prefetched on a copy stream into one of two device buffers, overlapping this step's F/B;
            # the copy starts once the previous update has been enqueued (so the buffer it overwrites,
            # read by update s-2, is free) and, in direct staging, once the library's copy-out of the
            # previous gradient slice is done
            g_in = e2e_io["bufs"][s % 2]
            begin = torch.cuda.Event()
            begin.record(stream)
            loader = e2e_io["stream"]
            loader.wait_event(begin)
            ctx.grad_fence(loader)
            with torch.cuda.stream(loader):
                g_in.copy_(h_grad[s % len(h_grad)], non_blocking=True)
            e2e_io["loaded"].record(loader)
        fb()                                                           # F/B stand-in
        ctx.grad_fence(stream)   # direct staging: the last gradient slice is out before we overwrite
        if h_grad is not None:
            stream.wait_event(e2e_io["loaded"])
        elif coll:
            # backward's full local gradient (harness generator), then the ZeRO-1 reduce-scatter
            G.h_generate(G.GEN_GRAD, full_grad.view(torch.int16), seed, s, 0, 1, 4)
            state["gen"] += 1
            dist.reduce_scatter_tensor(grad.view(torch.bfloat16), full_grad)
        else:
            G.h_generate(G.GEN_GRAD, grad, seed, s, rank * n, 1, 4)    # backward's gradient (harness)
            state["gen"] += 1
        if pre_wait is not None:      # async-o: the update may not run before the snapshot copy ends
            stream.wait_event(pre_wait)
        a = b = None
        if time_kernel and part == 0:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        ctx.submit(part, s, T_WARM + s, LR, g_in, 1.0, False, stream)
        if a is not None:
            b.record(stream)
            kern["plain_ms"].append((a, b))
        if h_grad is not None:   # e2e: the step's result (first 8 bytes of the updated bf16 params) to host
            result_host[s % 2].copy_(param[:4], non_blocking=True)
        if coll:
            dist.all_gather_into_tensor(full_param, param.view(torch.bfloat16))

    def baseline_snapshot():
        """NEXT-3: snapshot S(t0) of the full state; returns the event the next update must wait on."""
        srcs = (master, exp_avg, exp_avg_sq)
        if args.scheme == "sync":
            for h, d in zip(snap_host, srcs):
                G.d2h_copy(h, d, stream=stream)        # on the compute stream: training blocks
            return None
        ev = torch.cuda.Event()
        ev.record(stream)
        side.wait_event(ev)
        for h, d in zip(snap_host, srcs):
            G.d2h_copy(h, d, stream=side)
        done = torch.cuda.Event()
        done.record(side)
        return done

    def interval(ckpt=True, h_grad=None, time_kernel=False, step_events=None):
        for j in range(1, I + 1):
            if ckpt and not baseline and j == 1:
                ctx.begin_checkpoint(state["step"], 0 if state["auto"] else state["K"])
                state["K"] = ctx.stats()["last_session_k"]
            part = j if (ckpt and not baseline and j <= state["K"]) else 0
            train_step(part, h_grad, time_kernel, step_events, snapshot=ckpt and baseline and j == 1)
        if ckpt and baseline:
            return
        if ckpt:
            ck = ctx.finalize()
            assert ck.step == state["step"] - I + state["K"] - 1
            ctx.release()
            assert all_ranks_ok(True)

    def timed(nint, **kw):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(nint):
            interval(**kw)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return max_over_ranks(e0.elapsed_time(e1) / 1e3)

    # ---- warm-up (untimed); with --K 0 the library picks K here (NEXT-4) and it is then held
    for _ in range(args.warmup):
        interval(ckpt=True)
    torch.cuda.synchronize()
    K = state["K"]
    state["auto"] = False
    parts = G.plan_parts(n, K, 1024)
    session_bytes = sum(12 * (hi - lo) + (2 * hi if i < K - 1 else 0) for i, (lo, hi) in enumerate(parts))

    # ---- checkpoint-free reference, first half (the second half runs after the timed region, so
    #      clock/thermal drift cancels in the stall and throughput deltas)
    free_ev_a = []
    n_free_a = max(1, args.steps // 2)
    t_free_a = timed(n_free_a, ckpt=False, step_events=free_ev_a)

    # ---- timed region: GoCkpt on
    st0 = ctx.stats()
    gen0 = state["gen"]
    step_ev = []
    clocks = ClockSampler(local).start()
    t_ck = timed(args.steps, ckpt=True, time_kernel=True, step_events=step_ev)
    clk = clocks.stop()
    st1 = ctx.stats()
    gpu_launches = (st1["gpu_launches"] - st0["gpu_launches"]) + (state["gen"] - gen0)
    tokens_total = args.steps * I * T * world
    value = tokens_total / t_ck
    # step times inside the timed region (event deltas); session steps are the first K of each interval
    step_ms = [step_ev[k].elapsed_time(step_ev[k + 1]) for k in range(len(step_ev) - 1)]
    K_aff = 1 if baseline else K      # steps of an interval the checkpoint can delay
    sess_ms = [t for k, t in enumerate(step_ms) if (k % I) < K_aff]
    plain_ms_steps = [t for k, t in enumerate(step_ms) if (k % I) >= K_aff]
    kern_plain = [a.elapsed_time(b) for a, b in kern["plain_ms"]]
    kern["plain_ms"] = []
    sess_kernel_ms = st1["kernel_ms_total"] - st0["kernel_ms_total"]
    sess_launches = st1["kernel_launches_timed"] - st0["kernel_launches_timed"]
    # roofline of the dominant launch kind (plain steps: 28 B/element, I-K of every I launches)
    plain_mean_s = statistics.mean(kern_plain) / 1e3
    achieved = plain_bytes / plain_mean_s / 1e9
    # session launches additionally write the slot (12|P_i| + 2 hi_i bytes, = the drained bytes)
    # (direct / blocking staging: the D2H reads the live arrays; the kernel writes no slot bytes)
    kern_slot_bytes = session_bytes if args.staging == "ring" else 0
    sess_alg = args.steps * (K * plain_bytes + kern_slot_bytes)
    sess_achieved = sess_alg / (sess_kernel_ms / 1e3) / 1e9 if sess_kernel_ms > 0 and not baseline else None
    hbm_peak, peak_src = peaks()
    stall_wait_ms = (st1["stall_ms_total"] - st0["stall_ms_total"])
    d2h_bytes = st1["d2h_bytes"] - st0["d2h_bytes"]
    d2h_ms = st1["d2h_ms_total"] - st0["d2h_ms_total"]

    # ---- checkpoint-free run of the same work (for the stall / throughput delta)
    free_ev = []
    n_free_b = max(1, args.steps - n_free_a)
    t_free_b = timed(n_free_b, ckpt=False, step_events=free_ev)
    free_step_ms = ([free_ev_a[k].elapsed_time(free_ev_a[k + 1]) for k in range(len(free_ev_a) - 1)] +
                    [free_ev[k].elapsed_time(free_ev[k + 1]) for k in range(len(free_ev) - 1)])
    free_med = statistics.median(free_step_ms)
    t_free = (t_free_a + t_free_b) / (n_free_a + n_free_b) * args.steps   # per args.steps intervals
    value_free = tokens_total / t_free

    # ---- e2e: gradient from pinned host memory each step, result = the host checkpoint
    e2e = None
    if not args.no_e2e:
        result_host[:] = [torch.empty(4, dtype=torch.int16, pin_memory=True) for _ in range(2)]
        h_grads = [torch.empty(n, dtype=torch.int16, pin_memory=True) for _ in range(2)]
        e2e_io.update(bufs=[grad, torch.empty_like(grad)], stream=torch.cuda.Stream(device=dev),
                      loaded=torch.cuda.Event())
        for k, hg in enumerate(h_grads):
            tmp = torch.empty(n, dtype=torch.int16, device=dev)
            G.h_generate(G.GEN_GRAD, tmp, seed, 10_000 + k, rank * n, 1, 4)
            hg.copy_(tmp)
            del tmp
        torch.cuda.synchronize()
        interval(ckpt=True, h_grad=h_grads)   # warm the path
        t_e2e = timed(max(1, args.steps), ckpt=True, h_grad=h_grads)
        e2e = {"value": max(1, args.steps) * I * T * world / t_e2e, "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": 8 + session_bytes / I,
               "note": "the reduced bf16 gradient shard arrives by H2D from pinned host memory every step "
                       "(prefetched on a copy stream into one of two device buffers while the step's F/B runs, "
                       "inside the timed region; replaces generator + reduce-scatter); each "
                       "step reads 8 bytes of the updated params back (the step's result), and the "
                       "checkpoint the library drains is the session's result (D2H)"}

    # ---- oracle on host cores (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_s = min(args.cpu_sample, n)
        dt, _ = oracle_interval_seconds(n_s, K, I)
        per_interval = dt * n / n_s
        cpu = {"value": I * T / per_interval, "unit": "tokens/s", "cores": 1, "kind": "oracle",
               "sample": f"{n_s} of {n} elements of one {I}-step interval (K={K} session + replay), "
                         f"{dt:.1f} s measured, time scaled x{n / n_s:.1f}; AdamW + capture + replay only, no F/B"}

    sess_stall_delta = [max(0.0, t - free_med) for t in sess_ms]
    # bootstrap 95% CI of the mean delta per session step, resampling whole sessions
    per_sess = [statistics.mean(sess_stall_delta[k:k + K_aff]) for k in range(0, len(sess_stall_delta), K_aff)]
    rng = np.random.default_rng(0)
    boot = [float(np.mean(rng.choice(per_sess, len(per_sess)))) for _ in range(2000)]
    delta_ci95 = [float(np.percentile(boot, 2.5)), float(np.percentile(boot, 97.5))]
    ctx_stats_final = ctx.stats()
    # NEXT-4: the analytic model's K for this step time and link (smallest K whose largest per-step
    # transfer fits in one step), next to the K this run used
    k_rec, vmax_rec = G.recommend_k(n, link_peak, free_med / 1e3, 1.0, 64)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_ck / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": args.workload, "n_per_rank": n, "K": K, "interval": I, "tokens_per_step_per_rank": T,
                   "zero1_degree": args.W,
                   "fb_standin": f"{args.model} fwd+bwd GEMM chain (cuBLAS bf16, CUDA graph)",
                   "fb_tflop_per_step": fb.flops / 1e12, "copy_mode": args.copy_mode,
                   "ring_slots": args.ring_slots, "staging": args.staging, "scheme": args.scheme,
                   "replay_mode": args.replay_mode, "dist_backend": args.dist_backend if world > 1 else None,
                   "parallelism": f"zero1-dp{world}",
                   "l2": f"inputs larger than L2 ({12 * n / 1e9:.2f} GB fp32 state + {2 * n / 1e9:.2f} GB gradient "
                         f"per step per rank)",
                   "step": "one checkpoint interval (I training steps, one K-part session, finalize)"},
        "stall": {"wait_ms_per_session_step": stall_wait_ms / (args.steps * K),
                  "wait_ms_max": st1["stall_ms_max"],
                  "session_step_ms_median": statistics.median(sess_ms),
                  "plain_step_ms_median": statistics.median(plain_ms_steps),
                  "ckpt_free_step_ms_median": free_med,
                  "delta_ms_per_session_step_mean": statistics.mean(sess_stall_delta),
                  "delta_ms_per_session_step_max": max(sess_stall_delta),
                  "delta_ms_per_session_step_median": statistics.median(sess_stall_delta),
                  "delta_ms_per_session_step_p90": float(np.percentile(sess_stall_delta, 90)),
                  "session_steps_measured": len(sess_stall_delta),
                  "delta_ms_per_session_step_ci95": delta_ci95,
                  "delta_ci_how": f"bootstrap over the {len(per_sess)} sessions (2000 resamples)",
                  "delta_frac_of_step": statistics.mean(sess_stall_delta) / free_med,
                  "delta_ms_vs_plain_steps_same_intervals": statistics.mean(sess_ms) - statistics.median(plain_ms_steps),
                  "delta_note": "delta_* compare session steps with the checkpoint-free run measured before and after "
                                "the timed region (clock/thermal drift between the regions shows up in it: compare "
                                "plain_step_ms_median with ckpt_free_step_ms_median); *_vs_plain_steps_same_intervals "
                                "compares them with the plain steps of the same timed intervals",
                  "amortized_frac": (t_ck - t_free) / t_free},
        "ckpt_free": {"value": value_free, "unit": "tokens/s", "throughput_ratio": value / value_free,
                      "how": "checkpoint-free intervals measured before and after the timed region, same run"},
        "d2h": {"gbs": d2h_bytes / (d2h_ms / 1e3) / 1e9 if d2h_ms > 0 else None,
                "link_peak_gbs": link_peak, "frac": (d2h_bytes / (d2h_ms / 1e3) / 1e9) / link_peak if d2h_ms else None,
                "frac_of_nominal_pcie5_x16": (d2h_bytes / (d2h_ms / 1e3) / 1e9) / 64.0 if d2h_ms else None,
                "bytes_per_session": session_bytes, "link_peak_how": "best of 5 x 1 GiB cudaMemcpyAsync D2H "
                "into pinned memory, this run"},
        "model": {"recommended_K": k_rec, "v_max_bytes_at_recommended_K": vmax_rec, "K_used": K,
                  "K_automatic": auto_k, "auto_step_ms": ctx_stats_final.get("auto_step_ms"),
                  "auto_link_gbs": ctx_stats_final.get("auto_link_gbs"),
                  "note": "gck_recommend_k(n, measured link GB/s, checkpoint-free step time)"},
        "replay": {"host_ms_last_session": st1["last_replay_ms"], "threads": st1["replay_threads"],
                   "worker_ms_last_session": st1["last_worker_ms"],
                   "finalize_wait_ms_last": st1["last_finalize_wait_ms"], "mode": args.replay_mode,
                   "stream_wait_ms_last": st1.get("last_stream_wait_ms"),
                   "timing_note": "host_ms = the replay arithmetic; worker/finalize_wait are host wall times "
                                  "from the moment the host enqueued step K (the host runs up to an interval "
                                  "ahead of the GPU), so they include waiting for the queued steps to execute",
                   "element_updates_per_session": sum((K - 1 - j) * (hi - lo) for j, (lo, hi) in enumerate(parts))},
        "roofline": {"bound": "hbm", "kernel": "fused_adamw_pack (plain step)", "achieved": achieved,
                     "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak, "peak_source": peak_src,
                     "traffic": (ncu_traffic() or {}).get("dram_bytes_per_launch"),
                     "alg_bytes_per_launch": plain_bytes, "launches": len(kern_plain),
                     "mean_launch_us": plain_mean_s * 1e6,
                     "session_launches": {"launches": sess_launches, "alg_bytes_per_launch_mean":
                                          plain_bytes + kern_slot_bytes / K,
                                          "achieved_gbs": sess_achieved,
                                          "frac": sess_achieved / hbm_peak if sess_achieved else None}},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": clk,
    }
    ctx.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

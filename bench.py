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
    "flat-1m": "flat 1M-element fp32 param vector, AdamW, checkpoint split over K=4 steps, single GPU (CPU oracle runs in seconds)",
    "gpt2-small": "GPT-2 small 124M mixed-precision AdamW state, K=8 partitions, 1 B200",
    "llama2-7b": "Llama-2 7B ZeRO-1 optimizer shards across 8\u00d7B200, K=8, checkpoint every 100 steps",
    "llama2-13b": "Llama-2 13B ZeRO-1 across 2/4/8 B200, K sweep 2\u201316 (stall vs consistency-replay cost)",
}
DEFAULT_TOKENS = {"flat-1m": 1, "gpt2-small": 16 * 1024, "llama2-7b": 2 * 4096, "llama2-13b": 2048}
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
    ap.add_argument("--cpu-sample", type=int, default=1 << 22,
                    help="elements of the oracle sample, the same for the cpu_baseline leg and every step of "
                         "--impl reference (~5 s of one pinned core per interval at 2^22)")
    ap.add_argument("--spin-ms", type=float, default=1.0,
                    help="flat-1m only: the F/B stand-in is one spin kernel of this many ms (0 = none)")
    ap.add_argument("--rs-bucket-mb", type=int, default=512,
                    help="N > 1 with NCCL: gradient reduce-scatter bucket size (input bytes), issued per "
                         "bucket while the rest of the backward stand-in runs")
    ap.add_argument("--verify-drain", type=int, default=1,
                    help="1 (library default): checksum every drained slice on the device and the host "
                         "(a3 verification); 0: off")
    ap.add_argument("--plan", choices=["equal", "balanced"], default="equal",
                    help="partition plan (a1): equal parts (S:131, the paper's default) or the transfer-balanced "
                         "plan (DESIGN.md R17: the parts that minimise the largest per-step D2H)")
    ap.add_argument("--force-collectives", action="store_true",
                    help="run the NCCL reduce-scatter / all-gather path even at N = 1 (a process group of one; "
                         "needs the torchrun environment or MASTER_ADDR/MASTER_PORT)")
    ap.add_argument("--step-log", default="",
                    help="write one JSON line per timed training step to this path (rank-suffixed when N > 1)")
    return ap.parse_args()


def maybe_reexec(args):
    """`--gpus N` (N > 1) without a torchrun environment: relaunch this command under
    torch.distributed.run with N local ranks (the driver's launch), so the N-GPU path runs as-is."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)


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
_ORACLE_INPUTS = {}


def oracle_interval_seconds(n_sample: int, K: int, interval: int, seed: int = 42, plan: str = "equal") -> tuple[float, int]:
    """Time the oracle on the CPU work of one checkpoint interval over n_sample elements:
    `interval` AdamW updates (O1 trajectory) with a K-part session (capture + O2 replay).
    The seeded inputs are generated once per sample size (outside the timed region)."""
    import numpy as np

    import gockpt_inputs as gi
    import oracle

    key = (n_sample, interval, seed)
    if key not in _ORACLE_INPUTS:
        _ORACLE_INPUTS.clear()
        _ORACLE_INPUTS[key] = (gi.warm_state(seed, n_sample),
                               [gi.grad_bits(seed, T_WARM + s, n_sample) for s in range(1, interval + 1)],
                               [oracle.make_step_record(t=T_WARM + s, lr=LR, **HP) for s in range(1, interval + 1)])
    (p, m, v), grads, recs = _ORACLE_INPUTS[key]
    t_start = time.perf_counter()
    mk = oracle.make_parts_balanced if plan == "balanced" else oracle.make_parts
    parts = mk(n_sample, K, min(1024, max(1, n_sample // K)))
    cap, glog, live = oracle.capture_session(p, m, v, grads[:K], recs[:K], parts)   # session steps 1..K
    ck = oracle.replay(cap, glog, recs[:K], parts)
    p, m, v = live
    for s in range(K, interval):                                                     # the rest of the interval
        p, m, v, _ = oracle.adamw_update(p, m, v, grads[s], recs[s])
    dt = time.perf_counter() - t_start
    assert ck[0].dtype == np.float32
    return dt, 1


class OneCore:
    """Pin this process to one core while the oracle is timed ("a single Python process
    pinned to one core"), then restore the previous affinity."""

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        self.core = min(self.saved)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.saved)


def oracle_baseline(args, K, steps=1, warmup=0):
    """The oracle on one pinned core over the same bounded sample in both legs (the GPU arm's
    cpu_baseline and every step of --impl reference): seconds per interval of the sample, and the
    extrapolation to the full per-rank shard stated separately."""
    n_s = min(args.cpu_sample, args.n)
    with OneCore() as oc:
        for _ in range(warmup):
            oracle_interval_seconds(n_s, K, args.interval, plan=args.plan)
        times = [oracle_interval_seconds(n_s, K, args.interval, plan=args.plan)[0] for _ in range(steps)]
    per_sample = statistics.mean(times)
    factor = args.n / n_s
    per_interval = per_sample * factor
    tps = args.interval * args.tokens / per_interval
    return {"value": tps, "unit": unit_of(args), "cores": 1, "kind": "oracle",
            "sample": f"{n_s} of {args.n} elements of each {args.interval}-step interval (K={K} session + O2 replay "
                      f"+ O1 updates), on core {oc.core}; AdamW + capture + replay only, no F/B",
            "sample_elements": n_s, "measured_s_per_interval_sample": per_sample,
            "extrapolation_factor": factor, "extrapolated_s_per_interval": per_interval,
            "samples_timed": len(times)}


def host_info():
    """The run header of the bench line: CPU model, cores, sockets, NUMA nodes of the box."""
    model, sockets = None, set()
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name") and model is None:
                    model = line.split(":", 1)[1].strip()
                elif line.startswith("physical id"):
                    sockets.add(line.split(":", 1)[1].strip())
    except OSError:
        pass
    try:
        nodes = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node") and d[4:].isdigit()])
    except OSError:
        nodes = None
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0)),
            "sockets": len(sockets) or None, "numa_nodes": nodes}


def unit_of(args):
    return "steps/s" if args.model == "flat-1m" else "tokens/s"


def config_dict(args, world):
    """The `config` of both arms' lines (identical, so the driver can pair them)."""
    from paper_2511_07035_b200.harness import standin_flops
    fb = (f"spin kernel {args.spin_ms:g} ms" if args.model == "flat-1m"
          else f"{args.model} fwd+bwd GEMM chain (cuBLAS bf16, CUDA graphs)")
    return {"workload": args.workload, "n_per_rank": args.n, "K": args.K, "interval": args.interval,
            "tokens_per_step_per_rank": args.tokens, "zero1_degree": args.W,
            "fb_standin": fb,
            "fb_tflop_per_step": 0.0 if args.model == "flat-1m" else standin_flops(args.model, args.tokens) / 1e12,
            "copy_mode": args.copy_mode, "ring_slots": args.ring_slots, "staging": args.staging,
            "verify_drain": bool(args.verify_drain), "plan": args.plan,
            "scheme": args.scheme, "replay_mode": args.replay_mode,
            "dist_backend": args.dist_backend if world > 1 else None,
            "rs_bucket_mb": args.rs_bucket_mb if (world > 1 or getattr(args, "force_collectives", False))
            and args.dist_backend == "nccl" else None,
            "parallelism": f"zero1-dp{world}",
            "l2": f"inputs larger than L2 ({12 * args.n / 1e9:.2f} GB fp32 state + {2 * args.n / 1e9:.2f} GB "
                  f"gradient per step per rank)" if args.n * 14 > 126e6 else
                  "state smaller than L2: the checkpoint-free and session steps see the same cache state",
            "step": "one checkpoint interval (I training steps, one K-part session, finalize)"}


def resolve(args):
    """Per-rank shard size and tokens from --model / --shard-of (ZeRO-1)."""
    from paper_2511_07035_b200.harness import FLAT_1M, MODELS, zero1_shard
    world, rank, _ = dist_env()
    W = args.shard_of or world
    N = FLAT_1M if args.model == "flat-1m" else MODELS[args.model][0]
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
    t0 = time.perf_counter()
    cpu = oracle_baseline(args, args.K if args.K else 8, steps=args.steps, warmup=args.warmup)
    cpu["wall_s"] = time.perf_counter() - t0
    value = cpu["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit_of(args), "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["extrapolated_s_per_interval"] * 1e3,
        "ms_per_step_note": "extrapolated: measured_s_per_interval_sample x extrapolation_factor "
                            "(cpu_baseline); the measured wall time of this run is cpu_baseline.wall_s",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, world),
        "host": host_info(),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": unit_of(args), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- the GPU arm
def main():
    args = parse()
    maybe_reexec(args)
    args = resolve(args)
    world, _, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch N ranks for --gpus N)")
    if args.impl == "reference":
        return run_reference(args)
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    if args.dist_backend == "nccl" and (world > 1 or args.force_collectives):
        # NCCL's INFO lines (transport, NVLS) stay on, on stderr (stdout carries the JSON line); set
        # before torch loads NCCL, which reads them once
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("VERSION", ""):  # the image sets VERSION
            os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2511_07035_b200 as G
    from paper_2511_07035_b200 import build as gbuild
    from paper_2511_07035_b200.harness import (ClockSampler, SpinStandIn, TransformerGemmStandIn, all_ranks_ok,
                                               max_over_ranks, rs_buckets)

    world, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    local = local % torch.cuda.device_count()   # gloo smoke runs may put several ranks on one GPU
    torch.cuda.set_device(local)
    # the harness's NCCL reduce-scatter / all-gather (--force-collectives: also at N = 1, a process
    # group of one, so the bucketed-RS code path and NCCL's init run on a one-GPU box)
    coll = (world > 1 or args.force_collectives) and args.dist_backend == "nccl"
    if world > 1 or coll:
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
    if args.model == "flat-1m":
        fb = SpinStandIn(args.spin_ms, device=dev)
    else:
        fb = TransformerGemmStandIn(args.model, tokens=T, device=dev)
    # N > 1 (NCCL): the ZeRO-1 gradient reduce-scatter runs per bucket (512 MB buckets)
    # as soon as the backward part that "produced" the bucket is done, overlapping the rest of it
    buckets = rs_buckets(n, world, args.rs_bucket_mb << 20) if coll else []
    bwd_parts = max(1, min(8, len(buckets)))
    fb.capture(bwd_parts)
    part_buckets = [buckets[k * len(buckets) // bwd_parts:(k + 1) * len(buckets) // bwd_parts]
                    for k in range(bwd_parts)]
    auto_k = K == 0
    ctx = G.GoCkpt(master, exp_avg, exp_avg_sq, param, **HP, k_min=1 if auto_k else K, k_max=32 if auto_k else K,
                   part_align=1024,
                   ring_slots=args.ring_slots, copy_mode=args.copy_mode, replay_threads=args.replay_threads,
                   timing=True, eager_replay=True, staging=args.staging, replay_mode=args.replay_mode,
                   stream_buffers=args.stream_buffers, verify_drain=bool(args.verify_drain), plan=args.plan)
    baseline = args.scheme != "gockpt"
    if baseline:
        snap_host = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in range(3)]
        side = torch.cuda.Stream()
    state = {"step": 0, "gen": 0, "K": K if not auto_k else 32, "auto": auto_k}

    # ---- host-link peak: best-of-5 1 GiB D2H into pinned memory, measured in this run — rank 0 alone
    #      (the others wait at a barrier), then all ranks at once (the rate the sessions' drains share)
    link = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    link_h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)

    def d2h_peak():
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            link_h.copy_(link, non_blocking=True)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return (1 << 30) / best / 1e6

    if world > 1:
        dist.barrier()
    link_alone = d2h_peak() if rank == 0 else 0.0
    if world > 1:
        dist.barrier()
        link_peak = d2h_peak()          # this rank, all ranks copying concurrently
        dist.barrier()
    else:
        link_peak = link_alone
    del link, link_h

    result_host = []
    e2e_io = {}
    plain_bytes = 28 * n
    kern = {"plain_ms": [], "plain_step": [], "plain_bytes": 0, "sess_ms0": 0.0, "sess_n0": 0, "sess_bytes": 0}
    sess_log = []   # per timed session: (first training step, gck_get_session_steps entries)

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
        torch.cuda.nvtx.range_push(f"step {s} F/B")
        fb.forward()                                                   # F/B stand-in
        works = []
        for k in range(fb.bwd_parts):
            fb.backward(k)
            if h_grad is None and coll:
                # the buckets this backward part completed (harness generator = the local gradient,
                # bucket-major layout [bucket][rank][count]) go out while the rest of the backward runs
                for off, cnt in part_buckets[k]:
                    src = full_grad[world * off:world * (off + cnt)]
                    G.h_generate(G.GEN_GRAD, src.view(torch.int16), seed, s, world * off, 1, 4)
                    state["gen"] += 1
                    works.append(dist.reduce_scatter_tensor(grad[off:off + cnt].view(torch.bfloat16), src,
                                                            async_op=True))
        torch.cuda.nvtx.range_pop()
        ctx.grad_fence(stream)   # direct staging: the last gradient slice is out before we overwrite
        if h_grad is not None:
            stream.wait_event(e2e_io["loaded"])
        elif coll:
            for w in works:      # the update consumes the reduced shard
                w.wait()
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
            kern["plain_step"].append(s)
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
            if state.get("log_sessions"):
                sess_log.append((state["step"] - I + 1, ctx.session_steps()))
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
    parts = G.plan_parts(n, K, 1024, plan=args.plan)
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
    first_timed_step = state["step"] + 1
    state["log_sessions"] = True
    t_ck = timed(args.steps, ckpt=True, time_kernel=True, step_events=step_ev)
    state["log_sessions"] = False
    clk = clocks.stop()
    st1 = ctx.stats()
    gpu_launches = (st1["gpu_launches"] - st0["gpu_launches"]) + (state["gen"] - gen0)
    tokens_total = args.steps * I * T * world   # flat-1m: T = 1, the value is training steps/s
    value = tokens_total / t_ck
    # step times inside the timed region (event deltas); session steps are the first K of each interval
    step_ms = [step_ev[k].elapsed_time(step_ev[k + 1]) for k in range(len(step_ev) - 1)]
    K_aff = 1 if baseline else K      # steps of an interval the checkpoint can delay
    sess_ms = [t for k, t in enumerate(step_ms) if (k % I) < K_aff]
    plain_ms_steps = [t for k, t in enumerate(step_ms) if (k % I) >= K_aff]
    kern_plain = [a.elapsed_time(b) for a, b in kern["plain_ms"]]
    plain_kernel_of_step = dict(zip(kern["plain_step"], kern_plain))
    kern["plain_ms"], kern["plain_step"] = [], []
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
        e2e = {"value": max(1, args.steps) * I * T * world / t_e2e, "unit": unit_of(args),
               "h2d_bytes_per_step": 2 * n, "d2h_bytes_per_step": 8 + session_bytes / I,
               "note": "the reduced bf16 gradient shard arrives by H2D from pinned host memory every step "
                       "(prefetched on a copy stream into one of two device buffers while the step's F/B runs, "
                       "inside the timed region; replaces generator + reduce-scatter); each "
                       "step reads 8 bytes of the updated params back (the step's result), and the "
                       "checkpoint the library drains is the session's result (D2H)"}

    # ---- oracle on one pinned host core (rank 0, N=1 only), the same sample as --impl reference
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(args, K)

    sess_stall_delta = [max(0.0, t - free_med) for t in sess_ms]
    # bootstrap 95% CI of the mean delta per session step, resampling whole sessions
    per_sess = [statistics.mean(sess_stall_delta[k:k + K_aff]) for k in range(0, len(sess_stall_delta), K_aff)]
    rng = np.random.default_rng(0)
    boot = [float(np.mean(rng.choice(per_sess, len(per_sess)))) for _ in range(2000)]
    delta_ci95 = [float(np.percentile(boot, 2.5)), float(np.percentile(boot, 97.5))]
    ctx_stats_final = ctx.stats()
    d2h_gbs = d2h_bytes / (d2h_ms / 1e3) / 1e9 if d2h_ms > 0 else None
    mine = {"rank": rank, "wait_ms_per_session_step": stall_wait_ms / (args.steps * K),
            "delta_ms_per_session_step_mean": statistics.mean(sess_stall_delta),
            "delta_frac_of_step": statistics.mean(sess_stall_delta) / free_med,
            "d2h_gbs": d2h_gbs, "link_peak_concurrent_gbs": link_peak, "ckpt_free_step_ms_median": free_med}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    # ---- per-step log of the timed region (SURVEY §5 metrics): one JSON line per training step
    if args.step_log:
        recs = {}
        for s0, steps in sess_log:
            for e in steps:
                recs[s0 + e["part"] - 1] = e
        path = args.step_log if world == 1 else f"{args.step_log}.rank{rank}"
        with open(path, "w") as fh:
            for k, t in enumerate(step_ms):
                st_idx = first_timed_step + k
                e = recs.get(st_idx)
                fh.write(json.dumps({
                    "step": st_idx, "interval": k // I, "part": e["part"] if e else 0, "rank": rank,
                    "t_step_ms": t, "stall_ms": t - free_med, "wait_ms": e["wait_ms"] if e else 0.0,
                    "fused_ms": e["kernel_ms"] if e else plain_kernel_of_step.get(st_idx),
                    "d2h_bytes": e["d2h_bytes"] if e else 0, "d2h_ms": e["d2h_ms"] if e else 0.0,
                    "slot": (None if e["slot"] == 0xFFFFFFFF else e["slot"]) if e else None}) + "\n")
    # NEXT-4: the analytic model's K for this step time and link (smallest K whose largest per-step
    # transfer fits in one step), next to the K this run used
    k_rec, vmax_rec = G.recommend_k(n, link_peak, free_med / 1e3, 1.0, 64, plan=args.plan)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": unit_of(args),
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_ck / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": dict(config_dict(args, world), K=K),
        "host": host_info(),
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
        "per_rank": {"ranks": per_rank,
                     "max_wait_ms_per_session_step": max(r["wait_ms_per_session_step"] for r in per_rank),
                     "max_delta_ms_per_session_step_mean": max(r["delta_ms_per_session_step_mean"] for r in per_rank),
                     "max_delta_frac_of_step": max(r["delta_frac_of_step"] for r in per_rank),
                     "min_d2h_gbs": min((r["d2h_gbs"] or 0.0) for r in per_rank),
                     "max_d2h_gbs": max((r["d2h_gbs"] or 0.0) for r in per_rank),
                     "note": "SURVEY §8(d) M1 target: max over ranks of the per-session-step stall < 5% of the "
                             "checkpoint-free step"},
        "ckpt_free": {"value": value_free, "unit": unit_of(args), "throughput_ratio": value / value_free,
                      "how": "checkpoint-free intervals measured before and after the timed region, same run"},
        "d2h": {"gbs": d2h_gbs,
                "link_peak_gbs": link_peak, "frac": d2h_gbs / link_peak if d2h_gbs else None,
                "link_peak_alone_gbs": link_alone, "link_peak_concurrent_gbs": link_peak,
                "frac_of_nominal_pcie5_x16": d2h_gbs / 64.0 if d2h_gbs else None,
                "bytes_per_session": session_bytes, "link_peak_how": "best of 5 x 1 GiB cudaMemcpyAsync D2H "
                "into pinned memory, this run: rank 0 alone (the others at a barrier), then every rank at once "
                "(link_peak_gbs = this rank's concurrent figure; the two coincide at N = 1)"},
        "model": {"recommended_K": k_rec, "v_max_bytes_at_recommended_K": vmax_rec, "K_used": K,
                  "K_automatic": auto_k, "auto_step_ms": ctx_stats_final.get("auto_step_ms"),
                  "auto_link_gbs": ctx_stats_final.get("auto_link_gbs"),
                  "note": "gck_recommend_k(n, measured link GB/s, checkpoint-free step time)"},
        "replay": {"host_ms_last_session": st1["last_replay_ms"], "threads": st1["replay_threads"],
                   "verify_ms_last_session": st1.get("last_verify_ms"),
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
    if world > 1 or coll:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

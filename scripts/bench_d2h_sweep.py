"""BASELINE config 5: staging/transfer bandwidth sweep, 16 MiB .. 8 GiB per rank,
copy engine vs zero-copy, through the library's own drain mechanism (gck_d2h_copy).

python scripts/bench_d2h_sweep.py [--max-log2 9] [--reps 5] [--out gpurun_out/d2h_sweep.jsonl]
Under torchrun every rank sweeps concurrently (the "concurrent link peak"); rank 0 prints.
Each copy is verified byte-exact against the device source (full compare up to 1 GiB,
three 16 MiB windows beyond).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_07035_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-log2", type=int, default=9)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default="gpurun_out/d2h_sweep.jsonl")
ap.add_argument("--with-gemm", action="store_true", help="run a bf16 GEMM loop on another stream meanwhile")
args = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dev = torch.device("cuda", local)
MiB = 1 << 20
max_bytes = 16 * MiB << args.max_log2
src = torch.empty(max_bytes // 2, dtype=torch.int16, device=dev)
G.h_generate(G.GEN_GRAD, src, 1234 + rank, 0, 0, 0, 0)
dst = torch.empty(max_bytes, dtype=torch.uint8, pin_memory=True)
stream = torch.cuda.Stream(priority=0)
modes = [("ce", 0, 0), ("ce", 4 * MiB, 0), ("ce", 64 * MiB, 0)] + [("zerocopy", 0, c) for c in (8, 16, 32, 64, 148)]

gemm_stream = torch.cuda.Stream()
A = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
B = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)


def verify(nbytes):
    s = src.view(torch.uint8)[:nbytes]
    if nbytes <= 1 << 30:
        return bool(torch.equal(dst[:nbytes], s.cpu()))
    ok = True
    for off in (0, nbytes // 2, nbytes - 16 * MiB):
        ok &= bool(torch.equal(dst[off:off + 16 * MiB], s[off:off + 16 * MiB].cpu()))
    return ok


results = []
for k in range(args.max_log2 + 1):
    nbytes = 16 * MiB << k
    for mode, chunk, ctas in modes:
        if mode == "ce" and chunk and chunk >= nbytes:
            continue
        times = []
        for r in range(args.reps + 1):
            dst[:nbytes].zero_() if r == 0 else None
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            if args.with_gemm:
                with torch.cuda.stream(gemm_stream):
                    for _ in range(4):
                        torch.mm(A, B)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            G.d2h_copy(dst, src, nbytes, mode, chunk, ctas, stream)
            b.record(stream)
            torch.cuda.synchronize()
            if r == 0:
                ok = verify(nbytes)
                assert ok, (nbytes, mode, chunk, ctas)
                continue
            times.append(a.elapsed_time(b) / 1e3)
        best, med = min(times), statistics.median(times)
        rec = {"rank": rank, "world": world, "bytes": nbytes, "mode": mode, "chunk": chunk, "ctas": ctas,
               "best_gbs": nbytes / best / 1e9, "median_gbs": nbytes / med / 1e9, "verified": True,
               "with_gemm": args.with_gemm}
        if world > 1:
            t = torch.tensor([best, med], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            rec["slowest_rank_best_gbs"] = nbytes / float(t[0]) / 1e9
        results.append(rec)
        if rank == 0:
            print(json.dumps(rec), flush=True)
if rank == 0:
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "a") as fh:
        for rec in results:
            fh.write(json.dumps(rec) + "\n")
if world > 1:
    dist.destroy_process_group()

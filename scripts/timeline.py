"""Overlap evidence (the analog of the paper's breakdown timeline, §5.5, and its transfer
monitors, §5.6): a CUPTI activity trace (torch.profiler / Kineto records every kernel and
memcpy of the process, including libgockpt's own launches and copies) of GoCkpt intervals on the
bench's GPT-2 configuration, reduced to per-step numbers:

  - per training step: the F/B stand-in's GEMM time on the compute stream, the fused kernel, the
    compute stream's idle time (the stall shows up here), and the D2H copy-engine busy time;
  - the fraction of D2H busy time that overlaps GEMM execution (hidden transfer);
  - session steps vs plain steps.

nsys is not installed in this image; CUPTI through torch.profiler gives the same device timeline.
The library also emits NVTX ranges (gck_submit / drain enqueue / replay worker / finalize) for nsys.

python scripts/timeline.py [--K 8] [--interval 12] [--intervals 2] [--out profiles/r02_timeline]
"""
import argparse
import gzip
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def merge(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def total(iv):
    return sum(b - a for a, b in iv)


def intersect(x, y):
    i = j = 0
    out = 0.0
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            out += b - a
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return out


def clip(iv, lo, hi):
    return [[max(a, lo), min(b, hi)] for a, b in iv if b > lo and a < hi]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, default=8)
    ap.add_argument("--interval", type=int, default=12)
    ap.add_argument("--intervals", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=16 * 1024)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_timeline"))
    args = ap.parse_args()

    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2511_07035_b200 as G
    from paper_2511_07035_b200.harness import TransformerGemmStandIn

    n, K, I = 124_439_808, args.K, args.interval
    dev = torch.device("cuda", 0)
    p = torch.empty(n, dtype=torch.float32, device=dev)
    m, v = torch.empty_like(p), torch.empty_like(p)
    G.h_generate(G.GEN_MASTER, p, 42, 0, 0, 1)
    G.h_generate(G.GEN_EXP_AVG, m, 42)
    G.h_generate(G.GEN_EXP_AVG_SQ, v, 42)
    out = torch.empty(n, dtype=torch.int16, device=dev)
    g = torch.empty(n, dtype=torch.int16, device=dev)
    fb = TransformerGemmStandIn("gpt2-small", tokens=args.tokens, device=dev)
    fb.capture()
    ctx = G.GoCkpt(p, m, v, out, k_min=K, k_max=K, timing=True)
    stream = torch.cuda.current_stream()
    step = [100]

    def interval():
        for j in range(1, I + 1):
            if j == 1:
                ctx.begin_checkpoint(step[0], K)
            step[0] += 1
            s = step[0]
            torch.cuda.nvtx.range_push(f"step {s}")
            fb()
            G.h_generate(G.GEN_GRAD, g, 42, s, 0, 1, 4)
            ctx.submit(j if j <= K else 0, s, s, 3e-4, g, 1.0, False, stream)
            torch.cuda.nvtx.range_pop()
        ctx.finalize()
        ctx.release()

    for _ in range(3):
        interval()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(args.intervals):
            interval()
        torch.cuda.synchronize()
    raw = args.out + "_trace.json"
    prof.export_chrome_trace(raw)
    ev = json.load(open(raw))["traceEvents"]
    kern = [e for e in ev if e.get("cat") == "kernel"]
    cps = [e for e in ev if e.get("cat") == "gpu_memcpy"]
    fused = sorted([e for e in kern if "fused_adamw_pack" in e["name"]], key=lambda e: e["ts"])
    cstream = fused[0]["args"]["stream"]
    gemm = merge([[e["ts"], e["ts"] + e["dur"]] for e in kern
                  if e["args"]["stream"] == cstream and "adamw" not in e["name"] and "generate" not in e["name"]])
    comp_busy = merge([[e["ts"], e["ts"] + e["dur"]] for e in kern if e["args"]["stream"] == cstream])
    d2h = merge([[e["ts"], e["ts"] + e["dur"]] for e in cps if "DtoH" in e["name"] and
                 e["args"]["stream"] != cstream])
    d2h_bytes = sum(e["args"].get("bytes", 0) for e in cps if "DtoH" in e["name"] and e["args"]["stream"] != cstream)
    rows = []
    for k in range(1, len(fused)):
        lo, hi = fused[k - 1]["ts"] + fused[k - 1]["dur"], fused[k]["ts"] + fused[k]["dur"]
        sess = "<true" in fused[k]["name"] or "<1," in fused[k]["name"]
        gi, di, ci = clip(gemm, lo, hi), clip(d2h, lo, hi), clip(comp_busy, lo, hi)
        rows.append({"k": k, "session": sess, "step_ms": (hi - lo) / 1e3, "gemm_ms": total(gi) / 1e3,
                     "fused_ms": fused[k]["dur"] / 1e3, "compute_idle_ms": (hi - lo - total(ci)) / 1e3,
                     "d2h_busy_ms": total(di) / 1e3, "d2h_under_gemm_ms": intersect(di, gi) / 1e3})
    sess = [r for r in rows if r["session"]]
    plain = [r for r in rows if not r["session"]]
    d2h_tot, d2h_gemm = total(d2h), intersect(d2h, gemm)
    summary = {
        "config": {"n": n, "K": K, "interval": I, "intervals_traced": args.intervals, "tokens": args.tokens,
                   "source": "torch.profiler (CUPTI activity) trace of the whole process"},
        "d2h_busy_ms_total": d2h_tot / 1e3, "d2h_bytes_total": d2h_bytes,
        "d2h_gbs_while_busy": d2h_bytes / (d2h_tot / 1e6) / 1e9 if d2h_tot else None,
        "d2h_overlapping_gemm_frac": d2h_gemm / d2h_tot if d2h_tot else None,
        "session_step_ms_median": statistics.median(r["step_ms"] for r in sess),
        "plain_step_ms_median": statistics.median(r["step_ms"] for r in plain),
        "session_compute_idle_ms_median": statistics.median(r["compute_idle_ms"] for r in sess),
        "plain_compute_idle_ms_median": statistics.median(r["compute_idle_ms"] for r in plain),
        "session_fused_ms_median": statistics.median(r["fused_ms"] for r in sess),
        "plain_fused_ms_median": statistics.median(r["fused_ms"] for r in plain),
        "steps": rows,
    }
    json.dump(summary, open(args.out + ".json", "w"), indent=1)
    with gzip.open(raw + ".gz", "wt") as fh:   # keep the kernels + copies only, compressed
        json.dump({"traceEvents": [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]}, fh)
    os.unlink(raw)
    lines = [f"CUPTI trace (torch.profiler) of {args.intervals} GoCkpt intervals, GPT-2 small n={n}, K={K}, "
             f"interval {I}, F/B stand-in {args.tokens} tokens", "",
             f"D2H busy {d2h_tot / 1e3:.1f} ms for {d2h_bytes / 1e9:.3f} GB "
             f"({summary['d2h_gbs_while_busy']:.1f} GB/s while busy); "
             f"{100 * summary['d2h_overlapping_gemm_frac']:.1f}% of it overlaps F/B GEMMs on the compute stream", "",
             "step  sess  step_ms  gemm_ms  fused_ms  idle_ms  d2h_ms  d2h_under_gemm_ms"]
    for r in rows:
        lines.append(f"{r['k']:4d}  {'S' if r['session'] else '.':>4}  {r['step_ms']:7.2f}  {r['gemm_ms']:7.2f}  "
                     f"{r['fused_ms']:8.3f}  {r['compute_idle_ms']:7.3f}  {r['d2h_busy_ms']:6.2f}  "
                     f"{r['d2h_under_gemm_ms']:7.2f}")
    lines += ["", f"median step: session {summary['session_step_ms_median']:.3f} ms, plain "
                  f"{summary['plain_step_ms_median']:.3f} ms; compute-stream idle: session "
                  f"{summary['session_compute_idle_ms_median']:.3f} ms, plain {summary['plain_compute_idle_ms_median']:.3f} ms"]
    open(args.out + ".txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:4] + lines[-1:]))
    ctx.close()


if __name__ == "__main__":
    main()

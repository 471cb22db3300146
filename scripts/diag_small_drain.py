"""Diagnostic: per-step D2H time of small sessions (BASELINE config 1, n = 2^20, K = 4).

The C1 bench lines report ~0.5 ms per 4 MB slice drain (7 GB/s) against 56 GB/s for 16 MiB
copies. This separates the pieces: raw cudaMemcpyAsync of the same byte counts (torch, pinned),
gck_d2h_copy, and GoCkpt sessions with verification on / off, each with the library's own
per-step events (gck_get_session_steps). One JSON line per case.
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gockpt_inputs as gi  # noqa: E402
import paper_2511_07035_b200 as G  # noqa: E402


def raw_copies(nbytes_list, reps=20, side=True):
    dev = [torch.empty(b, dtype=torch.uint8, device="cuda") for b in nbytes_list]
    host = [torch.empty(b, dtype=torch.uint8, pin_memory=True) for b in nbytes_list]
    s = torch.cuda.Stream(priority=0) if side else torch.cuda.current_stream()
    ts = []
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for d, h in zip(dev, host):
                h.copy_(d, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    tot = sum(nbytes_list)
    return {"bytes": tot, "ms_median": ts[len(ts) // 2], "ms_min": ts[0], "gbs_median": tot / ts[len(ts) // 2] / 1e6}


def session(n, K, verify, spin_ms=0.0, sessions=6, interval=8, copy_mode="ce"):
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(1, n)
    p, m, v = (torch.from_numpy(x.copy()).cuda() for x in (p0, m0, v0))
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = torch.from_numpy(gi.grad_bits(1, 1, n).view(np.int16).copy()).cuda()
    ctx = G.GoCkpt(p, m, v, out, **hp, k_min=1, k_max=16, part_align=1024, verify_drain=verify,
                   copy_mode=copy_mode)
    step = 0
    rows = []
    wall = []
    spin = None
    if spin_ms > 0:
        a = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
        spin = lambda: a @ a  # noqa: E731
    for s_ in range(sessions):
        t0 = step
        ctx.begin_checkpoint(t0, K)
        tw = time.perf_counter()
        for i in range(1, K + 1):
            step += 1
            if spin is not None:
                spin()
            ctx.submit(i, step, step, 1e-3, g)
        ck = ctx.finalize()
        wall.append((time.perf_counter() - tw) * 1e3)
        if s_ >= 2:
            rows += ctx.session_steps()
        ctx.release()
        for _ in range(interval - K):
            step += 1
            ctx.submit(0, step, step, 1e-3, g)
        torch.cuda.synchronize()
    ctx.close()
    d2h = [r for r in rows if r.get("d2h_bytes")]
    keys = sorted(d2h[0].keys()) if d2h else []
    med = {k: float(np.median([r[k] for r in d2h])) for k in keys if isinstance(d2h[0][k], (int, float))}
    return {"n": n, "K": K, "verify": verify, "copy_mode": copy_mode, "spin_ms": spin_ms,
            "session_wall_ms_median": float(np.median(wall[2:])), "step_medians": med}


def main():
    torch.cuda.set_device(0)
    n, K = 1 << 20, 4
    pe = n // K
    print(json.dumps({"case": "raw 1x4MiB", **raw_copies([4 << 20])}), flush=True)
    print(json.dumps({"case": "raw 3x1MiB+2MiB (slice 2)", **raw_copies([pe * 4] * 3 + [2 * pe * 2])}), flush=True)
    print(json.dumps({"case": "raw 16MiB", **raw_copies([16 << 20])}), flush=True)
    print(json.dumps({"case": "raw 3x1MiB+2MiB current stream", **raw_copies([pe * 4] * 3 + [2 * pe * 2], side=False)}),
          flush=True)
    for verify in (True, False):
        for cm in ("ce", "zerocopy"):
            print(json.dumps({"case": "session", **session(n, K, verify, copy_mode=cm)}), flush=True)
    print(json.dumps({"case": "session", **session(n, K, True, spin_ms=1.0)}), flush=True)
    n2 = 1 << 24
    print(json.dumps({"case": "session 16M", **session(n2, K, True)}), flush=True)


if __name__ == "__main__" and not os.environ.get("DIAG_TRACE"):
    main()


def trace(n=1 << 20, K=4, verify=True):
    """CUPTI trace (torch.profiler) of one small session: GPU memcpy/kernel durations and the host
    API durations of the library's calls, to tell device time from host enqueue time."""
    from torch.profiler import ProfilerActivity, profile
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(1, n)
    p, m, v = (torch.from_numpy(x.copy()).cuda() for x in (p0, m0, v0))
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = torch.from_numpy(gi.grad_bits(1, 1, n).view(np.int16).copy()).cuda()
    ctx = G.GoCkpt(p, m, v, out, **hp, k_min=1, k_max=16, part_align=1024, verify_drain=verify)
    step = 0
    for s_ in range(4):
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) if s_ == 3 else _Null() as prof:
            ctx.begin_checkpoint(step, K)
            for i in range(1, K + 1):
                step += 1
                ctx.submit(i, step, step, 1e-3, g)
            ctx.finalize()
            torch.cuda.synchronize()
        print(json.dumps({"session": s_, "steps": ctx.session_steps()}), file=sys.stderr)
        ctx.release()
    ctx.close()
    prof.export_chrome_trace(os.environ.get("DIAG_TRACE_OUT", "/tmp/diag_trace.json"))
    evs = []
    for e in prof.events():
        evs.append({"name": e.name[:60], "dev": str(e.device_type), "start_us": e.time_range.start,
                    "dur_us": e.time_range.end - e.time_range.start})
    evs.sort(key=lambda x: x["start_us"])
    t0 = evs[0]["start_us"] if evs else 0
    for x in evs:
        x["start_us"] -= t0
    return evs


class _Null:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


if __name__ == "__main__" and os.environ.get("DIAG_TRACE"):
    torch.cuda.set_device(0)
    for x in trace(verify=os.environ.get("DIAG_TRACE") == "1"):
        print(json.dumps(x))

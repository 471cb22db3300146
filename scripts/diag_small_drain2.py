"""Diagnostic 2 for small sessions (n = 2^20, K = 4): per-step D2H / kernel event times and host
submit times when the session steps are (a) issued back to back, (b) separated by a host sleep,
(c) separated by a device synchronize, (d) separated by GPU work (a GEMM loop) on the compute stream."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gockpt_inputs as gi  # noqa: E402
import paper_2511_07035_b200 as G  # noqa: E402


def evict_all_cores(bufs):
    # one thread per core, pinned, each writes its own buffer (> its L2 + a share of L3): every
    # core's private caches drop the arena lines the replay threads left there
    import threading

    def work(c, b):
        os.sched_setaffinity(0, {c})
        b += 1

    ts = [threading.Thread(target=work, args=(c, b)) for c, b in zip(sorted(os.sched_getaffinity(0)), bufs)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def run(mode, n=1 << 20, K=4, sessions=6, evict_mb=0, **kw):
    evict = [np.zeros(evict_mb << 18, dtype=np.float32) for _ in os.sched_getaffinity(0)] if evict_mb else None
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(1, n)
    p, m, v = (torch.from_numpy(x.copy()).cuda() for x in (p0, m0, v0))
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = torch.from_numpy(gi.grad_bits(1, 1, n).view(np.int16).copy()).cuda()
    ctx = G.GoCkpt(p, m, v, out, **hp, k_min=1, k_max=16, part_align=1024, **kw)
    a = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
    step = 0
    rows, host, syncs = [], [], []
    for s_ in range(sessions):
        ctx.begin_checkpoint(step, K)
        for i in range(1, K + 1):
            step += 1
            if mode == "sleep":
                time.sleep(0.0005)
            elif mode == "sync":
                t = time.perf_counter()
                torch.cuda.synchronize()
                if i > 1:
                    syncs.append((time.perf_counter() - t) * 1e6)
            elif mode == "gemm":
                for _ in range(8):
                    a @ a
            t = time.perf_counter()
            ctx.submit(i, step, step, 1e-3, g)
            host.append((time.perf_counter() - t) * 1e6)
            if mode == "sync" and i == K:
                t = time.perf_counter()
                torch.cuda.synchronize()
                syncs.append((time.perf_counter() - t) * 1e6)
        ctx.finalize()
        if s_ >= 2:
            rows.append([{k: round(r[k] * 1e3, 1) for k in ("wait_ms", "kernel_ms", "d2h_ms")} for r in ctx.session_steps()])
        ctx.release()
        torch.cuda.synchronize()
        if evict is not None:
            evict_all_cores(evict)
    ctx.close()
    return {"mode": mode, "evict_mb": evict_mb, **{k: str(v) for k, v in kw.items()}, "host_submit_us_median": float(np.median(host)),
            "sync_wall_us": [round(x, 1) for x in syncs[-8:]],
            "steps_us": rows}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    modes = sys.argv[1:] or ["b2b", "sleep", "sync", "gemm"]
    for mode in modes:
        print(json.dumps(run(mode)), flush=True)
        print(json.dumps(run(mode, evict_mb=64)), flush=True)
        print(json.dumps(run(mode, verify_drain=False)), flush=True)
        print(json.dumps(run(mode, evict_mb=64, verify_drain=False)), flush=True)

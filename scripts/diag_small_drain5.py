"""Diagnostic 5: CUPTI device trace (CUDA activity only) of six small sessions in 'sync' mode, next
to the library's own per-step events: memcpy durations/bytes per session step."""
import json
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gockpt_inputs as gi  # noqa: E402
import paper_2511_07035_b200 as G  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n, K = 1 << 20, 4
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(1, n)
    p, m, v = (torch.from_numpy(x.copy()).cuda() for x in (p0, m0, v0))
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = torch.from_numpy(gi.grad_bits(1, 1, n).view(np.int16).copy()).cuda()
    ctx = G.GoCkpt(p, m, v, out, **hp, k_min=1, k_max=16, part_align=1024, verify_drain=False)
    step = 0
    logs = []
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for s_ in range(6):
            ctx.begin_checkpoint(step, K)
            for i in range(1, K + 1):
                step += 1
                torch.cuda.synchronize()
                ctx.submit(i, step, step, 1e-3, g)
            ctx.finalize()
            logs.append([round(r["d2h_ms"] * 1e3, 1) for r in ctx.session_steps()])
            ctx.release()
            torch.cuda.synchronize()
    ctx.close()
    prof.export_chrome_trace("gpurun_out/diag/trace5.json")
    print(json.dumps({"event_d2h_us": logs}))
    tr = json.load(open("gpurun_out/diag/trace5.json"))
    rows = [(e["ts"], e["dur"], e["name"], e.get("args", {}).get("bytes"), e.get("args", {}).get("stream"))
            for e in tr["traceEvents"] if e.get("cat") in ("gpu_memcpy", "kernel", "gpu_memset")]
    rows.sort()
    t0 = rows[0][0] if rows else 0
    for r in rows:
        print(json.dumps({"t_us": round(r[0] - t0, 1), "dur_us": r[1], "name": r[2][:50], "bytes": r[3], "stream": r[4]}))


if __name__ == "__main__":
    main()

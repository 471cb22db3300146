"""Diagnostic 3: standalone D2H copies (gck_d2h_copy, copy engine) of 512 KiB / 1 MiB into the
library's own pinned arena — the checkpoint arrays vs the gradient log — and into a torch pinned
buffer, each timed alone with CUDA events (repeated)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gockpt_inputs as gi  # noqa: E402
import paper_2511_07035_b200 as G  # noqa: E402


def tcopy(dst, src, nbytes, s, reps=10):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        G.d2h_copy(dst, src, nbytes, stream=s)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return round(ts[len(ts) // 2], 1)


def main():
    torch.cuda.set_device(0)
    n, K = 1 << 20, 4
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(1, n)
    p, m, v = (torch.from_numpy(x.copy()).cuda() for x in (p0, m0, v0))
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = torch.from_numpy(gi.grad_bits(1, 1, n).view(np.int16).copy()).cuda()
    ctx = G.GoCkpt(p, m, v, out, **hp, k_min=1, k_max=16, part_align=1024, eager_replay=False)
    for i in range(1, K + 1):
        if i == 1:
            ctx.begin_checkpoint(0, K)
        ctx.submit(i, i, i, 1e-3, g)
    ctx.wait_drained()
    st = ctx.staged()
    s = torch.cuda.Stream()
    src = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    pin = torch.empty(4 << 20, dtype=torch.uint8, pin_memory=True)
    for nb in (512 << 10, 1 << 20):
        res[f"torch_pinned_{nb}"] = tcopy(pin, src, nb, s)
        res[f"arena_master_{nb}"] = tcopy(torch.from_numpy(st["master"].view(np.uint8)), src, nb, s)
        res[f"arena_v_{nb}"] = tcopy(torch.from_numpy(st["exp_avg_sq"].view(np.uint8)), src, nb, s)
        for j, gl in enumerate(st["glog"]):
            res[f"arena_glog{j}_{nb}"] = tcopy(torch.from_numpy(gl.view(np.uint8)), src, min(nb, gl.nbytes), s)
    addrs = {"master": st["master"].ctypes.data, "v": st["exp_avg_sq"].ctypes.data,
             **{f"glog{j}": gl.ctypes.data for j, gl in enumerate(st["glog"])}}
    res["addrs_hex"] = {k: hex(a) for k, a in addrs.items()}
    # where does the slowness live: the first bytes of each glog slice, page by page
    gl = st["glog"][0].view(np.uint8)
    res["glog0_by_64k"] = [tcopy(torch.from_numpy(gl[o:o + (64 << 10)]), src, 64 << 10, s, reps=5)
                           for o in range(0, min(gl.nbytes, 512 << 10), 64 << 10)]
    res["master_by_64k"] = [tcopy(torch.from_numpy(st["master"].view(np.uint8)[o:o + (64 << 10)]), src, 64 << 10, s,
                                  reps=5) for o in range(0, 512 << 10, 64 << 10)]
    print(json.dumps(res))
    ctx.finalize()
    ctx.release()
    ctx.close()


if __name__ == "__main__":
    main()

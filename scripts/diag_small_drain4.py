"""Diagnostic 4: D2H copies out of the HBM staging ring (caller-owned, so its address is known)
after a session has packed it: state section vs gradient section of slot 0, standalone, timed with
CUDA events; then the same right after a fused step re-packs the slot."""
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
    return [round(ts[len(ts) // 2], 1), round(ts[0], 1), round(ts[-1], 1)]


def main():
    torch.cuda.set_device(0)
    n, K = 1 << 20, 4
    hp = dict(beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    p0, m0, v0 = gi.warm_state(1, n)
    p, m, v = (torch.from_numpy(x.copy()).cuda() for x in (p0, m0, v0))
    out = torch.zeros(n, dtype=torch.int16, device="cuda")
    g = torch.from_numpy(gi.grad_bits(1, 1, n).view(np.int16).copy()).cuda()
    rb = G.ring_bytes_required(n, 1, 16, 1024, 2)
    ring = torch.zeros(rb, dtype=torch.uint8, device="cuda")
    ctx = G.GoCkpt(p, m, v, out, **hp, k_min=1, k_max=16, part_align=1024, eager_replay=False, ring=ring,
                   verify_drain=False)
    ctx.begin_checkpoint(0, K)
    for i in range(1, K + 1):
        ctx.submit(i, i, i, 1e-3, g)
    ctx.wait_drained()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    pin = torch.empty(4 << 20, dtype=torch.uint8, pin_memory=True)
    pe = n // K
    st = 4 * pe  # 1 MiB, 256-aligned
    res = {"ring_bytes": rb}
    res["ring_state_1MiB"] = tcopy(pin, ring[0:], st, s)
    res["ring_grad_512KiB"] = tcopy(pin, ring[3 * st:], 2 * pe, s)
    res["ring_slot1_state_1MiB"] = tcopy(pin, ring[rb // 2:], st, s)
    res["ring_slot1_grad_1MiB"] = tcopy(pin, ring[rb // 2 + 3 * st:], 4 * pe, s)
    other = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
    res["other_1MiB"] = tcopy(pin, other, st, s)
    res["other_512KiB"] = tcopy(pin, other, 2 * pe, s)
    res["g_input_512KiB"] = tcopy(pin, g.view(torch.uint8), 2 * pe, s)
    res["whole_slot0"] = tcopy(pin, ring, 3 * st + 2 * pe, s)
    ctx.finalize()
    ctx.release()
    # the same copies right after a plain fused step (the slot untouched) and after a copy of g
    ctx.submit(0, 5, 5, 1e-3, g)
    torch.cuda.synchronize()
    res["after_plain_ring_grad_512KiB"] = tcopy(pin, ring[3 * st:], 2 * pe, s)
    print(json.dumps(res))
    ctx.close()


if __name__ == "__main__":
    main()

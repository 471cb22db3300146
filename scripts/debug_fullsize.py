"""Debug: run a full-size session and locate mismatches (staged vs oracle, live vs oracle, ckpt vs snapshot)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gockpt_inputs as gi  # noqa: E402
import oracle  # noqa: E402
import paper_2511_07035_b200 as G  # noqa: E402
from gpu_helpers import HP, down_f32  # noqa: E402

n = int(os.environ.get("N", 842_301_952))
K, t0, seed, LR = 8, 200, 7, 3e-4
dev = torch.device("cuda", 0)
p = torch.empty(n, dtype=torch.float32, device=dev)
m, v = torch.empty_like(p), torch.empty_like(p)
out = torch.empty(n, dtype=torch.int16, device=dev)
G.h_generate(1, p, seed, 0, 0, 0)
G.h_generate(2, m, seed)
G.h_generate(3, v, seed)
g = torch.empty(n, dtype=torch.int16, device=dev)
ctx = G.GoCkpt(p, m, v, out, **HP, k_min=K, k_max=K, eager_replay=False)
parts = G.plan_parts(n, K, 1024)
ctx.begin_checkpoint(t0, K)
lives = []
for i in range(1, K + 1):
    s = t0 + i
    G.h_generate(4, g, seed, s, 0, 1, 4)
    if i == K:
        snap = ctx.sync_snapshot()
    ctx.submit(i, s, s, LR, g)
torch.cuda.synchronize()
live = (down_f32(p), down_f32(m), down_f32(v))
ctx.wait_drained()
st = ctx.staged()
staged = [st[k].copy() for k in ("master", "exp_avg", "exp_avg_sq")]
ck = ctx.finalize()
ckpt = [ck.master.copy(), ck.exp_avg.copy(), ck.exp_avg_sq.copy()]
bad = np.zeros(n, bool)
for a, b in zip(ckpt, snap):
    bad |= a.view(np.uint32) != b.view(np.uint32)
idx = np.flatnonzero(bad)
print("ckpt vs snap mismatches:", idx.size, idx[:10], idx[-5:] if idx.size else "")
if idx.size:
    print("tiles:", np.unique(idx // 2048)[:20], "offsets in tile:", np.unique(idx % 2048)[:40])
    u = idx.astype(np.uint64)
    p0, m0, v0 = gi.warm_state(seed, u)
    grads = [gi.grad_bits(seed, t0 + i, u) for i in range(1, K + 1)]
    recs = [oracle.make_step_record(t=t0 + i, lr=LR, **HP) for i in range(1, K + 1)]
    traj = oracle.trajectory(p0, m0, v0, grads, recs)
    for nm, j in (("master", 0), ("m", 1), ("v", 2)):
        print(nm, "snap ok:", np.mean(snap[j][idx].view(np.uint32) == traj[K - 1][j].view(np.uint32)),
              "ckpt ok:", np.mean(ckpt[j][idx].view(np.uint32) == traj[K - 1][j].view(np.uint32)),
              "live ok:", np.mean(live[j][idx].view(np.uint32) == traj[K][j].view(np.uint32)))
    # staged: which part, version S(t0+i-1)
    part = np.searchsorted([hi for lo, hi in parts], idx, side="right")
    for j, nm in enumerate(("master", "m", "v")):
        ok = [staged[j][e] == traj[pi][j][q] for q, (e, pi) in enumerate(zip(idx, part))]
        print("staged", nm, "ok frac", np.mean(ok))
    print("parts of bad:", np.unique(part))

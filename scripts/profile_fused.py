"""Drive fused_adamw_pack at the bench config for ncu (3 plain launches, then a K=8 session).

ncu --set full --clock-control none --import-source on -k regex:fused_adamw_pack -s 2 -c 3 \
    -o gpurun_out/fused python scripts/profile_fused.py
captures launch 3 (plain, 28 B/element) and launches 4-5 (session parts 1-2, + pack bytes).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_07035_b200 as G  # noqa: E402

n = int(os.environ.get("GCK_N", 124_439_808))
K = 8
dev = torch.device("cuda", 0)
p = torch.empty(n, dtype=torch.float32, device=dev)
m, v = torch.empty_like(p), torch.empty_like(p)
out = torch.empty(n, dtype=torch.int16, device=dev)
g = torch.empty(n, dtype=torch.int16, device=dev)
G.h_generate(1, p, 42, 0, 0, 1)
G.h_generate(2, m, 42)
G.h_generate(3, v, 42)
G.h_generate(4, g, 42, 1, 0, 1, 4)
ctx = G.GoCkpt(p, m, v, out, k_min=K, k_max=K, timing=False)
step = 0
for _ in range(3):
    step += 1
    ctx.submit(0, step, 100 + step, 3e-4, g)
ctx.begin_checkpoint(step, K)
for i in range(1, K + 1):
    step += 1
    ctx.submit(i, step, 100 + step, 3e-4, g)
ck = ctx.finalize()
ctx.release()
torch.cuda.synchronize()
print("profile driver done, checkpoint step", ck.step)

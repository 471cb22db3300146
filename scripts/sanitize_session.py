"""A small full session for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
n just above the TMA threshold, ring + direct staging, plain + session launches, GPU replay."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_07035_b200 as G  # noqa: E402

n = int(os.environ.get("GCK_N", (1 << 18) + 2048 * 3 + 5))
K = 4
for staging in ("ring", "direct"):
    p = torch.empty(n, dtype=torch.float32, device="cuda")
    m, v = torch.empty_like(p), torch.empty_like(p)
    out = torch.empty(n, dtype=torch.int16, device="cuda")
    g = torch.empty(n, dtype=torch.int16, device="cuda")
    G.h_generate(1, p, 3, 0, 0, 0)
    G.h_generate(2, m, 3)
    G.h_generate(3, v, 3)
    ctx = G.GoCkpt(p, m, v, out, k_min=K, k_max=K, eager_replay=False, staging=staging,
                   verify_drain=os.environ.get("GCK_SANITIZE_VERIFY", "1") != "0")
    s = 0
    for _ in range(2):
        s += 1
        G.h_generate(4, g, 3, s, 0, 1, 4)
        ctx.submit(0, s, s, 1e-3, g)
    ctx.begin_checkpoint(s, K)
    for i in range(1, K + 1):
        s += 1
        ctx.grad_fence()
        G.h_generate(4, g, 3, s, 0, 1, 4)
        ctx.submit(i, s, s, 1e-3, g)
    ctx.wait_drained()
    dP, dM, dV = (torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3))
    dG = torch.empty(n * K + 1024, dtype=torch.int16, device="cuda")
    ctx.replay_gpu(dP, dM, dV, dG)
    ck = ctx.finalize()
    ctx.release()
    ctx.close()
torch.cuda.synchronize()
print("sanitize session ok")

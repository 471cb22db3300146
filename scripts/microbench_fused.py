"""Time fused_adamw_pack alone at the bench size (plain and session launches), CUDA events.

Env GCK_FUSED_IMPL / GCK_TMA_CFG select kernel variants (experiments). Prints one JSON line.
"""
import json
import os
import statistics
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
ctx = G.GoCkpt(p, m, v, out, k_min=K, k_max=K, timing=True)
step = 0


GEMM = os.environ.get("GCK_MB_GEMM") == "1"   # run a GEMM burst before each launch (power-capped clocks)
if GEMM:
    A = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    B = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)


def burst():
    if GEMM:
        for _ in range(8):
            torch.mm(A, B)


def plain(reps):
    global step
    ts = []
    for _ in range(reps):
        step += 1
        burst()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.submit(0, step, 100 + step, 3e-4, g)
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ts]


plain(5)
t_plain = plain(30)
sessions = []
for _ in range(3):
    ctx.begin_checkpoint(step, K)
    s0 = ctx.stats()
    for i in range(1, K + 1):
        step += 1
        burst()
        ctx.submit(i, step, 100 + step, 3e-4, g)
    ctx.finalize()
    s1 = ctx.stats()
    ctx.release()
    sessions.append((s1["kernel_ms_total"] - s0["kernel_ms_total"]) / K)
# per-part session launch times with every drain finished first (no slot wait inside the bracket)
per_part = []
ctx.begin_checkpoint(step, K)
for i in range(1, K + 1):
    step += 1
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.submit(i, step, 100 + step, 3e-4, g)
    b.record()
    torch.cuda.synchronize()
    per_part.append(a.elapsed_time(b) * 1e3)
ctx.finalize()
ctx.release()
parts = G.plan_parts(n, K, 1024)
sess_bytes = sum(12 * (hi - lo) + (2 * hi if i < K - 1 else 0) for i, (lo, hi) in enumerate(parts))
mean = statistics.mean(t_plain)
print(json.dumps({"impl": os.environ.get("GCK_FUSED_IMPL", "auto"), "cfg": os.environ.get("GCK_TMA_CFG", "default"),
                  "gemm_burst": GEMM,
                  "plain_us_mean": mean * 1e3, "plain_us_min": min(t_plain) * 1e3,
                  "plain_gbs": 28 * n / (mean / 1e3) / 1e9, "plain_gbs_best": 28 * n / (min(t_plain) / 1e3) / 1e9,
                  "session_us_mean": statistics.mean(sessions) * 1e3,
                  "session_gbs": (28 * n + sess_bytes / K) / (statistics.mean(sessions) / 1e3) / 1e9,
                  "per_part_us": [round(x, 1) for x in per_part],
                  "per_part_gbs": [round((28 * n + 12 * (hi - lo) + (2 * hi if i < K - 1 else 0)) / (t * 1e-6) / 1e9)
                                   for i, ((lo, hi), t) in enumerate(zip(parts, per_part))]}))

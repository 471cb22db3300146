"""a5 GPU variant: time the replay kernel (gck_replay_device) at the bench shard size, K = 8, and report
its HBM roofline: algorithmic bytes = sum_{j<K} |P_j| (24 + 2 (K - j)) per launch."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_07035_b200 as G  # noqa: E402

n = int(os.environ.get("GCK_N", 124_439_808))
K = int(os.environ.get("GCK_K", 8))
parts = G.plan_parts(n, K, 1024)
recs = [G.make_step_record(0.9, 0.999, 1e-8, 0.01, 100 + i, 3e-4) for i in range(1, K + 1)]
p = torch.empty(n, dtype=torch.float32, device="cuda")
m, v = torch.empty_like(p), torch.empty_like(p)
G.h_generate(1, p, 1, 0, 0, 1)
G.h_generate(2, m, 1)
G.h_generate(3, v, 1)
glog = []
for i in range(K - 1):
    t = torch.empty(parts[i][1], dtype=torch.int16, device="cuda")
    G.h_generate(4, t, 1, 101 + i, 0, 1, 4)
    glog.append(t)
alg = sum((hi - lo) * (24 + 2 * (K - 1 - j)) for j, (lo, hi) in enumerate(parts[:-1]))
from paper_2511_07035_b200.harness import ClockSampler  # noqa: E402
clocks = ClockSampler(0).start()
ts = []
for it in range(22):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    G.replay_device(recs, parts, p, m, v, glog)
    b.record()
    torch.cuda.synchronize()
    if it >= 2:
        ts.append(a.elapsed_time(b))
mean = statistics.mean(ts) / 1e3
clk = clocks.stop()
print(json.dumps({"n": n, "K": K, "element_updates": sum((hi - lo) * (K - 1 - j) for j, (lo, hi) in enumerate(parts[:-1])),
                  "alg_bytes": alg, "us_mean": mean * 1e6, "us_min": min(ts) * 1e3, "sm_mhz": clk.get("sm_mhz"), "gbs": alg / mean / 1e9, "frac_of_6500": alg / mean / 1e9 / 6500.6}))

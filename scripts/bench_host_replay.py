"""a5 host replay scaling (SURVEY §8(d) CPU plan): gck_replay_host on a staged GPT-2 (K=8) session at
1..all threads, with the host-DRAM roofline (STREAM triad, scripts/c/triad.c) measured on the same box.
Algorithmic host bytes per session: sum_{j<K} |P_j| (24 + 2 (K - j)); element-updates n(K-1)/2."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import gockpt_inputs as gi  # noqa: E402
import paper_2511_07035_b200 as G  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
exe = "/tmp/gck_triad"
subprocess.run(["gcc", "-O3", "-march=native", "-fopenmp", os.path.join(here, "c", "triad.c"), "-o", exe], check=True)
n = int(os.environ.get("GCK_N", 124_439_808))
K = int(os.environ.get("GCK_K", 8))
parts = G.plan_parts(n, K, 1024)
recs = [G.make_step_record(0.9, 0.999, 1e-8, 0.01, 100 + i, 3e-4) for i in range(1, K + 1)]
base = [x for x in gi.warm_state(1, n)]
glog = [gi.grad_bits(1, 101 + i, parts[i][1]) for i in range(K - 1)]
alg = sum((hi - lo) * (24 + 2 * (K - 1 - j)) for j, (lo, hi) in enumerate(parts[:-1]))
upd = sum((hi - lo) * (K - 1 - j) for j, (lo, hi) in enumerate(parts[:-1]))
cores = len(os.sched_getaffinity(0))
out = {"n": n, "K": K, "alg_bytes": alg, "element_updates": upd, "cores": cores, "runs": []}
for T in sorted({1, 2, 4, 8, 16, cores}):
    if T > cores:
        continue
    tri = json.loads(subprocess.run([exe, str(T)], capture_output=True, text=True).stdout)
    best = 1e9
    for _ in range(3):
        p, m, v = (x.copy() for x in base)
        t0 = time.perf_counter()
        G.replay_host(recs, parts, p, m, v, glog, threads=T)
        best = min(best, time.perf_counter() - t0)
    out["runs"].append({"threads": T, "ms": best * 1e3, "gbs": alg / best / 1e9, "gupd_s": upd / best / 1e9,
                        "triad_gbs": tri["triad_gbs"], "frac_of_triad": alg / best / 1e9 / tri["triad_gbs"]})
print(json.dumps(out))

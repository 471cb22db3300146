"""NEXT-1 measurement: persist (multithreaded write + CRC + fsync + atomic publish) and restore
(read + CRC verify + H2D + bf16 re-derivation) throughput at the bench shard sizes.

python scripts/bench_persist.py --dir /tmp/gck_persist [--n 124439808] [--threads 16] [--replay-mode deferred]

--replay-mode deferred (NEXT-2 replay-on-restore): finalize does no replay, the file carries the
captured parts + gradient log (version 2), and the restore replays on the GPU.
"""
import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_07035_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dir", default="/tmp/gck_persist")
ap.add_argument("--n", type=int, default=124_439_808)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--K", type=int, default=8)
ap.add_argument("--replay-mode", default="host", choices=["host", "gpu", "deferred"])
args = ap.parse_args()
os.makedirs(args.dir, exist_ok=True)
n, K = args.n, args.K
dev = torch.device("cuda", 0)
p = torch.empty(n, dtype=torch.float32, device=dev)
m, v = torch.empty_like(p), torch.empty_like(p)
out = torch.empty(n, dtype=torch.int16, device=dev)
g = torch.empty(n, dtype=torch.int16, device=dev)
G.h_generate(1, p, 1, 0, 0, 1)
G.h_generate(2, m, 1)
G.h_generate(3, v, 1)
ctx = G.GoCkpt(p, m, v, out, k_min=K, k_max=K, replay_threads=args.threads, replay_mode=args.replay_mode,
               eager_replay=False)
ctx.begin_checkpoint(100, K)
for i in range(1, K + 1):
    G.h_generate(4, g, 1, 100 + i, 0, 1, 4)
    ctx.submit(i, 100 + i, 100 + i, 3e-4, g)
ctx.wait_drained()
tf = time.perf_counter()
ck = ctx.finalize()                      # the replay (host / gpu), or nothing (deferred)
finalize_s = time.perf_counter() - tf
path = os.path.join(args.dir, f"ckpt_{ck.step}.rank0.bin")
t0 = time.perf_counter()
ctx.persist_begin(path, 0, 1, None)
ps = ctx.persist_wait()
ctx.release()
os.system("sync")
# drop this file from the page cache if we may (root): a cold read measures the device, not RAM
cold = os.system("echo 1 > /proc/sys/vm/drop_caches 2>/dev/null") == 0
torch.cuda.synchronize()
t1 = time.perf_counter()
h = ctx.restore(path)
t2 = time.perf_counter()
usage = shutil.disk_usage(args.dir)
# the restored S(T) must be the same bytes in every replay mode: print its CRCs to compare runs
import zlib  # noqa: E402
restored_crc = [zlib.crc32(t.cpu().numpy().tobytes()) for t in (p, m, v)]
res = {"n": n, "K": K, "replay_mode": args.replay_mode, "finalize_s": finalize_s, "file_bytes": ps["bytes"], "persist_gbs": ps["gbs"], "persist_s": ps["seconds"],
       "persist_data_s": ps["data_seconds"], "threads": ps["threads"], "restore_s": t2 - t1,
       "restore_gbs": 12 * n / (t2 - t1) / 1e9, "page_cache_dropped": cold, "dir": args.dir,
       "fs_free_gb": usage.free / 1e9, "step": h["step"], "restored_crc": restored_crc}
print(json.dumps(res))
ctx.close()
os.unlink(path)
